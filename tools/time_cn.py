"""CUDA-event time of the CN right-hand side and H update kernels on a 256^3 block:
python tools/time_cn.py [n=256] [reps=20]  (FMP_CN_RHS_PLANE=1: per-plane RHS kernel)."""
import json, sys, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import _lib
from paper_2508_07193_b200.plan import block_struct
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
E, H, R, Hn = (torch.rand(3, n, n, n, dtype=torch.float64, device="cuda") for _ in range(4))
blk = block_struct(n, n, n)
def rhs():
    _lib.call("fmp_cn_rhs", _lib.ref(blk), _lib.ref(blk), 0.1, _lib.ptr(E), _lib.ptr(H), _lib.ptr(R), _lib.stream())
def hup():
    _lib.call("fmp_cn_h_update", _lib.ref(blk), _lib.ref(blk), 0.1, _lib.ptr(H), _lib.ptr(E), _lib.ptr(R), _lib.ptr(Hn), _lib.stream())
out = {}
for name, f, nbytes in (("cn_rhs", rhs, 72), ("cn_h", hup, 96)):
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out[name + "_ms"] = round(ms, 4)
    out[name + "_tbs"] = round(nbytes * n ** 3 / ms / 1e9, 2)
print(json.dumps(out))

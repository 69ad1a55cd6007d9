"""SpMV (op.apply_into, mode 0) and fused-dot variants at cfg4 size: TMA kernel vs the legacy cp.async kernel."""
import json, os, sys, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, DistributedOperator
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
part = make_partition(Box(n, n, n), (n // 32,) * 3, 1)
op = DistributedOperator(part, 0.25, make_transport("cuda"))
x = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda")
w = torch.rand_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
ys = {}
for mode in ("legacy", "tma"):
    if mode == "legacy":
        os.environ["FMP_SPMV_LEGACY"] = "1"
    else:
        os.environ.pop("FMP_SPMV_LEGACY", None)
    y = torch.empty_like(x)
    for _ in range(3): op.apply_into(x, y)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); op.apply_into(x, y); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[len(ts) // 2]
    out[mode + "_ms"] = t
    out[mode + "_GBs"] = 48 * n ** 3 / t / 1e6
    d = op.apply_dots(x, y, w, both=True)
    r = float(op.residual_norm2(x, w))
    out[mode + "_dots"] = d + [r]
    ys[mode] = y.clone()
out["max_abs_diff"] = float((ys["tma"] - ys["legacy"]).abs().max())
print(json.dumps(out))

"""Zero-slice skipping in the Ozaki GEMM is exact: RAS applies with FMP_OZ_DENSE=1 (every C^-1
slice block streamed and multiplied) and without (all-zero slice blocks skipped) must agree bit
for bit when both run whole tiles (FMP_OZ_NOSPLIT=1: no K segments, whose FP64 partial sums
depend on where the schedule cuts); prints the apply times of the default schedules too.  python tools/oz_sparse_check.py [subdomain=32] [n=256]"""
import json, os, sys, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, RasPreconditioner
sd = int(sys.argv[1]) if len(sys.argv) > 1 else 32
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
part = make_partition(Box(n, n, n), (n // sd,) * 3, 1)
tr = make_transport("cuda")
x = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(7))
out = {"subdomain": sd, "grid": n}
zs = {}
for mode in ("1", "0"):
    os.environ["FMP_OZ_DENSE"] = mode
    prec = RasPreconditioner(part, 0.25, tr)
    z = torch.empty_like(x)
    for _ in range(3):
        prec.apply_into(x, z)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10):
        prec.apply_into(x, z)
    e1.record(); torch.cuda.synchronize()
    out["apply_ms_dense" if mode == "1" else "apply_ms_sparse"] = round(e0.elapsed_time(e1) / 10, 4)
    zs[mode] = z.clone()
    del prec
out["default_schedules_max_abs_diff"] = float((zs["0"] - zs["1"]).abs().max())
os.environ["FMP_OZ_NOSPLIT"] = "1"
for mode in ("1", "0"):
    os.environ["FMP_OZ_DENSE"] = mode
    prec = RasPreconditioner(part, 0.25, tr)
    z = torch.empty_like(x)
    prec.apply_into(x, z)
    zs["ns" + mode] = z.clone()
    del prec
out["nosplit_bitwise_equal"] = bool(torch.equal(zs["ns0"], zs["ns1"]))
print(json.dumps(out))

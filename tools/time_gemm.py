"""Precond apply time with the own DMMA GEMM vs cuBLAS (cfg4)."""
import os, sys, json, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, RasPreconditioner
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
part = make_partition(Box(n, n, n), (n // 32,) * 3, 1)
tr = make_transport("cuda")
x = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda")
out = {}
zs = {}
for mode in ("ozaki", "cublas", "own"):
    os.environ["FMP_GEMM"] = mode
    prec = RasPreconditioner(part, 0.25, tr)
    z = torch.empty_like(x)
    for _ in range(3): prec.apply_into(x, z)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10): prec.apply_into(x, z)
    e1.record(); torch.cuda.synchronize()
    out[mode] = e0.elapsed_time(e1) / 10
    zs[mode] = z.clone()
    del prec
out["own_vs_cublas"] = float((zs["own"] - zs["cublas"]).abs().max() / zs["cublas"].abs().max())
out["ozaki_vs_cublas"] = float((zs["ozaki"] - zs["cublas"]).abs().max() / zs["cublas"].abs().max())
print(json.dumps(out))

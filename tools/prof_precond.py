"""Profiling driver: build the cfg4 (256^3, 32^3 subdomains) operator + preconditioner and run a
few applies, for ncu launch lists / full captures (never time under ncu)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, RasPreconditioner, DistributedOperator
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
part = make_partition(Box(n, n, n), (n // 32,) * 3, 1)
tr = make_transport("cuda")
prec = RasPreconditioner(part, 0.25, tr)
op = DistributedOperator(part, 0.25, tr)
x = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda")
z = torch.empty_like(x)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measure")
for _ in range(3):
    prec.apply_into(x, z)
    op.apply_into(x, z)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")

"""Profiling driver for config 5's 64^3 subdomains (256^3 block, 4x4x4 subdomains of ext 65/66):
a few RAS applies inside the NVTX range "measure"."""
import sys, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, RasPreconditioner
n, sd = 256, int(sys.argv[1]) if len(sys.argv) > 1 else 64
part = make_partition(Box(n, n, n), (n // sd,) * 3, 1)
prec = RasPreconditioner(part, 0.25, make_transport("cuda"))
x = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda")
z = torch.empty_like(x)
prec.apply_into(x, z)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measure")
for _ in range(2):
    prec.apply_into(x, z)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")

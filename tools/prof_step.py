"""Profiling driver: one cfg4 CN-FDTD step (256^3, 32^3 subdomains, BiCGSTAB + RAS) inside the NVTX
range "measure", after one warm-up step, for ncu launch lists (never time under ncu)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, CnSolver, DeviceCnStepper, SolverConfig, make_transport
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
solver = CnSolver(Box(n, n, n), (n // 32,) * 3, 1, 0.25, SolverConfig(), make_transport("cuda"))
g = torch.Generator(device="cuda").manual_seed(42)
E = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
H = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
st = DeviceCnStepper(solver, E, H, 1.0)
st.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measure")
rep = st.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("iterations", rep.iterations)

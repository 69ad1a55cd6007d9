"""HostStepPipeline steady state: ms per step for K independent host-field CN steps (cfg4), and
the same with the device->host copies or the host->device copies alone, to see what serialises."""
import json, sys, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, CnSolver, HostStepPipeline, SolverConfig, make_transport
n = 256
solver = CnSolver(Box(n, n, n), (8, 8, 8), 1, 0.25, SolverConfig(), make_transport("cuda"))
g = torch.Generator(device="cuda").manual_seed(42)
E0 = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
H0 = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
Eh, Hh = E0.cpu().pin_memory(), H0.cpu().pin_memory()
Eo, Ho = torch.empty_like(Eh).pin_memory(), torch.empty_like(Hh).pin_memory()
pipe = HostStepPipeline(solver, 1.0)
pipe.run(Eh, Hh, Eo, Ho, steps=2)
out = {}
for k in [int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2", "4", "8", "12", "16"])]:
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    pipe.run(Eh, Hh, Eo, Ho, steps=k)
    a1.record()
    torch.cuda.synchronize()
    out[k] = round(a0.elapsed_time(a1) / k, 2)
print(json.dumps({"ms_per_step_by_K": out, "mem_alloc_GB": round(torch.cuda.memory_allocated() / 1e9, 1),
                  "mem_reserved_GB": round(torch.cuda.memory_reserved() / 1e9, 1)}))

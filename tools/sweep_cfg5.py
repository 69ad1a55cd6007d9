"""BASELINE config 5 on one GPU: subdomain-size sweep (16^3 / 32^3 / 64^3) at 256^3 per GPU,
GMRES(30) vs BiCGSTAB, iteration count vs time (the 8-GPU 512^3 run is the same per-GPU block).
One CN step per case after one warm-up step; prints one JSON line per case."""
import json, sys, time
import torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, SolverConfig
from paper_2508_07193_b200.cn_driver import CnSolver, DeviceCnStepper
from paper_2508_07193_b200.schwarz import make_transport

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
subs = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16, 32, 64]
methods = sys.argv[3].split(",") if len(sys.argv) > 3 else ["bicgstab", "gmres"]
dt = 1.0
for sd in subs:
    for method in methods:
        t0 = time.perf_counter()
        solver = CnSolver(Box(n, n, n), (n // sd,) * 3, 1, dt * dt / 4, SolverConfig(method=method),
                          make_transport("cuda"))
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        g = torch.Generator(device="cuda").manual_seed(42)
        E = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        H = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        st = DeviceCnStepper(solver, E, H, dt)
        st.step()
        torch.cuda.synchronize()
        times = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rep = st.step()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = min(times)
        print(json.dumps({"grid": n, "subdomain": sd, "method": method, "iters": rep.iterations,
                          "final_relres": rep.final_relres, "step_ms": round(ms, 3),
                          "mdofs": round(3 * n ** 3 / ms / 1e3, 1), "setup_s": round(setup, 2),
                          "gemm": "ozaki (2 K parts)" if sd >= 64 else "ozaki"}), flush=True)
        del st, solver
        torch.cuda.empty_cache()

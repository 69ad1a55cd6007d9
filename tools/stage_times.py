"""Per-stage CUDA-event times of one RAS apply at 256^3 (fmp_precond_profile), averaged over
reps, plus the whole apply: python tools/stage_times.py [subdomain=32] [reps=10]."""
import json, sys, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, RasPreconditioner
n, sd = 256, int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
prec = RasPreconditioner(make_partition(Box(n, n, n), (n // sd,) * 3, 1), 0.25, make_transport("cuda"))
x = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda")
z = torch.empty_like(x)
for _ in range(3):
    prec.apply_into(x, z)
acc = {}
prec.plan.profile(True)
for _ in range(reps):
    prec.apply_into(x, z)
    for k, v in prec.plan.stage_ms().items():
        acc[k] = acc.get(k, 0.0) + v / reps
prec.plan.profile(False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(reps):
    prec.apply_into(x, z)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"subdomain": sd, "apply_ms": round(e0.elapsed_time(e1) / reps, 4),
                  **{k: round(v, 4) for k, v in acc.items()}}))

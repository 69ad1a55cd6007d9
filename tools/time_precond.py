"""CUDA-event timing of one RAS apply and one SpMV at cfg4 size (no profiler)."""
import sys, json, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, RasPreconditioner, DistributedOperator
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
part = make_partition(Box(n, n, n), (n // 32,) * 3, 1)
tr = make_transport("cuda")
prec = RasPreconditioner(part, 0.25, tr)
op = DistributedOperator(part, 0.25, tr)
x = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda")
z = torch.empty_like(x)
def t(fn, reps=10):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
print(json.dumps({"precond_ms": t(lambda: prec.apply_into(x, z)), "spmv_ms": t(lambda: op.apply_into(x, z))}))

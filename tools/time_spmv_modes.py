"""SpMV modes at cfg4 (256^3): y = A x (0), + (w, y) (1), + (w, y), (y, y) (2), ||w - A x||^2 (3);
median of 20 CUDA-event timings each with an L2 flush in between.  python tools/time_spmv_modes.py"""
import json, sys, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, DistributedOperator
n = 256
op = DistributedOperator(make_partition(Box(n, n, n), (8, 8, 8), 1), 0.25, make_transport("cuda"))
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g)
w = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g)
y = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
calls = {0: lambda: op.apply_into(x, y), 1: lambda: op._run(1, x, y, w), 2: lambda: op._run(2, x, y, w),
         3: lambda: op._run(3, x, None, w)}
out = {}
for m, f in calls.items():
    for _ in range(3):
        f()
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[f"mode{m}_us"] = round(sorted(ts)[10] * 1000, 1)
op.apply_into(x, y)
out["y_checksum"] = float(y.double().sum())
out["dots"] = op.apply_dots(x, y, w, both=True) + [float(op.residual_norm2(x, w))]
print(json.dumps(out))

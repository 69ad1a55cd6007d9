"""cuBLAS DGEMM peak probe (FP64 roofline denominator; MEASURED_PEAKS.json has no FP64 entry)."""
import json, torch
def t(m, n, k, reps=10):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda"); b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return 2.0 * m * n * k / (best * 1e-3) / 1e12, best
out = {}
for name, (m, n, k) in {"8192^3": (8192, 8192, 8192), "woodbury_6834x216": (6834, 216, 6834),
                        "woodbury_6048x512": (6048, 512, 6048), "woodbury_6834x64": (6834, 64, 6834)}.items():
    tf, ms = t(m, n, k)
    out[name] = {"tflops": round(tf, 2), "ms": round(ms, 4)}
print(json.dumps(out))

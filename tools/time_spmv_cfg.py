"""SpMV timing for the bulk kernel's ring configurations (FMP_SPMV_NS4) and the legacy kernel."""
import json, os, sys, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, DistributedOperator
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
part = make_partition(Box(n, n, n), (n // 32,) * 3, 1)
op = DistributedOperator(part, 0.25, make_transport("cuda"))
x = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda")
w = torch.rand_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out, ys = {}, {}
for cfg, env in (("legacy", {"FMP_SPMV_LEGACY": "1"}), ("ns6", {"FMP_SPMV_NS6": "1"}), ("ns4", {})):
    for k in ("FMP_SPMV_LEGACY", "FMP_SPMV_NS6"):
        os.environ.pop(k, None)
    os.environ.update(env)
    y = torch.empty_like(x)
    for _ in range(3): op.apply_into(x, y)
    for name, fn in (("spmv", lambda: op.apply_into(x, y)), ("dots2", lambda: op.apply_dots(x, y, w, both=True)),
                     ("resid", lambda: op.residual_norm2(x, w))):
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[f"{cfg}_{name}_us"] = round(sorted(ts)[5] * 1e3, 1)
    op.apply_into(x, y)
    out[f"{cfg}_spmv_GBs"] = round(48 * n ** 3 / out[f"{cfg}_spmv_us"] / 1e3, 1)
    ys[cfg] = (y.clone(), op.apply_dots(x, y, w, both=True), float(op.residual_norm2(x, w)))
for cfg in ("ns6", "ns4"):
    out[f"{cfg}_maxdiff"] = float((ys[cfg][0] - ys["legacy"][0]).abs().max())
    out[f"{cfg}_dots"] = ys[cfg][1] + [ys[cfg][2]]
out["legacy_dots"] = ys["legacy"][1] + [ys["legacy"][2]]
print(json.dumps(out))

"""MMA-warp timeline of the Ozaki GEMM (FMP_OZ_PROF=1): per CTA total cycles, cycles waiting
for operand stages and for the epilogue, over one RAS apply at 256^3 / 32^3 subdomains."""
import ctypes, json, os, sys
os.environ["FMP_OZ_PROF"] = "1"
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, RasPreconditioner
from paper_2508_07193_b200 import _lib
sd = int(sys.argv[1]) if len(sys.argv) > 1 else 32
prec = RasPreconditioner(make_partition(Box(256, 256, 256), (256 // sd,) * 3, 1), 0.25, make_transport("cuda"))
x = torch.rand(3, 256, 256, 256, dtype=torch.float64, device="cuda")
z = torch.empty_like(x)
for _ in range(3):
    prec.apply_into(x, z)
torch.cuda.synchronize()
lib = ctypes.CDLL(str(_lib.LIB_PATH))
buf = np.zeros((148, 8), dtype=np.int64)
assert lib.fmp_debug_ozaki_prof(buf.ctypes.data_as(ctypes.c_void_p), 148) == 0
tot, full, empty, tiles, ts, te, first = buf.T[:7]
t0 = ts.min()
busy = tot - full - empty
if os.environ.get("FMP_OZ_DUMP"):
    print(json.dumps({"per_cta": [[int(tot[i]), int(full[i]), int(empty[i]), int(ts[i] - t0), int(te[i] - t0)] for i in range(148)]}))
print(json.dumps({"ctas": 148, "total_max_us": round(tot.max() / 1965, 1), "total_mean_us": round(tot.mean() / 1965, 1),
                  "wait_full_mean_us": round(full.mean() / 1965, 1), "wait_full_first_chunk_mean_us": round(first.mean() / 1965, 1), "wait_epilogue_mean_us": round(empty.mean() / 1965, 1),
                  "issue_mean_us": round(busy.mean() / 1965, 1), "tiles_mean": float(tiles.mean()),
                  "wait_full_max_us": round(full.max() / 1965, 1),
                  "cta_start_spread_us": round((ts.max() - t0) / 1e3, 1), "cta_end_min_us": round((te.min() - t0) / 1e3, 1),
                  "cta_end_max_us": round((te.max() - t0) / 1e3, 1), "cta_span_mean_us": round((te - ts).mean() / 1e3, 1)}))

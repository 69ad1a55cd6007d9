"""Times the fused Krylov-update applies against their two-pass forms at cfg4 (256^3, 32^3
subdomains): apply, lincomb + apply vs fmp_precond_apply_lincomb, copy + bicg_p + apply vs
fmp_precond_apply_bicg_p (CUDA events, 20 back-to-back calls each, after warm-up)."""
import sys, json
import torch
sys.path.insert(0, ".")
from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport, _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
part = make_partition(Box(n, n, n), (n // 32,) * 3, 1)
prec = RasPreconditioner(part, 0.25, make_transport("cuda"))
g = torch.Generator(device="cuda").manual_seed(1)
r, v, p, s, z, p2 = (torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g) for _ in range(6))


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def two_pass_s():
    _lib.call("fmp_vec_lincomb", r.numel(), 1.0, _lib.ptr(r), -0.3, _lib.ptr(v), _lib.ptr(s), _lib.stream())
    prec.apply_into(s, z)


def two_pass_p():
    p2.copy_(p)
    _lib.call("fmp_bicg_p", r.numel(), _lib.ptr(r), _lib.ptr(p2), _lib.ptr(v), 0.4, 1.1, _lib.stream())
    prec.apply_into(p2, z)


out = {"apply": timed(lambda: prec.apply_into(r, z)),
       "lincomb+apply": timed(two_pass_s),
       "apply_lincomb (fused)": timed(lambda: prec.apply_lincomb_into(r, v, -0.3, s, z)),
       "copy+bicg_p+apply": timed(two_pass_p),
       "apply_bicg_p (fused)": timed(lambda: prec.apply_bicg_p_into(r, p, v, 0.4, 1.1, p2, z))}
print(json.dumps({k: round(t, 4) for k, t in out.items()}))

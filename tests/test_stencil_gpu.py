"""GPU parity: matrix-free stencils and Krylov vector kernels vs the oracle / reference goldens."""

import numpy as np
import pytest
import torch

import flashmp_oracle as O
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

EXTS = [(3, 3, 3), (4, 5, 6), (1, 3, 4), (8, 8, 8), (2, 7, 3)]


def rel(a, b):
    a, b = np.ravel(np.asarray(a)), np.ravel(np.asarray(b))
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dev(x, ext):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().view(3, ext[2], ext[1], ext[0])


@pytest.mark.parametrize("ext", EXTS)
def test_stencil_matches_reference(ext):
    from paper_2508_07193_b200.operators import stencil_apply
    from paper_2508_07193_b200 import apply_curl, apply_double_curl
    g = np.load(GOLDEN / "operators.npz")
    tag = "_".join(map(str, ext))
    x = dev(g[f"x_{tag}"], ext)
    assert rel(stencil_apply(x, 0.25, True).cpu(), g[f"A_{tag}"]) <= 1e-14
    assert rel(stencil_apply(x, 0.25, True).cpu(), g[f"Acsr_{tag}"]) <= 1e-14
    assert rel(stencil_apply(x, 0.25, False).cpu(), g[f"A0_{tag}"]) <= 1e-14
    assert rel(apply_curl("forward", x).cpu(), g[f"curlf_{tag}"]) <= 1e-15
    assert rel(apply_curl("backward", x).cpu(), g[f"curlb_{tag}"]) <= 1e-15
    assert rel(apply_double_curl(x).cpu(), g[f"M_{tag}"]) <= 1e-14


@pytest.mark.parametrize("ext", [(37, 9, 19), (64, 64, 64), (33, 34, 35)])
@pytest.mark.parametrize("boundary", [True, False])
def test_stencil_matches_oracle_larger(ext, boundary):
    from paper_2508_07193_b200.operators import stencil_apply
    x = np.random.default_rng(1).uniform(-1, 1, (3, ext[2], ext[1], ext[0]))
    got = stencil_apply(dev(x, ext), 0.25, boundary).cpu().numpy()
    want = O.apply_A(0.25, x, boundary)
    assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max()


def test_stencil_fused_dots_and_residual():
    from paper_2508_07193_b200 import _lib
    from paper_2508_07193_b200.plan import block_struct
    ext = (40, 24, 16)
    rng = np.random.default_rng(2)
    x, w = (rng.uniform(-1, 1, (3, ext[2], ext[1], ext[0])) for _ in range(2))
    X, W = dev(x, ext), dev(w, ext)
    Y = torch.empty_like(X)
    dots = torch.zeros(2, dtype=torch.float64, device="cuda")
    scratch = torch.zeros(int(_lib.lib().fmp_reduce_scratch_doubles()), dtype=torch.float64, device="cuda")
    blk = block_struct(*ext)
    y = O.apply_A(0.3, x, True)
    for mode in (1, 2, 3):
        _lib.call("fmp_stencil_apply", _lib.ref(blk), 0.3, 1, mode, X.data_ptr(),
                  Y.data_ptr() if mode < 3 else None, W.data_ptr(), dots.data_ptr(), scratch.data_ptr(),
                  _lib.stream())
        d = dots.cpu().numpy()
        if mode < 3:
            assert rel(Y.cpu(), y) <= 1e-14
            assert abs(d[0] - np.sum(y * w)) <= 1e-12 * np.sum(np.abs(y * w))
        if mode == 2:
            assert abs(d[1] - np.sum(y * y)) <= 1e-13 * np.sum(y * y)
        if mode == 3:
            assert abs(d[0] - np.sum((w - y) ** 2)) <= 1e-13 * np.sum((w - y) ** 2)


def test_stencil_symmetric_and_deterministic():
    """A is SPD: (Ax, y) == (x, Ay); repeated launches are bitwise equal."""
    from paper_2508_07193_b200.operators import stencil_apply
    ext = (48, 40, 32)
    rng = np.random.default_rng(3)
    x, y = (dev(rng.uniform(-1, 1, (3, ext[2], ext[1], ext[0])), ext) for _ in range(2))
    ax, ay = stencil_apply(x, 0.25), stencil_apply(y, 0.25)
    lhs, rhs = float((ax * y).sum()), float((x * ay).sum())
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    assert torch.equal(stencil_apply(x, 0.25), ax)


def test_vector_kernels_bitwise_numpy():
    from paper_2508_07193_b200 import _lib
    n = 1_000_003
    rng = np.random.default_rng(4)
    a, b, c, d, e, f = (rng.uniform(-1, 1, n) for _ in range(6))
    keep = []

    def T(v):  # keep every device copy alive until the kernels have run (no allocator reuse)
        t = torch.from_numpy(v.copy()).cuda()
        keep.append(t)
        return t

    st = _lib.stream()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.call("fmp_vec_lincomb", n, 0.7, T(a).data_ptr(), -1.3, T(b).data_ptr(), out.data_ptr(), st)
    assert np.array_equal(out.cpu().numpy(), 0.7 * a + -1.3 * b)
    y = T(b)
    _lib.call("fmp_vec_axpy", n, 0.37, T(a).data_ptr(), y.data_ptr(), st)
    bb = b.copy()
    bb += 0.37 * a
    assert np.array_equal(y.cpu().numpy(), bb)
    _lib.call("fmp_vec_scale", n, 1.0 / 3.0, T(a).data_ptr(), out.data_ptr(), st)
    assert np.array_equal(out.cpu().numpy(), (1.0 / 3.0) * a)
    # BiCGSTAB p update: p = 1.0*r + beta*(1.0*p + (-omega)*v)   (ref:krylov.py:181-182)
    p = T(b)
    _lib.call("fmp_bicg_p", n, T(a).data_ptr(), p.data_ptr(), T(c).data_ptr(), 0.9, 0.4, st)
    p1 = 1.0 * b + (-0.4) * c
    assert np.array_equal(p.cpu().numpy(), 1.0 * a + 0.9 * p1)
    # BiCGSTAB tail + next rho
    x, r = T(a), T(b)
    dots = torch.zeros(2, dtype=torch.float64, device="cuda")
    scratch = torch.zeros(int(_lib.lib().fmp_reduce_scratch_doubles()), dtype=torch.float64, device="cuda")
    _lib.call("fmp_bicg_xr", n, x.data_ptr(), T(c).data_ptr(), T(d).data_ptr(), T(e).data_ptr(), T(f).data_ptr(),
              r.data_ptr(), T(c).data_ptr(), 0.3, 0.6, dots.data_ptr(), scratch.data_ptr(), st)
    xx = a.copy()
    xx += 0.3 * c
    xx += 0.6 * d
    rr = 1.0 * e + (-0.6) * f
    assert np.array_equal(x.cpu().numpy(), xx)
    assert np.array_equal(r.cpu().numpy(), rr)
    assert abs(float(dots[0]) - float(c @ rr)) <= 1e-12 * np.sum(np.abs(c * rr))
    _lib.call("fmp_vec_dot", n, T(a).data_ptr(), T(b).data_ptr(), dots.data_ptr(), scratch.data_ptr(), st)
    assert abs(float(dots[0]) - float(a @ b)) <= 1e-12 * np.sum(np.abs(a * b))


def test_cn_stencils_match_reference():
    from paper_2508_07193_b200 import EmState, FieldVector, Box, build_rhs
    g = np.load(GOLDEN / "cn.npz")
    for gext, tag in [((8, 8, 8), "8_8_8_g111_o1"), ((16, 16, 16), "16_16_16_g222_o1")]:
        rng = np.random.default_rng(42)
        box = Box(*gext)
        E = FieldVector(box, rng.uniform(-1, 1, box.dof))
        H = FieldVector(box, rng.uniform(-1, 1, box.dof))
        R = build_rhs(EmState(E, H, 0, 1.0))
        assert rel(R.data, g[f"rhs_{tag}"]) <= 1e-14


def test_fused_dots_are_deterministic():
    """The SpMV's fused dot products do not depend on the dynamic unit scheduling: repeated
    launches give bitwise-identical sums (per-unit partials, fixed-order final reduction)."""
    from paper_2508_07193_b200 import Box, DistributedOperator, make_partition, make_transport
    n = 128
    op = DistributedOperator(make_partition(Box(n, n, n), (4, 4, 4), 1), 0.25, make_transport("cuda"))
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g)
    w = torch.rand_like(x)
    y = torch.empty_like(x)
    first = (op.apply_dots(x, y, w, both=True), op.residual_norm2(x, w))
    for _ in range(8):
        assert (op.apply_dots(x, y, w, both=True), op.residual_norm2(x, w)) == first


def test_double_curl_is_formed_directly():
    """apply_double_curl forms M x in the kernel with the identity dropped (FMP_STENCIL_NO_IDENTITY),
    not as (x + M x) - x.  Integer-valued fields make every stencil sum exact, so the result must
    equal the oracle bit for bit; on a nearly curl-free field (discrete gradient + 1e-9 noise) the
    error stays at the stencil's own rounding, ~eps |x|."""
    from paper_2508_07193_b200 import apply_double_curl
    ext = (24, 20, 16)
    nz, ny, nx = ext[2], ext[1], ext[0]
    rng = np.random.default_rng(14)
    xi = rng.integers(-1000, 1000, (3, nz, ny, nx)).astype(np.float64)
    assert np.array_equal(apply_double_curl(dev(xi, ext)).cpu().numpy(), O.double_curl(xi))
    phi = np.zeros((nz + 1, ny + 1, nx + 1))
    phi[:nz, :ny, :nx] = rng.uniform(-1, 1, (nz, ny, nx))
    grad = np.stack([phi[:nz, :ny, 1:] - phi[:nz, :ny, :nx], phi[:nz, 1:, :nx] - phi[:nz, :ny, :nx],
                     phi[1:, :ny, :nx] - phi[:nz, :ny, :nx]])
    x = grad + 1e-9 * rng.uniform(-1, 1, grad.shape)
    got = apply_double_curl(dev(x, ext)).cpu().numpy()
    assert np.abs(got - O.double_curl(x)).max() <= 64 * np.finfo(float).eps * np.abs(x).max()


def test_host_tensor_rejected_not_faulted():
    """A CPU tensor handed to a device entry point raises FlashMPError instead of passing a host
    pointer into a kernel."""
    from paper_2508_07193_b200 import apply_curl, FlashMPError
    from paper_2508_07193_b200.operators import stencil_apply
    x = torch.zeros(3, 4, 4, 4, dtype=torch.float64)
    with pytest.raises(FlashMPError):
        apply_curl("forward", x)
    with pytest.raises(FlashMPError):
        stencil_apply(x, 0.25)


def test_stencil_full_256_block_matches_oracle():
    """SURVEY §7 step-2 gate: the SpMV over a whole 256^3 GPU block against the oracle."""
    from paper_2508_07193_b200.operators import stencil_apply
    n = 256
    x = np.random.default_rng(15).uniform(-1, 1, (3, n, n, n))
    got = stencil_apply(dev(x, (n, n, n)), 0.25, True).cpu().numpy()
    want = O.apply_A(0.25, x, True)
    assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max()


@pytest.mark.parametrize("ext", [(64, 48, 40), (70, 33, 9), (8, 8, 8)])
def test_cn_rhs_zmarch_matches_point_kernel(ext, monkeypatch):
    """fmp_cn_rhs on the TMA z-march (SpMV mode 4: E through the plane ring, curl_b(H) per point)
    against the thread-per-point k_cn_rhs (FMP_CN_RHS_POINT=1), ref:cn_driver.py:54-59 (the
    reference-pinned CN tests in test_krylov_gpu.py run the z-march path).  The two kernels sum
    the C_b C_f bracket in different orders, so they agree to rounding, not bitwise."""
    from paper_2508_07193_b200 import _lib
    from paper_2508_07193_b200.plan import block_struct
    gen = torch.Generator(device="cuda").manual_seed(11)
    E = torch.rand(3, ext[2], ext[1], ext[0], dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    H = torch.rand(3, ext[2], ext[1], ext[0], dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    blk = block_struct(*ext)
    out = []
    for flag in ("0", "1"):
        monkeypatch.setenv("FMP_CN_RHS_POINT", flag)
        R = torch.full_like(E, float("nan"))
        _lib.call("fmp_cn_rhs", _lib.ref(blk), _lib.ref(blk), 0.7, _lib.ptr(E), _lib.ptr(H), _lib.ptr(R),
                  _lib.stream())
        torch.cuda.synchronize()
        out.append(R.cpu().numpy())
    assert np.isfinite(out[0]).all()
    assert np.max(np.abs(out[0] - out[1])) <= 1e-14 * np.max(np.abs(out[1]))


def test_bicg_xr0_is_bicg_xr_on_zero_x():
    """fmp_bicg_xr0 (x = 0 on entry, written without being read) gives bit for bit the x, r and
    next rho of fmp_bicg_xr on a zeroed x, signed zeros included (ref:krylov.py:154, 213-216)."""
    from paper_2508_07193_b200 import _lib
    n = 3 * 40 * 33 * 17
    gen = torch.Generator(device="cuda").manual_seed(5)
    ph, sh, s, t, rs = (torch.rand(n, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1 for _ in range(5))
    ph[::7] = -0.0
    sh[::7] = 0.0
    scratch = torch.zeros(int(_lib.lib().fmp_reduce_scratch_doubles()), dtype=torch.float64, device="cuda")
    outs = []
    for name in ("fmp_bicg_xr", "fmp_bicg_xr0"):
        x = torch.zeros(n, dtype=torch.float64, device="cuda") if name == "fmp_bicg_xr" else \
            torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
        r = torch.empty_like(x)
        dots = torch.zeros(2, dtype=torch.float64, device="cuda")
        _lib.call(name, n, _lib.ptr(x), _lib.ptr(ph), _lib.ptr(sh), _lib.ptr(s), _lib.ptr(t), _lib.ptr(r),
                  _lib.ptr(rs), 0.37, -1.3, _lib.ptr(dots), _lib.ptr(scratch), _lib.stream())
        torch.cuda.synchronize()
        outs.append((x.cpu().numpy(), r.cpu().numpy(), dots[0].item()))
    (x0, r0, d0), (x1, r1, d1) = outs
    assert np.array_equal(x0.view(np.int64), x1.view(np.int64))
    assert np.array_equal(r0, r1) and d0 == d1

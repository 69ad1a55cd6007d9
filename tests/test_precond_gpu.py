"""GPU parity: subdomain exact solve, Woodbury solve, GPU-built C^-1, RAS apply and the
restriction index maps, against the reference goldens and the oracle."""

import numpy as np
import pytest
import torch

import flashmp_oracle as O
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

SUB_EXTS = [(1, 1, 1), (2, 2, 2), (3, 3, 3), (4, 5, 6), (6, 2, 4), (1, 3, 4), (5, 1, 2)]


def rel(a, b):
    a, b = np.ravel(np.asarray(a)), np.ravel(np.asarray(b))
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("ext", SUB_EXTS)
@pytest.mark.parametrize("alpha", [0.05, 0.25, 1.0])
def test_subdomain_solves_match_reference(ext, alpha):
    from paper_2508_07193_b200 import Box, FieldVector, OperatorParams, exact_solve, precompute, solve
    g = np.load(GOLDEN / "subdomain.npz")
    tag = "_".join(map(str, ext)) + f"_a{alpha}"
    data = precompute(OperatorParams(Box(*ext), alpha))
    r = FieldVector(Box(*ext), g[f"r_{tag}"])
    assert rel(exact_solve(data, r).data, g[f"exact_{tag}"]) <= 1e-12
    assert rel(solve(data, r).data, g[f"solve_{tag}"]) <= 1e-11
    if f"rows_{tag}" in g:
        assert np.array_equal(data.corr.rows, g[f"rows_{tag}"])
        assert np.array_equal(data.corr.values, g[f"values_{tag}"])
        assert np.abs(data.corr.inverse.cpu().numpy() - g[f"Cinv_{tag}"]).max() <= 1e-12


def test_alpha_zero_is_identity():
    from paper_2508_07193_b200 import Box, FieldVector, OperatorParams, exact_solve, precompute, solve
    box = Box(3, 4, 5)
    data = precompute(OperatorParams(box, 0.0))
    v = FieldVector(box, np.random.default_rng(0).uniform(-1, 1, box.dof))
    assert data.corr is None
    assert np.array_equal(exact_solve(data, v).data, v.data)
    assert np.array_equal(solve(data, v).data, v.data)


@pytest.mark.parametrize("ext", [(17, 18, 17), (34, 34, 34), (33, 34, 33)])
def test_solve_round_trip_against_stencil(ext):
    """A (solve r) == r on the config-3/4 extended shapes (size-independent property)."""
    from paper_2508_07193_b200 import Box, FieldVector, OperatorParams, precompute, solve
    from paper_2508_07193_b200.operators import stencil_apply
    box = Box(*ext)
    data = precompute(OperatorParams(box, 0.25))
    r = np.random.default_rng(5).uniform(-1, 1, box.dof)
    e = solve(data, FieldVector(box, r)).data
    back = stencil_apply(torch.from_numpy(e).cuda().view(box.shape4), 0.25, True).cpu().numpy().ravel()
    assert rel(back, r) <= 1e-12
    # and against the oracle's exact solve (no correction) on the same input
    if ext == (17, 18, 17):
        od = O.precompute(ext, 0.25)
        assert rel(e, O.solve(od, r)) <= 1e-11


def test_precompute_cinv_matches_oracle_34():
    """GPU-assembled C^-1 on a 34^3-class shape vs the oracle (ref algorithm) -- 12x12x12 here
    to keep the oracle's CPU precompute short."""
    from paper_2508_07193_b200 import Box, OperatorParams, precompute
    ext = (12, 11, 13)
    data = precompute(OperatorParams(Box(*ext), 0.25))
    od = O.precompute(ext, 0.25)
    assert np.array_equal(data.corr.rows, od.rows)
    assert np.abs(data.corr.inverse.cpu().numpy() - od.Cinv).max() <= 1e-12


SCHWARZ = [((8, 8, 8), (2, 1, 1), 0), ((8, 8, 8), (2, 1, 1), 1), ((8, 8, 4), (2, 2, 1), 1),
           ((12, 8, 8), (3, 2, 2), 2), ((8, 4, 6), (2, 2, 3), 1)]


@pytest.mark.parametrize("gext,grid,ov", SCHWARZ)
def test_ras_and_index_maps_match_reference(gext, grid, ov):
    from paper_2508_07193_b200 import (Box, DistributedOperator, Exchanger, RasPreconditioner, gather_field,
                                       make_partition, make_transport, scatter_field)
    g = np.load(GOLDEN / "schwarz.npz")
    tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_o{ov}"
    part = make_partition(Box(*gext), grid, ov)
    tr = make_transport("serial", part.nranks)
    r = g[f"r_{tag}"]
    prec = RasPreconditioner(part, 0.25, tr)
    got = gather_field(part, prec.apply(scatter_field(part, r)))
    assert rel(got, g[f"ras_{tag}"]) <= 1e-11
    op = DistributedOperator(part, 0.25, tr)
    assert rel(gather_field(part, op.apply(scatter_field(part, r))), g[f"spmv_{tag}"]) <= 1e-14
    ex = Exchanger(part, tr)
    lin = np.arange(3 * int(np.prod(gext)), dtype=np.float64)
    exts = ex.exchange(scatter_field(part, lin))
    assert np.array_equal(np.concatenate(exts).astype(np.int64), g[f"extidx_{tag}"])


def test_ras_device_tensor_path_and_no_aliasing():
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport
    part = make_partition(Box(16, 16, 16), (2, 2, 2), 1)
    prec = RasPreconditioner(part, 0.25, make_transport("cuda"))
    r = torch.from_numpy(np.random.default_rng(6).uniform(-1, 1, part.global_box.dof)).cuda().view(3, 16, 16, 16)
    z1 = prec.apply(r)
    z2 = prec.apply(r)
    assert z1.data_ptr() != z2.data_ptr() and z1.data_ptr() != r.data_ptr()
    assert torch.equal(z1, z2)   # deterministic
    want = O.ras_apply((16, 16, 16), O.partition((16, 16, 16), (2, 2, 2), 1), 0.25, r.cpu().numpy().ravel())
    assert rel(z1.cpu().numpy(), want) <= 1e-11
    assert not prec.apply(torch.zeros_like(r)).any()


@pytest.mark.parametrize("gext,grid", [((32, 32, 32), (2, 2, 2)), ((48, 32, 32), (3, 2, 2)), ((16, 16, 16), (1, 1, 1)),
                                       ((64, 64, 64), (2, 2, 2))])
def test_fast_and_general_paths_agree(gext, grid, monkeypatch):
    """The warp-independent fast kernels (<= 2 distinct extents <= 36) and the general
    CTA-synchronous kernels compute the same preconditioner."""
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport
    part = make_partition(Box(*gext), grid, 1)
    tr = make_transport("cuda")
    r = torch.from_numpy(np.random.default_rng(7).uniform(-1, 1, part.global_box.dof)).cuda().view(
        part.global_box.shape4)
    monkeypatch.setenv("FMP_FORCE_GENERAL", "0")
    z_fast = RasPreconditioner(part, 0.25, tr).apply(r)
    monkeypatch.setenv("FMP_FORCE_GENERAL", "1")
    z_gen = RasPreconditioner(part, 0.25, tr).apply(r)
    assert rel(z_fast.cpu().numpy(), z_gen.cpu().numpy()) <= 1e-13
    if int(np.prod(gext)) <= 32 ** 3:
        want = O.ras_apply(gext, O.partition(gext, grid, 1), 0.25, r.cpu().numpy().ravel())
        assert rel(z_fast.cpu().numpy(), want) <= 1e-11


def test_large_and_general_paths_agree(monkeypatch):
    """64^3-class subdomains (extents 65/66, two z extents -> two column launches): the
    warp-independent large-extent kernels and the general CTA-synchronous kernels compute the
    same preconditioner (Woodbury, Ozaki GEMM with two K parts), and the exact single-subdomain
    solve of a 65 x 66 x 66 box on the large path matches the oracle's dense-transform solve."""
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport
    from paper_2508_07193_b200 import FieldVector, OperatorParams
    from paper_2508_07193_b200.subdomain import SubdomainSolverData, analytic_cost, correction_size, exact_solve
    from paper_2508_07193_b200.transform import TransformSet
    part = make_partition(Box(128, 128, 192), (2, 2, 3), 1)
    tr = make_transport("cuda")
    r = torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, part.global_box.dof)).cuda().view(
        part.global_box.shape4)
    monkeypatch.setenv("FMP_FORCE_GENERAL", "0")
    prec = RasPreconditioner(part, 0.25, tr)
    assert prec.plan.path() == "large"
    z_large = prec.apply(r)
    monkeypatch.setenv("FMP_FORCE_GENERAL", "1")
    gen = RasPreconditioner(part, 0.25, tr)
    assert gen.plan.path() == "general"
    z_gen = gen.apply(r)
    assert rel(z_large.cpu().numpy(), z_gen.cpu().numpy()) <= 1e-13
    monkeypatch.setenv("FMP_FORCE_GENERAL", "0")
    box = Box(65, 66, 66)
    data = SubdomainSolverData(OperatorParams(box, 0.25), TransformSet.for_box(box), None,
                               analytic_cost(box, correction_size(box)), torch.device("cuda"))
    x = np.random.default_rng(4).uniform(-1, 1, box.dof)
    got = exact_solve(data, FieldVector(box, x))
    want = O.exact_solve((65, 66, 66), O.point_block_inverses((65, 66, 66), 0.25), x)
    assert rel(np.asarray(got.data), want) <= 1e-12


def test_own_gemm_matches_cublas(monkeypatch):
    """The own DMMA Woodbury GEMM (FMP_GEMM=own) and cuBLAS DGEMM (FMP_GEMM=cublas) agree (the
    default Ozaki GEMM is checked against both in test_ozaki_gpu.py)."""
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport
    part = make_partition(Box(48, 32, 32), (3, 2, 2), 1)   # 3 shapes, n_s = 4 / 2 / ... columns
    tr = make_transport("cuda")
    r = torch.from_numpy(np.random.default_rng(8).uniform(-1, 1, part.global_box.dof)).cuda().view(
        part.global_box.shape4)
    monkeypatch.setenv("FMP_GEMM", "own")
    z_own = RasPreconditioner(part, 0.25, tr).apply(r)
    monkeypatch.setenv("FMP_GEMM", "cublas")
    z_blas = RasPreconditioner(part, 0.25, tr).apply(r)
    assert rel(z_own.cpu().numpy(), z_blas.cpu().numpy()) <= 1e-14


def test_stage_timing_api():
    """fmp_precond_profile / fmp_precond_stage_ms: eight non-negative stage times whose sum
    matches the whole apply measured with events on the same stream (within launch gaps)."""
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport
    part = make_partition(Box(64, 64, 64), (2, 2, 2), 1)
    prec = RasPreconditioner(part, 0.25, make_transport("cuda"))
    r = torch.rand(3, 64, 64, 64, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    prec.apply_into(r, z)
    want = z.clone()
    prec.plan.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    prec.apply_into(r, z)
    e1.record()
    st = prec.plan.stage_ms()
    prec.plan.profile(False)
    torch.cuda.synchronize()
    assert list(st) == list(prec.plan.STAGES)
    assert all(v >= 0.0 for v in st.values())
    assert sum(st.values()) <= e0.elapsed_time(e1) * 1.05 + 0.05
    assert torch.equal(z, want)   # timing does not change the result


@pytest.mark.parametrize("n", [49, 66])
def test_single_subdomain_preconditioner_is_the_exact_inverse(n):
    """With one subdomain covering the box, RAS is the exact solve: M^-1 (A x) == x.  Covers the
    large-extent paths: general (CTA) transform kernels, the 9-tile face kernels (extent > 40), the
    Ozaki GEMM at m = 14,259 (n = 49) and its K-split form past the int32 level bound (n = 66,
    m = 25,938: two K parts added in FP64)."""
    from paper_2508_07193_b200 import Box, DistributedOperator, RasPreconditioner, make_partition, make_transport
    part = make_partition(Box(n, n, n), (1, 1, 1), 1)
    tr = make_transport("cuda")
    op = DistributedOperator(part, 0.25, tr)
    prec = RasPreconditioner(part, 0.25, tr)
    x = torch.from_numpy(np.random.default_rng(11).uniform(-1, 1, 3 * n ** 3)).cuda().view(3, n, n, n)
    z = prec.apply(op.apply(x))
    assert rel(z.cpu().numpy(), x.cpu().numpy()) <= 1e-11


@pytest.mark.parametrize("gext,grid", [((64, 64, 64), (2, 2, 2)), ((48, 48, 48), (3, 3, 3))])
def test_column_tile_paths_bitwise(gext, grid, monkeypatch):
    """The column passes' TMA tiles (per-subdomain tensor maps, zero fill past ez), the cp.async
    tile loads (FMP_COL_NO_TMA) and the contiguous per-warp tile / plane orders (FMP_COL_CONTIG,
    FMP_PLANE_CONTIG) run the
    same arithmetic: bit-identical preconditioner outputs, including ragged last 8-column tiles."""
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport
    part = make_partition(Box(*gext), grid, 1)
    tr = make_transport("cuda")
    r = torch.from_numpy(np.random.default_rng(12).uniform(-1, 1, part.global_box.dof)).cuda().view(
        part.global_box.shape4)
    z0 = RasPreconditioner(part, 0.25, tr).apply(r)
    monkeypatch.setenv("FMP_COL_NO_TMA", "1")
    z1 = RasPreconditioner(part, 0.25, tr).apply(r)
    monkeypatch.delenv("FMP_COL_NO_TMA")
    monkeypatch.setenv("FMP_COL_CONTIG", "1")
    monkeypatch.setenv("FMP_PLANE_CONTIG", "1")
    z2 = RasPreconditioner(part, 0.25, tr).apply(r)
    assert torch.equal(z0, z1) and torch.equal(z0, z2)


def test_column_remainder_rows_match_dmma_tile(monkeypatch):
    """Forward column pass on 33/34-point columns: the DFMA remainder rows (default) and the
    fifth DMMA row tile (FMP_COL_NO_REM) agree to rounding."""
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport
    part = make_partition(Box(96, 64, 64), (3, 2, 2), 1)   # extents 33 and 34
    tr = make_transport("cuda")
    r = torch.from_numpy(np.random.default_rng(13).uniform(-1, 1, part.global_box.dof)).cuda().view(
        part.global_box.shape4)
    z0 = RasPreconditioner(part, 0.25, tr).apply(r)
    monkeypatch.setenv("FMP_COL_NO_REM", "1")
    z1 = RasPreconditioner(part, 0.25, tr).apply(r)
    assert rel(z0.cpu().numpy(), z1.cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("n,grid,overlap", [(64, (2, 2, 2), 1), (96, (3, 3, 3), 1), (48, (3, 3, 3), 1),
                                            (40, (2, 2, 2), 2), (64, (2, 2, 2), 2)])
def test_fused_lincomb_apply_is_bitwise_two_pass(n, grid, overlap):
    """fmp_precond_apply_lincomb (BiCGSTAB's s = r - alpha v formed inside the forward plane pass)
    gives exactly the s and z of fmp_vec_lincomb + fmp_precond_apply (ref:krylov.py:199-201):
    interior subdomains (TMA planes), block-boundary ones (cp.async planes), rotated shapes;
    16^3-class plans (and overlap 2 there) take the two-pass form and must give the same."""
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport, _lib
    part = make_partition(Box(n, n, n), grid, overlap)
    prec = RasPreconditioner(part, 0.25, make_transport("cuda"))
    gen = torch.Generator(device="cuda").manual_seed(7)
    r = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    v = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    alpha = 0.731
    s1, z1 = torch.full_like(r, float("nan")), torch.full_like(r, float("nan"))
    prec.apply_lincomb_into(r, v, -alpha, s1, z1)
    s2, z2 = torch.empty_like(r), torch.empty_like(r)
    _lib.call("fmp_vec_lincomb", r.numel(), 1.0, _lib.ptr(r), -alpha, _lib.ptr(v), _lib.ptr(s2), _lib.stream())
    prec.apply_into(s2, z2)
    torch.cuda.synchronize()
    assert torch.equal(s1, s2)
    assert torch.equal(z1, z2)
    assert prec.plan.path() == "fast"
    # the direction update p_new = r + beta (p - omega v) fused into M p_new (ref:krylov.py:179-187)
    p_old = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    beta, omega = 0.377, 1.19
    p1, z1 = torch.full_like(r, float("nan")), torch.full_like(r, float("nan"))
    prec.apply_bicg_p_into(r, p_old, v, beta, omega, p1, z1)
    p2 = p_old.clone()
    _lib.call("fmp_bicg_p", r.numel(), _lib.ptr(r), _lib.ptr(p2), _lib.ptr(v), beta, omega, _lib.stream())
    prec.apply_into(p2, z2)
    torch.cuda.synchronize()
    assert torch.equal(p1, p2)
    assert torch.equal(z1, z2)

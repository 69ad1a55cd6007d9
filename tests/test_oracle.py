"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz, made by
tests/golden/make_golden.py from /root/reference) and its known-answer values."""

import math

import numpy as np
import pytest

import flashmp_oracle as O
from conftest import GOLDEN


def load(name):
    return np.load(GOLDEN / name)


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


# ---------------------------------------------------------------- known answers
@pytest.mark.parametrize("n", [1, 2, 3, 7, 16, 32, 33, 34, 66])
def test_sigma_closed_form(n):
    assert np.abs(O.axis_svd(n).S - O.sigma_closed_form(n)).max() <= 2e-15


def test_svd_n1_gauge():
    s = O.axis_svd(1)      # ref:tests/test_transform.py:28-32
    assert s.U[0, 0] == -1.0 and s.S[0] == 1.0 and s.Vt[0, 0] == 1.0


def test_correction_sizes():
    assert O.correction_size((1, 1, 1)) == 3          # ref:tests/test_subdomain.py:56-61
    assert O.correction_size((32, 32, 32)) == 6 * 32 * 32 - 3 * 32 == 6048
    rows, vals = O.correction_rows((3, 4, 5))
    assert rows.size == O.correction_size((3, 4, 5))
    assert set(np.unique(vals)) <= {1.0, 2.0}


def test_flop_totals():
    f = O.analytic_flops((32, 32, 32), 6048)           # ref:tests/test_subdomain.py:162-182
    assert 144 * 32 ** 4 + 18 * 32 ** 3 == 151_584_768
    assert f["exact"] == 36 * 32 ** 4 + 18 * 32 ** 3
    assert f["correction"] == 2 * 6048 * 6048
    f34 = O.analytic_flops((34, 34, 34), O.correction_size((34, 34, 34)))
    assert f34["solve"] == 191_038_248


def test_proc_grid_for():
    assert [O.proc_grid_for(n) for n in (1, 2, 4, 8)] == [(1, 1, 1), (2, 1, 1), (2, 1, 2), (2, 2, 2)]


# ---------------------------------------------------------------- golden vectors
def test_svd_matches_reference():
    g = load("svd.npz")
    for n in (1, 2, 3, 4, 5, 8, 16, 17, 18, 32, 33, 34):
        s = O.axis_svd(n)
        assert np.abs(s.S - g[f"S_{n}"]).max() <= 1e-14
        assert np.abs(s.U - g[f"U_{n}"]).max() <= 1e-12
        assert np.abs(s.Vt - g[f"Vt_{n}"]).max() <= 1e-12


@pytest.mark.parametrize("ext", [(3, 3, 3), (4, 5, 6), (1, 3, 4), (8, 8, 8), (2, 7, 3)])
def test_operators_match_reference(ext):
    g = load("operators.npz")
    tag = "_".join(map(str, ext))
    nx, ny, nz = ext
    x = g[f"x_{tag}"].reshape(3, nz, ny, nx)
    assert rel(O.apply_A(0.25, x, True), g[f"A_{tag}"]) <= 1e-15
    assert rel(O.apply_A(0.25, x, True), g[f"Acsr_{tag}"]) <= 1e-14
    assert rel(O.apply_A(0.25, x, False), g[f"A0_{tag}"]) <= 1e-15
    assert rel(O.curl("forward", x), g[f"curlf_{tag}"]) <= 1e-15
    assert rel(O.curl("backward", x), g[f"curlb_{tag}"]) <= 1e-15
    assert rel(O.double_curl(x), g[f"M_{tag}"]) <= 1e-15
    assert rel(O.transform(x, ext, False), g[f"G_{tag}"]) <= 1e-13
    assert rel(O.transform(x, ext, True), g[f"Ginv_{tag}"]) <= 1e-13


@pytest.mark.parametrize("ext", [(1, 1, 1), (2, 2, 2), (3, 3, 3), (4, 5, 6), (6, 2, 4), (1, 3, 4), (5, 1, 2)])
@pytest.mark.parametrize("alpha", [0.05, 0.25, 1.0])
def test_subdomain_solves_match_reference(ext, alpha):
    g = load("subdomain.npz")
    tag = "_".join(map(str, ext)) + f"_a{alpha}"
    data = O.precompute(ext, alpha)
    r = g[f"r_{tag}"]
    assert rel(O.exact_solve(ext, data.binv, r), g[f"exact_{tag}"]) <= 1e-12
    assert rel(O.solve(data, r), g[f"solve_{tag}"]) <= 1e-12
    if f"rows_{tag}" in g:
        assert np.array_equal(data.rows, g[f"rows_{tag}"])
        assert np.array_equal(data.values, g[f"values_{tag}"])
        assert np.abs(data.Cinv - g[f"Cinv_{tag}"]).max() <= 1e-12


@pytest.mark.parametrize("ext", [(1, 1, 1), (2, 2, 2), (3, 3, 3), (4, 5, 6), (6, 2, 4), (1, 3, 4), (5, 1, 2),
                                 (9, 8, 7)])
@pytest.mark.parametrize("alpha", [0.05, 0.25])
def test_precompute_faces_equals_precompute(ext, alpha):
    """The closed-form C assembly (bench CPU baseline setup) equals the reference's m exact solves:
    same rows/values, C^-1 to rounding, and the reference golden C^-1 where one exists."""
    a, b = O.precompute(ext, alpha), O.precompute_faces(ext, alpha)
    assert np.array_equal(a.rows, b.rows) and np.array_equal(a.values, b.values)
    assert np.abs(a.Cinv - b.Cinv).max() <= 1e-14 * max(1.0, np.abs(a.Cinv).max())
    tag = "_".join(map(str, ext)) + f"_a{alpha}"
    g = load("subdomain.npz")
    if f"Cinv_{tag}" in g:
        assert np.abs(b.Cinv - g[f"Cinv_{tag}"]).max() <= 1e-12


SCHWARZ = [((8, 8, 8), (2, 1, 1), 0), ((8, 8, 8), (2, 1, 1), 1), ((8, 8, 4), (2, 2, 1), 1),
           ((12, 8, 8), (3, 2, 2), 2), ((8, 4, 6), (2, 2, 3), 1)]


@pytest.mark.parametrize("gext,grid,ov", SCHWARZ)
def test_schwarz_matches_reference(gext, grid, ov):
    g = load("schwarz.npz")
    tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_o{ov}"
    ranks = O.partition(gext, grid, ov)
    geom = np.array([[*r.owned_lo, *r.owned, *r.ext_lo, *r.ext] for r in ranks])
    assert np.array_equal(geom, g[f"geom_{tag}"])
    r = g[f"r_{tag}"]
    assert rel(O.ras_apply(gext, ranks, 0.25, r), g[f"ras_{tag}"]) <= 1e-12
    assert rel(O.op_apply(gext, 0.25, r), g[f"spmv_{tag}"]) <= 1e-14
    # index maps: restriction of a linear-index field == the reference exchanger output
    lin = np.arange(3 * np.prod(gext), dtype=np.float64).reshape(3, gext[2], gext[1], gext[0])
    got = np.concatenate([O.region(lin, rk.ext_lo, rk.ext).ravel() for rk in ranks]).astype(np.int64)
    assert np.array_equal(got, g[f"extidx_{tag}"])


KRYLOV = [((16, 16, 16), (2, 2, 2), 1, 0.25, "bicgstab", True),
          ((16, 16, 16), (2, 2, 2), 1, 0.25, "gmres", True),
          ((16, 16, 16), (2, 2, 2), 1, 0.25, "bicgstab", False),
          ((16, 16, 16), (2, 2, 2), 1, 0.25, "gmres", False),
          ((16, 16, 16), (2, 2, 2), 2, 0.25, "bicgstab", True),
          ((12, 12, 8), (3, 2, 1), 1, 1.0, "bicgstab", True),
          ((12, 12, 8), (3, 2, 1), 1, 1.0, "gmres", True),
          ((8, 8, 8), (1, 1, 1), 1, 0.25, "bicgstab", True)]


def krylov_tag(gext, grid, ov, alpha, method, prec_on):
    return "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_o{ov}_a{alpha}_{method}_" + (
        "ras" if prec_on else "none")


def oracle_solve(gext, grid, ov, alpha, method, prec_on, seed=42):
    ranks = O.partition(gext, grid, ov)
    x0 = np.random.default_rng(seed).uniform(-1.0, 1.0, 3 * int(np.prod(gext)))
    op = lambda u: O.op_apply(gext, alpha, u)
    prec = (lambda u: O.ras_apply(gext, ranks, alpha, u)) if prec_on else None
    b = op(x0)
    if method == "bicgstab":
        return O.bicgstab(op, prec, b)
    return O.gmres(op, prec, b)


@pytest.mark.parametrize("case", KRYLOV)
def test_krylov_matches_reference(case):
    g = load("krylov.npz")
    tag = krylov_tag(*case)
    x, rep = oracle_solve(*case)
    want = g[f"relres_{tag}"]
    assert rep.iterations == int(g[f"meta_{tag}"][0])
    assert rep.converged == bool(g[f"meta_{tag}"][1])
    assert len(rep.relres) == len(want)
    assert np.abs(np.array(rep.relres) - want).max() <= 1e-10
    assert rel(x, g[f"x_{tag}"]) <= 1e-10


@pytest.mark.parametrize("gext,grid", [((8, 8, 8), (1, 1, 1)), ((16, 16, 16), (2, 2, 2))])
def test_cn_step_matches_reference(gext, grid):
    g = load("cn.npz")
    tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + "_o1"
    rng = np.random.default_rng(42)
    n = 3 * int(np.prod(gext))
    shape = (3, gext[2], gext[1], gext[0])
    E = rng.uniform(-1.0, 1.0, n).reshape(shape)
    H = rng.uniform(-1.0, 1.0, n).reshape(shape)
    dt = 2.0 * math.sqrt(0.25)
    assert rel(O.build_rhs(E, H, dt), g[f"rhs_{tag}"]) <= 1e-15
    ranks = O.partition(gext, grid, 1)
    op = lambda u: O.op_apply(gext, 0.25, u)
    prec = lambda u: O.ras_apply(gext, ranks, 0.25, u)
    e1, h1, rep = O.cn_step(E, H, dt, lambda R: O.bicgstab(op, prec, R.ravel()))
    assert rep.iterations == int(g[f"iters_{tag}"][0])
    assert rel(e1, g[f"E1_{tag}"]) <= 1e-10
    assert rel(h1, g[f"H1_{tag}"]) <= 1e-10

"""GPU parity at the benchmarked sizes against the REFERENCE's own runs (tests/golden/huge.npz,
made by `make_golden.py --huge`, which imports /root/reference in the build container).

* 256^3, 8x8x8 subdomains of 32^3 (BASELINE configs 3/4, the bench workload): RAS apply,
  BiCGSTAB solve (ref:cli.py:98-136, krylov.py:146-239, schwarz.py:308-339) and one CN step
  (ref:cli.py:139-182, cn_driver.py:82-94);
* 96^3, 3x3x3 subdomains of 32^3: every extended shape of the 256^3 census, including the
  rotated (34,33,33)-type members whose Woodbury data the plan shares through row maps
  (plan.rotation_groups) -- also run with the sharing switched off;
* 64^3, 4x4x4 subdomains of 16^3 (the 16^3 point of BASELINE config 5), BiCGSTAB and GMRES.

The fixtures hold SAMPLE sampled entries (indices from default_rng(0)), the 2-norm and the sum
of every (component, z-plane) of each field, so every subdomain contributes to the checked sums.
Bars (north_star): equal iteration counts, |relres - ref| <= 1e-10, solution <= 1e-10 relative.
"""

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

HUGE = GOLDEN / "huge.npz"


@pytest.fixture(scope="module")
def g():
    if not HUGE.exists():
        pytest.skip("huge.npz not generated")
    return np.load(HUGE)


def check_field(g, tag, vec, tol):
    """Sampled entries, 2-norm and per-(component, z-plane) sums of a global field."""
    vec = np.asarray(vec).ravel()
    idx, want = g[f"idx_{tag}"], g[f"s_{tag}"]
    scale = np.linalg.norm(want)
    assert np.linalg.norm(vec[idx] - want) <= tol * scale, tag
    nrm = g[f"norm_{tag}"][0]
    assert abs(np.linalg.norm(vec) - nrm) <= tol * nrm, tag
    zs = g[f"zsum_{tag}"]
    got = vec.reshape(zs.shape[0], zs.shape[1], -1).sum(axis=2)
    # a plane sum adds ~n^2 terms of size ~|x|: compare against that magnitude, not the sum itself
    mag = np.abs(vec).reshape(zs.shape[0], zs.shape[1], -1).sum(axis=2)
    assert np.all(np.abs(got - zs) <= tol * mag + 1e-300), tag


def check_trace(g, tag, rep):
    want = g[f"relres_{tag}"]
    assert rep.iterations == int(g[f"meta_{tag}"][0]), (rep.iterations, g[f"meta_{tag}"])
    assert rep.converged == bool(g[f"meta_{tag}"][1])
    got = np.array([t[1] for t in rep.trace])
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= 1e-10
    big = want >= 1e-6
    assert np.all(np.abs(got[big] - want[big]) <= 1e-10 * want[big])


def _setup(gext, grid, method, share_rotations=True):
    from paper_2508_07193_b200 import (Box, DistributedOperator, RasPreconditioner, make_partition,
                                       make_transport)
    gbox = Box(*gext)
    part = make_partition(gbox, grid, 1)
    tr = make_transport("cuda")
    op = DistributedOperator(part, 0.25, tr)
    prec = RasPreconditioner(part, 0.25, tr, share_rotations=share_rotations)
    return gbox, part, op, prec


def _dev(a, gbox):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().view(gbox.shape4)


def _solve_case(g, gext, grid, method, share_rotations=True, ras=False):
    from paper_2508_07193_b200 import SolverConfig, bicgstab, gmres
    tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_{method}"
    gbox, part, op, prec = _setup(gext, grid, method, share_rotations)
    if ras:   # r = default_rng(3) U[-1, 1) over the global DOF (make_golden.rng_field)
        r = _dev(np.random.default_rng(3).uniform(-1.0, 1.0, gbox.dof), gbox)
        check_field(g, f"ras_{tag}", prec.apply(r).cpu().numpy(), 1e-11)
        del r
    x0 = _dev(np.random.default_rng(42).uniform(-1.0, 1.0, gbox.dof), gbox)   # ref:cli.py:98-102
    b = op.apply(x0)
    del x0
    runner = bicgstab if method == "bicgstab" else gmres
    x, rep = runner(op, prec, b, SolverConfig(method=method))
    check_trace(g, tag, rep)
    check_field(g, f"x_{tag}", x.cpu().numpy(), 1e-10)
    return gbox, part, op, prec


@pytest.mark.parametrize("share", [True, False])
def test_rotation_group_shapes_96(g, share):
    """All 8 extended shapes of the 256^3 census; with share=True the rotated members run through
    the row maps of k_faces / k_corr against their group's canonical C^-1."""
    _solve_case(g, (96, 96, 96), (3, 3, 3), "bicgstab", share_rotations=share, ras=True)


@pytest.mark.parametrize("method", ["bicgstab", "gmres"])
def test_16cube_subdomains_64(g, method):
    _solve_case(g, (64, 64, 64), (4, 4, 4), method)


def test_cfg4_256_ras_solve_and_cn_step(g):
    """The bench workload itself: 256^3 with 512 subdomains of 32^3 on one GPU."""
    from paper_2508_07193_b200 import SolverConfig
    from paper_2508_07193_b200.cn_driver import DeviceCnStepper
    gbox, part, op, prec = _solve_case(g, (256, 256, 256), (8, 8, 8), "bicgstab", ras=True)
    tag = "cn_256_256_256_g888_bicgstab"
    rng = np.random.default_rng(42)                       # ref:cli.py:143-149
    E = _dev(rng.uniform(-1.0, 1.0, gbox.dof), gbox)
    H = _dev(rng.uniform(-1.0, 1.0, gbox.dof), gbox)

    class _Solver:   # CnSolver's interface over the operator / preconditioner built above
        def __init__(self):
            self.op, self.prec, self.config, self.partition = op, prec, SolverConfig(), part

        def solve_device(self, rhs):
            from paper_2508_07193_b200 import bicgstab
            return bicgstab(self.op, self.prec, rhs, self.config)

    st = DeviceCnStepper(_Solver(), E, H, 1.0)   # dt = 2 sqrt(alpha) = 1 (ref:cli.py:145)
    rep = st.step()
    check_trace(g, tag, rep)
    check_field(g, f"E1_{tag}", st.E.cpu().numpy(), 1e-10)
    check_field(g, f"H1_{tag}", st.H.cpu().numpy(), 1e-10)

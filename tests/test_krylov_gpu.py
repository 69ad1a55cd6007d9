"""GPU parity of the drop-in solvers: iteration counts, residual histories (<= 1e-10) and
solutions (<= 1e-10 relative) against the reference's own runs (tests/golden)."""

import math

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

KRYLOV = [((16, 16, 16), (2, 2, 2), 1, 0.25, "bicgstab", True),
          ((16, 16, 16), (2, 2, 2), 1, 0.25, "gmres", True),
          ((16, 16, 16), (2, 2, 2), 1, 0.25, "bicgstab", False),
          ((16, 16, 16), (2, 2, 2), 1, 0.25, "gmres", False),
          ((16, 16, 16), (2, 2, 2), 2, 0.25, "bicgstab", True),
          ((12, 12, 8), (3, 2, 1), 1, 1.0, "bicgstab", True),
          ((12, 12, 8), (3, 2, 1), 1, 1.0, "gmres", True),
          ((8, 8, 8), (1, 1, 1), 1, 0.25, "bicgstab", True)]


def tag_of(gext, grid, ov, alpha, method, prec_on):
    return "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_o{ov}_a{alpha}_{method}_" + (
        "ras" if prec_on else "none")


def run(gext, grid, ov, alpha, method, prec_on, seed=42, list_form=True):
    from paper_2508_07193_b200 import (Box, DistributedOperator, RasPreconditioner, SolverConfig, bicgstab,
                                       gather_field, gmres, make_partition, make_transport, scatter_field)
    gbox = Box(*gext)
    part = make_partition(gbox, grid, ov)
    tr = make_transport("serial", part.nranks)
    op = DistributedOperator(part, alpha, tr)
    prec = RasPreconditioner(part, alpha, tr) if prec_on else None
    x0 = np.random.default_rng(seed).uniform(-1.0, 1.0, gbox.dof)
    b = op.apply(scatter_field(part, x0))
    cfg = SolverConfig(method=method, preconditioner="ras" if prec_on else "none")
    runner = bicgstab if method == "bicgstab" else gmres
    if list_form:
        x, rep = runner(op, prec, b, cfg)
        return gather_field(part, x), rep
    bt = torch.from_numpy(gather_field(part, b)).cuda().view(gbox.shape4)
    x, rep = runner(op, prec, bt, cfg)
    return x.cpu().numpy().ravel(), rep


def check(rep, x, g, tag, xkey=None):
    want = g[f"relres_{tag}"]
    assert rep.iterations == int(g[f"meta_{tag}"][0])
    assert rep.converged == bool(g[f"meta_{tag}"][1])
    got = np.array([t[1] for t in rep.trace])
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= 1e-10
    big = want >= 1e-6
    assert np.all(np.abs(got[big] - want[big]) <= 1e-10 * want[big])
    if f"x_{tag}" in g:
        xw = g[f"x_{tag}"]
        assert np.linalg.norm(x - xw) / np.linalg.norm(xw) <= 1e-10
    else:
        idx = g[f"xidx_{tag}"]
        assert np.linalg.norm(x[idx] - g[f"xs_{tag}"]) / np.linalg.norm(g[f"xs_{tag}"]) <= 1e-10
        assert abs(np.linalg.norm(x) - g[f"xnorm_{tag}"][0]) <= 1e-10 * g[f"xnorm_{tag}"][0]


@pytest.mark.parametrize("case", KRYLOV)
def test_solvers_match_reference(case):
    g = np.load(GOLDEN / "krylov.npz")
    x, rep = run(*case)
    check(rep, x, g, tag_of(*case))
    if case[4] == "bicgstab" and case[5]:
        for w in rep.work_per_iteration:
            assert w == {"precond": 2, "spmv": 2, "dot": 4, "axpy": 6}   # ref:tests/test_krylov.py:68-78
    if case[4] == "gmres":
        for pos, w in enumerate(rep.work_per_iteration[:rep.restart_cycles[0]]):
            assert w["dot"] == pos + 2 and w["axpy"] == pos + 1


@pytest.mark.parametrize("method", ["bicgstab", "gmres"])
def test_config2_matches_reference(method):
    """BASELINE config 2: 64^3, 2x2x2 subdomains of 32^3, overlap 1, alpha 0.25, seed 42."""
    g = np.load(GOLDEN / "krylov_big.npz")
    case = ((64, 64, 64), (2, 2, 2), 1, 0.25, method, True)
    x, rep = run(*case, list_form=False)
    check(rep, x, g, tag_of(*case))
    print(f"config2 {method}: iters={rep.iterations} margin relres/tol="
          f"{rep.final_relres / 1e-12:.3f} seconds={rep.seconds:.4f}")


def test_zero_rhs():
    from paper_2508_07193_b200 import (Box, DistributedOperator, RasPreconditioner, SolverConfig, bicgstab,
                                       gmres, make_partition, make_transport)
    part = make_partition(Box(8, 8, 8), (2, 2, 2), 1)
    tr = make_transport("cuda")
    op, prec = DistributedOperator(part, 0.25, tr), RasPreconditioner(part, 0.25, tr)
    b = torch.zeros(3, 8, 8, 8, dtype=torch.float64, device="cuda")
    for runner, m in ((bicgstab, "bicgstab"), (gmres, "gmres")):
        x, rep = runner(op, prec, b, SolverConfig(method=m))
        assert rep.converged and rep.final_relres == 0.0 and not x.any()


def test_cn_step_matches_reference():
    from paper_2508_07193_b200 import Box, CnSolver, EmState, FieldVector, SolverConfig, cn_step, make_transport
    g = np.load(GOLDEN / "cn.npz")
    for gext, grid, tag in [((8, 8, 8), (1, 1, 1), "8_8_8_g111_o1"), ((16, 16, 16), (2, 2, 2), "16_16_16_g222_o1")]:
        box = Box(*gext)
        rng = np.random.default_rng(42)
        E = FieldVector(box, rng.uniform(-1, 1, box.dof))
        H = FieldVector(box, rng.uniform(-1, 1, box.dof))
        solver = CnSolver(box, grid, 1, 0.25, SolverConfig(), make_transport("serial"))
        new, rep = cn_step(EmState(E, H, 0, 2.0 * math.sqrt(0.25)), solver)
        assert rep.iterations == int(g[f"iters_{tag}"][0])
        assert np.linalg.norm(new.E.data - g[f"E1_{tag}"]) / np.linalg.norm(g[f"E1_{tag}"]) <= 1e-10
        assert np.linalg.norm(new.H.data - g[f"H1_{tag}"]) / np.linalg.norm(g[f"H1_{tag}"]) <= 1e-10


def test_cn_step_config1_matches_reference():
    """BASELINE config 1: 32^3, one subdomain, one CN step, BiCGSTAB + FlashMP."""
    from paper_2508_07193_b200 import Box, CnSolver, EmState, FieldVector, SolverConfig, cn_step, make_transport
    g = np.load(GOLDEN / "cn_big.npz")
    tag = "32_32_32_g111_o1"
    box = Box(32, 32, 32)
    rng = np.random.default_rng(42)
    E = FieldVector(box, rng.uniform(-1, 1, box.dof))
    H = FieldVector(box, rng.uniform(-1, 1, box.dof))
    solver = CnSolver(box, (1, 1, 1), 1, 0.25, SolverConfig(), make_transport("serial"))
    new, rep = cn_step(EmState(E, H, 0, 1.0), solver)
    assert rep.iterations == int(g[f"iters_{tag}"][0])
    idx = g[f"idx_{tag}"]
    assert np.linalg.norm(new.E.data[idx] - g[f"E1_{tag}"]) / np.linalg.norm(g[f"E1_{tag}"]) <= 1e-10
    assert np.linalg.norm(new.H.data[idx] - g[f"H1_{tag}"]) / np.linalg.norm(g[f"H1_{tag}"]) <= 1e-10


def test_host_step_pipeline_matches_device_steps():
    """HostStepPipeline (host fields, overlapped transfers) == DeviceCnStepper on the same fields."""
    from paper_2508_07193_b200 import Box, CnSolver, DeviceCnStepper, HostStepPipeline, SolverConfig, make_transport
    n = 32
    solver = CnSolver(Box(n, n, n), (2, 2, 2), 1, 0.25, SolverConfig(), make_transport("cuda"))
    g = torch.Generator(device="cuda").manual_seed(3)
    E = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g)
    H = torch.rand(3, n, n, n, dtype=torch.float64, device="cuda", generator=g)
    st = DeviceCnStepper(solver, E.clone(), H.clone(), 1.0)
    st.step()
    Eh, Hh = E.cpu().pin_memory(), H.cpu().pin_memory()
    Eo, Ho = torch.empty_like(Eh).pin_memory(), torch.empty_like(Hh).pin_memory()
    reps = HostStepPipeline(solver, 1.0).run(Eh, Hh, Eo, Ho, steps=3)
    torch.cuda.synchronize()
    assert len(reps) == 3 and all(r.converged for r in reps)
    assert torch.equal(Eo, st.E.cpu()) and torch.equal(Ho, st.H.cpu())

"""Ozaki-scheme Woodbury GEMM on the INT8 tensor cores (FMP_GEMM=ozaki) against FP64 DGEMM:
the preconditioner agrees to ~1e-13 and the solvers keep the reference's iteration counts,
traces (<= 1e-10) and solutions (<= 1e-10)."""

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.ravel(np.asarray(a)), np.ravel(np.asarray(b))
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("gext,grid", [((64, 64, 64), (2, 2, 2)), ((48, 32, 32), (3, 2, 2)), ((8, 8, 8), (1, 1, 1))])
def test_ozaki_precond_matches_fp64(gext, grid, monkeypatch):
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport
    part = make_partition(Box(*gext), grid, 1)
    tr = make_transport("cuda")
    r = torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, part.global_box.dof)).cuda().view(
        part.global_box.shape4)
    monkeypatch.setenv("FMP_GEMM", "cublas")
    z64 = RasPreconditioner(part, 0.25, tr).apply(r)
    monkeypatch.setenv("FMP_GEMM", "ozaki")
    zoz = RasPreconditioner(part, 0.25, tr).apply(r)
    err = rel(zoz.cpu().numpy(), z64.cpu().numpy())
    print(f"ozaki vs fp64 RAS rel diff {err:.2e}")
    assert err <= 1e-12


def test_ozaki_solver_parity_config2(monkeypatch):
    import test_krylov_gpu as K
    monkeypatch.setenv("FMP_GEMM", "ozaki")
    g = np.load(GOLDEN / "krylov_big.npz")
    for method in ("bicgstab", "gmres"):
        case = ((64, 64, 64), (2, 2, 2), 1, 0.25, method, True)
        x, rep = K.run(*case, list_form=False)
        K.check(rep, x, g, K.tag_of(*case))


@pytest.mark.parametrize("case", [((16, 16, 16), (2, 2, 2), 1, 0.25, "bicgstab", True),
                                  ((12, 12, 8), (3, 2, 1), 1, 1.0, "gmres", True)])
def test_ozaki_solver_parity_small(case, monkeypatch):
    import test_krylov_gpu as K
    monkeypatch.setenv("FMP_GEMM", "ozaki")
    g = np.load(GOLDEN / "krylov.npz")
    x, rep = K.run(*case)
    K.check(rep, x, g, K.tag_of(*case))

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


@pytest.mark.parametrize("gext,grid", [((256, 256, 256), (8, 8, 8)), ((66, 66, 66), (1, 1, 1))])
def test_ozaki_elementwise_vs_dgemm(gext, grid):
    """Per-element accuracy of the Ozaki Z = C^-1 Y on the REAL Y of an apply: the cfg4 block
    (4 rotation groups, m = 6834 for the 34^3 group, 216 columns) and one 66^3 subdomain
    (m = 25,938: the K-split form, two int32 parts added in FP64), against cuBLAS DGEMM on the
    same operands.  Row/column power-of-two scaling keeps each entry to 2^-53 of its row's
    (column's) maximum, so the bound is per element:
        |dZ_ij| <= 2^-52 (max_k|C_ik| ||Y_j||_1 + max_k|Y_kj| ||C_i||_1) + m 2^-53 (|C||Y|)_ij
    (the last term is DGEMM's own rounding), and normwise ||dZ||_F <= 1e-14 ||Z||_F."""
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport
    part = make_partition(Box(*gext), grid, 1)
    prec = RasPreconditioner(part, 0.25, make_transport("cuda"))
    assert prec.plan.gemm_kind() == "ozaki"
    gbox = part.global_box
    r = torch.from_numpy(np.random.default_rng(16).uniform(-1, 1, gbox.dof)).cuda().view(gbox.shape4)
    prec.apply(r)
    torch.cuda.synchronize()
    plan = prec.plan
    worst = 0.0
    for q, (gi, _) in enumerate(plan.groups):
        if gi != q:
            continue
        m, ncol = plan.m[q], plan.gcols[q]
        Y, Z, Ci = plan.ymat[q][:ncol, :m], plan.zmat[q][:ncol, :m], plan.cinv[q][:, :m]
        Zref = Y @ Ci.T                                # cuBLAS DGEMM, FP64
        dZ = (Z - Zref).abs()
        Ca, Ya = Ci.abs(), Y.abs()
        bound = 2.0 ** -52 * (Ya.sum(1)[:, None] * Ca.amax(1)[None, :] + Ya.amax(1)[:, None] * Ca.sum(1)[None, :])
        bound += m * 2.0 ** -53 * (Ya @ Ca.T)
        ratio = float((dZ / bound).max())
        nrm = float(torch.linalg.norm(Z - Zref) / torch.linalg.norm(Zref))
        print(f"group {plan.shapes[q]} m={m} cols={ncol}: max |dZ|/bound {ratio:.3f}, normwise {nrm:.2e}")
        assert ratio <= 1.0
        assert nrm <= 1e-14
        worst = max(worst, ratio)
    assert worst > 0.0   # the comparison actually ran on nonzero differences or bounds


@pytest.mark.parametrize("gext,grid", [((96, 96, 96), (3, 3, 3)), ((64, 64, 64), (4, 4, 4))])
def test_zero_slice_skipping_is_exact(gext, grid, monkeypatch):
    """Skipping the all-zero C^-1 slice blocks (and whole all-zero K chunks) and the locality row
    order change no bit: with whole-tile items (FMP_OZ_NOSPLIT, so no schedule-dependent K
    segments) the sparse GEMM equals the dense one, and the dense one in the reference row order,
    bitwise.  96^3/3^3 holds every 32^3 shape of the cfg4 census (rotation groups);
    64^3/4^3 the 16^3 subdomains of config 5."""
    from paper_2508_07193_b200 import Box, RasPreconditioner, make_partition, make_transport
    part = make_partition(Box(*gext), grid, 1)
    tr = make_transport("cuda")
    r = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, part.global_box.dof)).cuda().view(
        part.global_box.shape4)
    monkeypatch.setenv("FMP_GEMM", "ozaki")
    monkeypatch.setenv("FMP_OZ_NOSPLIT", "1")
    monkeypatch.setenv("FMP_OZ_DENSE", "1")
    z_dense = RasPreconditioner(part, 0.25, tr).apply(r)
    monkeypatch.setenv("FMP_OZ_DENSE", "0")
    prec = RasPreconditioner(part, 0.25, tr)
    z_sparse = prec.apply(r)
    assert torch.equal(z_dense, z_sparse)
    assert prec.plan.ozaki_kept_slices() < 0.9   # the skipping is active at these sizes
    # the locality row order only permutes exact integer sums: reference order, dense, bit-identical
    monkeypatch.setenv("FMP_OZ_NOPERM", "1")
    monkeypatch.setenv("FMP_OZ_DENSE", "1")
    assert torch.equal(RasPreconditioner(part, 0.25, tr).apply(r), z_dense)

"""Exact subdomain solver on the GPU (mirror of ref:subdomain.py).

`precompute` builds, per extended box and alpha, the Woodbury data of the
boundary-corrected operator I + alpha (M + Lambda) (ref:subdomain.py:182-252):

  rows / values   the m boundary slots with nonzero delta, component-major ascending
  C = Q^T (I + alpha M)^-1 Q + diag(1/(alpha delta)),  C^-1 dense (m x m, FP64)

The reference assembles C with m exact solves on identity columns and a CPU
`np.linalg.inv` (38-55 s per 32^3-class box).  Here the m columns go through the
same batched GPU kernels as the preconditioner (mode FACES: forward transform,
block solve, and the inverse transform evaluated on the two boundary faces only),
and the inverse is a device Cholesky inverse (C is SPD; LU fallback), with the
reference's 1-norm condition guard.

`exact_solve` / `solve` run a one-subdomain plan; the RAS preconditioner
(schwarz.py) batches every subdomain of a GPU block into one plan.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .grid import Box, FieldVector
from .instrument import NULL_TIMER, FlopCounter
from .operators import OperatorParams
from .plan import SolvePlan, SubSpec, block_struct, correction_counts, lead_dim, pad_rows
from .transform import TransformSet

CONDITION_LIMIT = 1e14          # ref:subdomain.py:48
# device memory budget for one chunk of precompute columns (inputs + 2 workspaces)
PRECOMPUTE_CHUNK_BYTES = 3 << 30


class DegenerateConfigurationError(RuntimeError):
    """The boundary-correction matrix is numerically singular (ref:subdomain.py:52-56)."""


@dataclass(frozen=True)
class BoundaryCorrection:
    rows: np.ndarray            # (m,) component-major slot of each nonzero delta
    values: np.ndarray          # (m,) delta in {1, 2}
    m_per_component: tuple[int, int, int]
    weight_inv: np.ndarray      # 1 / (alpha delta)
    padded: torch.Tensor        # (m, ld) C^-1 on the device, rows zero-padded to ld (GEMM operand)

    @property
    def inverse(self) -> torch.Tensor:
        """(m, m) view of C^-1 (ref:subdomain.py:74 `inverse`)."""
        return self.padded[:, : self.m]

    @property
    def m(self) -> int:
        return int(self.rows.size)


@dataclass(frozen=True)
class CostModel:
    """Analytic flop/byte counts (ref:subdomain.py:82-104)."""

    box: Box
    m: int
    flops_per_exact_solve: int
    flops_per_correction: int
    bytes_resident: int

    @property
    def flops_per_solve(self) -> int:
        return 2 * self.flops_per_exact_solve + self.flops_per_correction

    @property
    def flops_total(self) -> int | None:
        b = self.box
        if not (b.nx == b.ny == b.nz):
            return None
        return 144 * b.nx ** 4 + 18 * b.nx ** 3

    @property
    def flops_executed(self) -> int:
        """Flops of the algorithm this build runs: two transforms (forward G, inverse
        G^-1) plus the block solve plus the C^-1 product; the face projections and the
        rank-structured correction are O(n^3) and counted too (csrc/precond.cu)."""
        nx, ny, nz = self.box.extents
        V = self.box.volume
        faces = 2 * 3 * 2 * V + 2 * 2 * (nx * ny * (nx + ny) + nz * nx * (nz + nx) + nz * ny * (nz + ny))
        return 12 * V * (nx + ny + nz) + 18 * V * 2 + 2 * self.m * self.m + 2 * faces


def analytic_cost(box: Box, m: int) -> CostModel:
    """ref:subdomain.py:221-232."""
    V = box.volume
    factors = sum(8 * (2 * n * n + n) for n in box.extents)
    return CostModel(box, m, 12 * V * sum(box.extents) + 18 * V, 2 * m * m,
                     8 * m * m + 48 * V + 72 * V + factors)


def correction_size(box: Box) -> int:
    return sum(correction_counts(box.extents))


def direct_method_flops(n: int) -> int:
    return 18 * n ** 6


def direct_method_inverse_bytes(n: int) -> int:
    return 72 * n ** 6


def direct_method_vector_bytes(n: int) -> int:
    return 48 * n ** 3


def correction_rows(box: Box) -> tuple[np.ndarray, np.ndarray, tuple[int, int, int]]:
    """Boundary slots and weights (ref:subdomain.py:183-194, ref:operators.py:151-164)."""
    nx, ny, nz = box.extents
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    i0, j0, k0 = (i == 0).astype(np.int64), (j == 0).astype(np.int64), (k == 0).astype(np.int64)
    weights = (j0 + k0, i0 + k0, i0 + j0)
    rows, vals, per = [], [], []
    for c, w in enumerate(weights):
        flat = w.ravel()
        idx = np.flatnonzero(flat)
        rows.append(idx + c * box.volume)
        vals.append(flat[idx].astype(np.float64))
        per.append(int(idx.size))
    return np.concatenate(rows).astype(np.int64), np.concatenate(vals), tuple(per)


@dataclass(frozen=True)
class SubdomainSolverData:
    """Everything precomputed for solves on one box/alpha (ref:subdomain.py:122-134)."""

    params: OperatorParams
    ts: TransformSet
    corr: BoundaryCorrection | None
    cost: CostModel
    device: torch.device = field(default=None)

    @property
    def box(self) -> Box:
        return self.params.box


def _assemble_correction(box: Box, alpha: float, device) -> BoundaryCorrection:
    rows, values, per = correction_rows(box)
    m, dof = rows.size, box.dof
    chunk = int(max(1, min(m, PRECOMPUTE_CHUNK_BYTES // (3 * 8 * dof))))
    subs = [SubSpec(box.extents, (0, 0, 0), (0, 0, 0), box.extents, in_off=q * dof) for q in range(chunk)]
    plan = SolvePlan(subs, alpha, device, need_woodbury=False)
    blk = block_struct(*box.extents)
    X = torch.zeros((chunk, dof), dtype=torch.float64, device=device)
    CT = torch.empty((m, m), dtype=torch.float64, device=device)   # CT[col] = column col of C
    rows_dev = torch.from_numpy(rows).to(device)
    ar = torch.arange(chunk, device=device)
    for lo in range(0, m, chunk):
        hi = min(lo + chunk, m)
        X.zero_()
        X[ar[: hi - lo], rows_dev[lo:hi]] = 1.0
        plan.apply(blk, _lib.FMP_SOLVE_FACES, X, None)
        CT[lo:hi] = plan.ymat[0][: hi - lo, :m]
    weight_inv = 1.0 / (alpha * values)
    Cm = CT.t().contiguous()
    Cm.diagonal().add_(torch.from_numpy(weight_inv).to(device))
    # C = Q^T (I + alpha M)^-1 Q + diag(1 / (alpha delta)) is symmetric positive definite (the
    # double-curl operator is SPD), so the inverse goes through a Cholesky factorisation of its
    # lower triangle (an exactly symmetric C^-1, as SURVEY 8f #1 plans); LU only if the
    # factorisation reports a non-positive pivot.
    L, info = torch.linalg.cholesky_ex(Cm)
    if int(info) == 0:
        inv = torch.cholesky_inverse(L)
    else:
        try:
            inv = torch.linalg.inv(Cm)
        except RuntimeError as exc:   # torch raises on exactly singular input
            raise DegenerateConfigurationError(
                f"correction matrix singular for box {box.extents}, alpha={alpha}") from exc
    del L
    cond1 = float(Cm.abs().sum(0).max() * inv.abs().sum(0).max())
    if not np.isfinite(cond1) or cond1 > CONDITION_LIMIT:
        raise DegenerateConfigurationError(
            f"correction matrix condition ~{cond1:.2e} exceeds {CONDITION_LIMIT:.0e} "
            f"for box {box.extents}, alpha={alpha}")
    return BoundaryCorrection(rows, values, per, weight_inv, pad_rows(inv, lead_dim(m)))


def precompute(params: OperatorParams, device=None) -> SubdomainSolverData:
    """Factors + Woodbury data for one box (ref:subdomain.py:241-252); GPU-built C^-1."""
    dev = _lib.require_cuda(device)
    box = params.box
    ts = TransformSet.for_box(box)
    corr = None if params.alpha == 0.0 else _assemble_correction(box, params.alpha, dev)
    m = corr.m if corr is not None else correction_size(box)
    return SubdomainSolverData(params, ts, corr, analytic_cost(box, m), dev)


def _single_plan(data: SubdomainSolverData, woodbury: bool) -> SolvePlan:
    e = data.box.extents
    cinv = {e: data.corr.padded} if (woodbury and data.corr is not None) else None
    return SolvePlan([SubSpec(e, (0, 0, 0), (0, 0, 0), e)], data.params.alpha, data.device, cinv=cinv,
                     need_woodbury=woodbury)


def _run_single(data: SubdomainSolverData, X, mode: int, counter: FlopCounter | None):
    if X.box != data.box:
        raise ValueError(f"field box {X.box.extents} != solver box {data.box.extents}")
    if data.params.alpha == 0.0:
        return X.copy()
    plan = _single_plan(data, mode == _lib.FMP_SOLVE_WOODBURY)
    src = torch.from_numpy(np.ascontiguousarray(X.data)).to(data.device)
    out = torch.empty_like(src)
    plan.apply(block_struct(*data.box.extents), mode, src, out)
    if counter is not None:
        V, nsum = data.box.volume, sum(data.box.extents)
        passes = 1 if mode == _lib.FMP_SOLVE_EXACT else 2
        counter.gemm += passes * 12 * V * nsum
        counter.bspmv += passes * 18 * V
        if mode == _lib.FMP_SOLVE_WOODBURY:
            counter.gemv += 2 * data.corr.m ** 2
    return FieldVector(X.box, out.cpu().numpy())


def exact_solve(data: SubdomainSolverData, X: FieldVector, counter: FlopCounter | None = None,
                timer=NULL_TIMER) -> FieldVector:
    """(I + alpha M)^-1 X, no boundary term (ref:subdomain.py:255-262)."""
    with timer.phase("fast_solve"):
        return _run_single(data, X, _lib.FMP_SOLVE_EXACT, counter)


def solve(data: SubdomainSolverData, R: FieldVector, counter: FlopCounter | None = None,
          timer=NULL_TIMER) -> FieldVector:
    """(I + alpha (M + Lambda))^-1 R via Woodbury (ref:subdomain.py:265-287)."""
    with timer.phase("fast_solve"):
        return _run_single(data, R, _lib.FMP_SOLVE_WOODBURY, counter)


def cost_report(data: SubdomainSolverData) -> CostModel:
    return data.cost

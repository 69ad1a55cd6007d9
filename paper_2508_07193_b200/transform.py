"""Per-axis SVD factors of the 1-D forward difference (mirror of ref:transform.py:36-76).

The factorisation is setup, not hot path: it is computed once per axis extent on
the host with LAPACK (numpy.linalg.svd, the same call the reference makes) and
the same sign gauge, so the factors are bit-identical to the reference's, then
uploaded once.  The transforms themselves run on the GPU (csrc/precond.cu).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .grid import Box


@dataclass(frozen=True)
class AxisSvd:
    """D = U diag(S) Vt for the n x n forward difference."""

    n: int
    U: np.ndarray
    S: np.ndarray
    Vt: np.ndarray


def forward_difference(n: int) -> np.ndarray:
    """-1 on the diagonal, +1 on the superdiagonal (ref:operators.py:58-65)."""
    if n < 1:
        raise ValueError("difference matrix size must be >= 1")
    return np.eye(n, k=1) - np.eye(n)


@lru_cache(maxsize=None)
def svd_of_difference(n: int) -> AxisSvd:
    """SVD with the reference gauge: the first entry above 1e-14 in magnitude of each
    row of Vt is positive, the matching column of U flips with it (ref:transform.py:46-63)."""
    U, S, Vt = np.linalg.svd(forward_difference(n))
    lead = np.argmax(np.abs(Vt) > 1e-14, axis=1)
    sign = np.where(Vt[np.arange(n), lead] < 0, -1.0, 1.0)
    Vt *= sign[:, None]
    U *= sign[None, :]
    for a in (U, S, Vt):
        a.setflags(write=False)
    return AxisSvd(n, U, S, Vt)


@dataclass(frozen=True)
class TransformSet:
    svd_x: AxisSvd
    svd_y: AxisSvd
    svd_z: AxisSvd

    @classmethod
    def for_box(cls, box: Box) -> "TransformSet":
        return cls(*(svd_of_difference(n) for n in box.extents))

    def axes(self):
        return (self.svd_x, self.svd_y, self.svd_z)

"""Matrix-free curls and the corrected operator on the GPU (mirror of ref:operators.py).

    A = I + alpha (C_b C_f + Lambda)          (ref:operators.py:167-175)

is evaluated by the stencil kernel of csrc/stencil.cu as the zero-ghost double
curl; with_boundary=False drops Lambda.  Inputs may be
host FieldVectors (copied to the device and back, for API parity) or device
tensors of shape (3, nz, ny, nx).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .grid import Box, FieldVector
from .plan import block_struct


@dataclass(frozen=True)
class OperatorParams:
    """alpha = dt^2 / 4 and the box it acts on (ref:operators.py:37-46)."""

    box: Box
    alpha: float = 0.25

    def __post_init__(self):
        if self.alpha < 0:
            raise ValueError(f"alpha must be >= 0, got {self.alpha}")


def _to_device(E, box: Box) -> torch.Tensor:
    if isinstance(E, FieldVector):
        if E.box != box:
            raise ValueError(f"field box {E.box.extents} != operator box {box.extents}")
        return torch.from_numpy(np.ascontiguousarray(E.data)).to(_lib.require_cuda()).view(box.shape4)
    if isinstance(E, torch.Tensor):
        if tuple(E.shape) != box.shape4 and E.numel() != box.dof:
            raise ValueError(f"tensor of {tuple(E.shape)} does not match box {box.extents}")
        _lib.require_cuda()
        if not E.is_cuda or E.dtype != torch.float64:
            raise _lib.FlashMPError("device fields must be float64 CUDA tensors (host data: pass a FieldVector)")
        return E.reshape(box.shape4).contiguous()
    raise TypeError(f"unsupported field type {type(E)!r}")


def _like_input(E, box: Box, out: torch.Tensor):
    return FieldVector(box, out.cpu().numpy().ravel()) if isinstance(E, FieldVector) else out


FMP_STENCIL_LAMBDA, FMP_STENCIL_NO_IDENTITY = 1, 2   # fmp_stencil_apply boundary flags


def stencil_apply(x: torch.Tensor, alpha: float, with_boundary: bool = True, blk=None,
                  identity: bool = True) -> torch.Tensor:
    """y = A x on a device block (single-GPU block covers the global box); identity=False
    gives y = alpha (C_b C_f [+ Lambda]) x."""
    if blk is None:
        blk = block_struct(x.shape[3], x.shape[2], x.shape[1])
    y = torch.empty_like(x)
    flags = (FMP_STENCIL_LAMBDA if with_boundary else 0) | (0 if identity else FMP_STENCIL_NO_IDENTITY)
    _lib.call("fmp_stencil_apply", _lib.ref(blk), float(alpha), flags, 0,
              _lib.ptr(x), _lib.ptr(y), None, None, None, _lib.stream())
    return y


def apply_operator(params: OperatorParams, with_boundary: bool, E):
    """A E = E + alpha (M E [+ Lambda E])."""
    x = _to_device(E, params.box)
    return _like_input(E, params.box, stencil_apply(x, params.alpha, with_boundary))


def apply_curl(kind: str, E):
    """Curl with all-forward or all-backward differences (ref:operators.py:119-125)."""
    if kind not in ("forward", "backward"):
        raise ValueError(f"kind must be 'forward' or 'backward', got {kind!r}")
    box = E.box if isinstance(E, FieldVector) else Box(E.shape[-1], E.shape[-2], E.shape[-3])
    x = _to_device(E, box)
    out = torch.empty_like(x)
    blk = block_struct(*box.extents)
    _lib.call("fmp_curl", _lib.ref(blk), 0 if kind == "forward" else 1, _lib.ptr(x), _lib.ptr(out),
              _lib.stream())
    return _like_input(E, box, out)


def apply_double_curl(E):
    """C_b C_f E (ref:operators.py:128-131): the stencil without the identity and Lambda, alpha = 1,
    so M E is formed directly (no cancellation against E)."""
    box = E.box if isinstance(E, FieldVector) else Box(E.shape[-1], E.shape[-2], E.shape[-3])
    x = _to_device(E, box)
    out = stencil_apply(x, 1.0, with_boundary=False, identity=False)
    return _like_input(E, box, out)

"""ctypes binding of libflashmp_b200.so (the C ABI in include/flashmp_b200.h).

There is no fallback: if the library is missing or cannot be loaded, every entry
point raises.  Build it with ``python -m paper_2508_07193_b200.build`` (or
``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "libflashmp_b200.so"
ABI_VERSION = 1

# Every symbol declared in include/flashmp_b200.h, with its ctypes signature.
_p, _i64, _d, _i = C.c_void_p, C.c_int64, C.c_double, C.c_int
SIGNATURES = {
    "fmp_abi_version": (_i, []),
    "fmp_last_error": (_i, [C.c_char_p, C.c_size_t]),
    "fmp_reduce_scratch_doubles": (_i64, []),
    "fmp_launch_count": (_i64, []),
    "fmp_stencil_apply": (_i, [_p, _d, _i, _i, _p, _p, _p, _p, _p, _p]),
    "fmp_curl": (_i, [_p, _i, _p, _p, _p]),
    "fmp_cn_rhs": (_i, [_p, _p, _d, _p, _p, _p, _p]),
    "fmp_cn_h_update": (_i, [_p, _p, _d, _p, _p, _p, _p, _p]),
    "fmp_vec_lincomb": (_i, [_i64, _d, _p, _d, _p, _p, _p]),
    "fmp_vec_axpy": (_i, [_i64, _d, _p, _p, _p]),
    "fmp_vec_scale": (_i, [_i64, _d, _p, _p, _p]),
    "fmp_vec_dot": (_i, [_i64, _p, _p, _p, _p, _p]),
    "fmp_vec_axpy_dot": (_i, [_i64, _d, _p, _p, _p, _p, _p, _p]),
    "fmp_vec_combine": (_i, [_i64, _p, _i, _p, _p, _p, _p]),
    "fmp_bicg_p": (_i, [_i64, _p, _p, _p, _d, _d, _p]),
    "fmp_bicg_xr": (_i, [_i64, _p, _p, _p, _p, _p, _p, _p, _d, _d, _p, _p, _p]),
    "fmp_bicg_xr0": (_i, [_i64, _p, _p, _p, _p, _p, _p, _p, _d, _d, _p, _p, _p]),
    "fmp_precond_create": (_i, [_p, C.POINTER(_p)]),
    "fmp_precond_destroy": (_i, [_p]),
    "fmp_precond_apply": (_i, [_p, _p, _i, _p, _p, _p]),
    "fmp_precond_restrict": (_i, [_p, _p, _p, _p, _p]),
    "fmp_precond_profile": (_i, [_p, _i]),
    "fmp_precond_stage_ms": (_i, [_p, C.POINTER(C.c_float), _i]),
    "fmp_precond_path": (_i, [_p]),
    "fmp_precond_ozaki_stats": (_i, [_p, _p, _i]),
    "fmp_debug_ozaki_prof": (_i, [_p, _i]),
    "fmp_stencil_apply_part": (_i, [_p, _d, _i, _i, _i, _p, _p, _p, _p, _p, _p]),
    "fmp_precond_apply_part": (_i, [_p, _p, _i, _i, _p, _p, _p]),
    "fmp_precond_apply_lincomb": (_i, [_p, _p, _i, _p, _p, _d, _p, _p, _p]),
    "fmp_precond_apply_bicg_p": (_i, [_p, _p, _i, _p, _p, _p, _d, _d, _p, _p, _p]),
    "fmp_halo_slab_doubles": (_i64, [_p, _i]),
    "fmp_halo_pack": (_i, [_p, _i, _i, _p, _p, _d, _p]),
    "fmp_halo_unpack": (_i, [_p, _i, _i, _p, _d, _p, _p]),
}

FMP_PART_ALL, FMP_PART_INTERIOR, FMP_PART_BOUNDARY = 0, 1, 2
FMP_HALO_Z, FMP_HALO_Y, FMP_HALO_X = 0, 1, 2

FMP_SOLVE_WOODBURY, FMP_SOLVE_EXACT, FMP_SOLVE_FACES = 0, 1, 2


class FmpBlock(C.Structure):
    """fmp_block: one GPU's block of the global grid plus its ghost shell."""

    _fields_ = [("bx", C.c_int64), ("by", C.c_int64), ("bz", C.c_int64),
                ("gx0", C.c_int64), ("gy0", C.c_int64), ("gz0", C.c_int64),
                ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("halo", C.c_int64), ("ghost", C.c_void_p * 6)]


class FmpPrecondDesc(C.Structure):
    _fields_ = [("alpha", C.c_double), ("n_sub", C.c_int64), ("n_shape", C.c_int64),
                ("subs", C.c_void_p), ("shapes", C.c_void_p),
                ("subs_host", C.c_void_p), ("shapes_host", C.c_void_p),
                ("shape_first", C.c_void_p), ("factors", C.c_void_p), ("cinv", C.c_void_p),
                ("work_a", C.c_void_p), ("work_b", C.c_void_p), ("corr", C.c_void_p),
                ("ymat", C.c_void_p), ("zmat", C.c_void_p), ("pmax", C.c_int64), ("rowmap", C.c_void_p)]


class FlashMPError(RuntimeError):
    """Raised when a libflashmp_b200 call reports an error."""


_LIB = None


def lib():
    """Load the library once; raise loudly when it is absent (no CPU fallback)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise FlashMPError(f"{LIB_PATH} not built: run `python -m paper_2508_07193_b200.build`")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype, fn.argtypes = res, args
        if handle.fmp_abi_version() != ABI_VERSION:
            raise FlashMPError("libflashmp_b200.so ABI version mismatch")
        _LIB = handle
    return _LIB


def last_error() -> str:
    buf = C.create_string_buffer(512)
    lib().fmp_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise FlashMPError(f"{what} failed ({rc}): {last_error()}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise FlashMPError("libflashmp_b200 needs CUDA tensors (no CPU fallback)")
    return t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def require_cuda(device=None) -> torch.device:
    """The hot path runs only on a CUDA device with the native library loaded."""
    if not torch.cuda.is_available():
        raise FlashMPError("paper_2508_07193_b200 needs a CUDA device (B200); no CPU fallback")
    lib()
    return torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)


class HostScalars:
    """A few FP64 reduction results that kernels write straight into pinned, device-mapped
    (UVA) host memory.  Reading them costs one stream synchronisation and no copy, so the
    Krylov scalars never queue behind bulk transfers on a copy engine."""

    def __init__(self, n: int):
        self.t = torch.zeros(n, dtype=torch.float64, pin_memory=True)

    def ptr(self) -> int:
        return self.t.data_ptr()

    def read(self, n: int | None = None) -> list[float]:
        torch.cuda.current_stream().synchronize()
        return self.t[: n if n is not None else self.t.numel()].tolist()


def ref(struct):
    """ctypes.byref for the C structs passed by pointer."""
    return C.byref(struct)

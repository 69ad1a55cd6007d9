"""Host-side builder of a batched subdomain-solve plan (fmp_precond in the C ABI).

A plan covers a list of subdomains that share one input field (a GPU block, or
compact per-column inputs during precompute).  Subdomains are grouped by
extended shape; every shape carries its SVD factors, its correction rows and
(for Woodbury solves) its dense C^-1.  All buffers are torch CUDA tensors owned
by the plan; the C library only sees their addresses.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .transform import svd_of_difference


@dataclass(frozen=True)
class SubSpec:
    """One subdomain: extended box + owned tile, in block-local coordinates."""

    ext: tuple[int, int, int]
    ext_lo: tuple[int, int, int]
    own_off: tuple[int, int, int]
    own: tuple[int, int, int]
    in_off: int = 0


def lead_dim(m: int) -> int:
    """Row stride of C^-1 / Y / Z: m rounded up to 4 doubles (32-byte rows for the GEMM)."""
    return (m + 3) // 4 * 4


def pad_rows(t: torch.Tensor, ld: int) -> torch.Tensor:
    """(m, m) -> (m, ld) with zero padding columns (shared when already padded)."""
    m = t.shape[0]
    if ld == m and t.is_contiguous():
        return t
    out = torch.zeros((m, ld), dtype=t.dtype, device=t.device)
    out[:, :m] = t
    return out


def rotate(ext):
    """Cyclic axis rotation (x, y, z) -> (y, z, x) of a box: new x' = old y, y' = z, z' = x."""
    return (ext[1], ext[2], ext[0])


def rotation_groups(shapes) -> list[tuple[int, int]]:
    """(index of the group's canonical shape, t) for every shape, with shape = rotate^t(canonical).

    The double-curl operator is invariant under cyclic relabelling of the axes (component
    x -> z', y -> x', z -> y', point (i, j, k) -> (j, k, i)), and so are the boundary deltas,
    so the Woodbury matrices of rotated boxes are equal up to a permutation of their rows and
    columns (checked in tests/test_host.py).  One C^-1 and one GEMM then serve a whole group."""
    out = []
    for q, e in enumerate(shapes):
        hit = None
        for g, (rep, t) in enumerate(out):
            if rep != g:
                continue
            r = shapes[g]
            for tt in (1, 2):
                r = rotate(r)
                if r == e and r != shapes[g]:
                    hit = (g, tt)
                    break
            if hit:
                break
        out.append(hit if hit else (q, 0))
    return out


def correction_points(ext) -> np.ndarray:
    """(m, 4) int array of (c, i, j, k) per correction row, in row order
    (component-major, ascending linear index: ref:subdomain.py:183-194)."""
    nx, ny, nz = ext
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    i0, j0, k0 = i == 0, j == 0, k == 0
    pts = []
    for c, w in enumerate(((j0 | k0), (i0 | k0), (i0 | j0))):
        idx = np.flatnonzero(w.ravel())
        pts.append(np.stack([np.full(idx.size, c), i.ravel()[idx], j.ravel()[idx], k.ravel()[idx]], axis=1))
    return np.concatenate(pts).astype(np.int64)


def rotation_rowmap(rep, t: int) -> np.ndarray:
    """int32 map from the correction rows of rotate^t(rep) to the rows of rep."""
    pts = correction_points(rep)
    e = tuple(rep)
    for _ in range(t):
        c, i, j, k = pts.T
        pts = np.stack([(c + 2) % 3, j, k, i], axis=1)
        e = rotate(e)
    nx, ny, nz = e
    V = nx * ny * nz
    key_rep = pts[:, 0] * V + pts[:, 3] * nx * ny + pts[:, 2] * nx + pts[:, 1]   # rows of rep, in e's indices
    own = correction_points(e)
    key_own = own[:, 0] * V + own[:, 3] * nx * ny + own[:, 2] * nx + own[:, 1]
    pos = np.full(3 * V, -1, dtype=np.int64)
    pos[key_own] = np.arange(key_own.size)
    rowmap = np.empty(key_own.size, dtype=np.int32)
    rowmap[pos[key_rep]] = np.arange(key_rep.size, dtype=np.int32)
    return rowmap


def correction_counts(ext) -> tuple[int, int, int]:
    """Rows per component (ref:subdomain.py:235-238)."""
    nx, ny, nz = ext
    return (nx * (ny + nz - 1), ny * (nx + nz - 1), nz * (nx + ny - 1))


class FactorTable:
    """One device buffer with, per distinct axis extent, U^T, V^T (row-major) and S, and per
    extended shape the block-inverse table: (q, w) per transformed point (c', b, a) with
    q = 1/(1 + alpha |s|^2), w = (1 - q)/|s|^2, so B^-1 y = q y + w s (s . y)
    (the closed form of ref:subdomain.py:137-153)."""

    def __init__(self, shapes, alpha: float, device):
        blocks, self.offsets, self.qw, off = [], {}, {}, 0

        def push(arr):
            nonlocal off
            start = off
            blocks.append(np.ascontiguousarray(arr, dtype=np.float64).ravel())
            off += blocks[-1].size
            pad = (-off) % 8
            if pad:
                blocks.append(np.zeros(pad))
                off += pad
            return start

        for n in sorted({n for e in shapes for n in e}):
            sv = svd_of_difference(n)
            self.offsets[n] = (push(sv.U.T), push(sv.Vt), push(sv.S))
        for e in shapes:
            nx, ny, nz = e
            S = [svd_of_difference(n).S for n in e]
            s2 = S[2][:, None, None] ** 2 + S[1][None, :, None] ** 2 + S[0][None, None, :] ** 2
            q = 1.0 / (1.0 + alpha * s2)
            w = (1.0 - q) / s2
            self.qw[e] = push(np.stack([q, w], axis=-1))
        self.host = np.concatenate(blocks) if blocks else np.zeros(8)
        self.device = torch.from_numpy(self.host).to(device)


class SolvePlan:
    """Batched FlashMP subdomain solves over `subs` (see csrc/precond.cu)."""

    def __init__(self, subs: list[SubSpec], alpha: float, device, cinv: dict | None = None,
                 need_woodbury: bool = True, share_rotations: bool = True):
        _lib.lib()
        self._gemm = os.environ.get("FMP_GEMM", "ozaki")   # read by fmp_precond_create below
        self.device = torch.device(device)
        self.alpha = float(alpha)
        shapes: list[tuple[int, int, int]] = []
        for s in subs:
            if s.ext not in shapes:
                shapes.append(s.ext)
        order = sorted(range(len(subs)), key=lambda q: shapes.index(subs[q].ext))
        self.subs = [subs[q] for q in order]
        self.order = order
        self.shapes = shapes
        self.factors = FactorTable(shapes, self.alpha, self.device)
        self.pmax = max(max(e) for e in shapes)
        # ---- rotation groups (one C^-1 / Y / Z / GEMM per group) and their row maps
        self.groups = rotation_groups(shapes) if share_rotations else [(q, 0) for q in range(len(shapes))]
        maps, rm_off, off = [], [], 0
        for g, t in self.groups:
            if t == 0:
                rm_off.append(-1)
            else:
                maps.append(rotation_rowmap(shapes[g], t))
                rm_off.append(off)
                off += maps[-1].size
        self.rowmap = torch.from_numpy(np.concatenate(maps)).to(self.device) if maps else None
        # ---- shape table
        sh_rec = np.zeros((len(shapes), 20), dtype=np.int64)
        self.m = []
        for q, e in enumerate(shapes):
            mc = correction_counts(e)
            self.m.append(sum(mc))
            offs = [self.factors.offsets[n] for n in e]
            sh_rec[q] = [*e, sum(mc), *mc, *(o[0] for o in offs), *(o[1] for o in offs), *(o[2] for o in offs),
                         self.factors.qw[e], lead_dim(sum(mc)), self.groups[q][0], rm_off[q]]
        # ---- subdomain table, workspace layout
        sub_rec = np.zeros((len(self.subs), 16), dtype=np.int64)
        first = np.zeros(len(shapes) + 1, dtype=np.int64)
        col_of_shape = [0] * len(shapes)
        ws = 0
        col_of_group = [0] * len(shapes)
        for q, s in enumerate(self.subs):
            sid = shapes.index(s.ext)
            gid = self.groups[sid][0]
            sub_rec[q] = [*s.ext, *s.ext_lo, *s.own_off, *s.own, sid, col_of_group[gid], ws, s.in_off]
            col_of_shape[sid] += 1
            col_of_group[gid] += 1
            ps = (s.ext[0] * s.ext[1] + 3) // 4 * 4      # plane stride of a workspace slot (csrc SubD::ps)
            ws += (3 * s.ext[2] * ps + 7) // 8 * 8
        for q in range(len(shapes)):
            first[q + 1] = first[q] + col_of_shape[q]
        self.ncols = col_of_shape
        self.ws_size = ws
        self._sub_host, self._sh_host, self._first = sub_rec, sh_rec, first
        self.sub_dev = torch.from_numpy(sub_rec).to(self.device)
        self.sh_dev = torch.from_numpy(sh_rec).to(self.device)
        f64 = dict(dtype=torch.float64, device=self.device)
        # zero-filled: the plane-stride padding of every slot must stay finite (it is read as
        # DMMA operand padding and multiplied by zero factor entries)
        self.work_a = torch.zeros(ws, **f64)
        self.work_b = torch.zeros(ws, **f64)
        self.corr = torch.zeros(len(self.subs) * 6 * self.pmax * self.pmax, **f64)
        # per-group Y/Z matrices: row j = group column j, row stride ld (zero padding); the
        # members of a group alias the canonical shape's matrices
        self.ld = [lead_dim(m) for m in self.m]
        self.gcols = col_of_group
        self.ymat, self.zmat = [], []
        for q, (g, _) in enumerate(self.groups):
            if g == q:
                self.ymat.append(torch.zeros((max(1, col_of_group[q]), self.ld[q]), **f64))
                self.zmat.append(torch.zeros((max(1, col_of_group[q]), self.ld[q]), **f64))
            else:
                self.ymat.append(self.ymat[g])
                self.zmat.append(self.zmat[g])
        self.cinv = []
        for q, (e, m, ld) in enumerate(zip(shapes, self.m, self.ld)):
            g = self.groups[q][0]
            if g != q:
                self.cinv.append(self.cinv[g])
                continue
            t = (cinv or {}).get(e)
            if t is None:
                if need_woodbury:
                    raise ValueError(f"missing C^-1 for shape {e}")
                t = torch.zeros(1, **f64)
            else:
                if t.dtype != torch.float64 or t.shape not in ((m, m), (m, ld)):
                    raise ValueError(f"C^-1 for {e} must be a float64 ({m}, {m}) or ({m}, {ld}) tensor")
                if t.shape != (m, ld) or not t.is_contiguous():
                    t = pad_rows(t, ld)
            self.cinv.append(t)
        P = C.c_void_p
        # null C^-1 pointers tell the library this plan never applies the Woodbury correction
        self._cinv_arr = (P * len(shapes))(*[(t.data_ptr() if t.numel() > 1 or need_woodbury else None)
                                               for t in self.cinv])
        self._y_arr = (P * len(shapes))(*[t.data_ptr() for t in self.ymat])
        self._z_arr = (P * len(shapes))(*[t.data_ptr() for t in self.zmat])
        desc = _lib.FmpPrecondDesc()
        desc.alpha = self.alpha
        desc.n_sub, desc.n_shape = len(self.subs), len(shapes)
        desc.subs, desc.shapes = self.sub_dev.data_ptr(), self.sh_dev.data_ptr()
        desc.subs_host, desc.shapes_host = sub_rec.ctypes.data, sh_rec.ctypes.data
        desc.shape_first = first.ctypes.data
        desc.factors = self.factors.device.data_ptr()
        desc.cinv = C.cast(self._cinv_arr, P)
        desc.work_a, desc.work_b = self.work_a.data_ptr(), self.work_b.data_ptr()
        desc.corr = self.corr.data_ptr()
        desc.ymat, desc.zmat = C.cast(self._y_arr, P), C.cast(self._z_arr, P)
        desc.pmax = self.pmax
        desc.rowmap = self.rowmap.data_ptr() if self.rowmap is not None else None
        handle = C.c_void_p()
        _lib.check(_lib.lib().fmp_precond_create(C.byref(desc), C.byref(handle)), "fmp_precond_create")
        self._handle = handle

    def apply(self, blk: _lib.FmpBlock, mode: int, r: torch.Tensor, z: torch.Tensor | None,
              part: int = _lib.FMP_PART_ALL) -> None:
        """fmp_precond_apply; part = FMP_PART_INTERIOR / _BOUNDARY splits it around a ghost exchange."""
        zp = _lib.ptr(z) if z is not None else None
        if part == _lib.FMP_PART_ALL:
            rc = _lib.lib().fmp_precond_apply(self._handle, C.byref(blk), mode, _lib.ptr(r), zp, _lib.stream())
        else:
            rc = _lib.lib().fmp_precond_apply_part(self._handle, C.byref(blk), mode, part, _lib.ptr(r), zp,
                                                   _lib.stream())
        _lib.check(rc, "fmp_precond_apply")

    def apply_lincomb(self, blk: _lib.FmpBlock, mode: int, r: torch.Tensor, v: torch.Tensor, beta: float,
                      s: torch.Tensor, z: torch.Tensor) -> None:
        """fmp_precond_apply_lincomb: s = r + beta v, z = M s in one apply (BiCGSTAB's s update
        fused into the forward plane pass; bit-identical to the two-pass form)."""
        rc = _lib.lib().fmp_precond_apply_lincomb(self._handle, C.byref(blk), mode, _lib.ptr(r), _lib.ptr(v),
                                                  float(beta), _lib.ptr(s), _lib.ptr(z), _lib.stream())
        _lib.check(rc, "fmp_precond_apply_lincomb")

    def apply_bicg_p(self, blk: _lib.FmpBlock, mode: int, r: torch.Tensor, p_old: torch.Tensor, v: torch.Tensor,
                     beta: float, omega: float, p_new: torch.Tensor, z: torch.Tensor) -> None:
        """fmp_precond_apply_bicg_p: p_new = r + beta (p_old - omega v), z = M p_new in one apply."""
        rc = _lib.lib().fmp_precond_apply_bicg_p(self._handle, C.byref(blk), mode, _lib.ptr(r), _lib.ptr(p_old),
                                                 _lib.ptr(v), float(beta), float(omega), _lib.ptr(p_new),
                                                 _lib.ptr(z), _lib.stream())
        _lib.check(rc, "fmp_precond_apply_bicg_p")

    def path(self) -> str:
        """Transform kernel family of this plan: 'fast', 'large' or 'general' (fmp_precond_path)."""
        return {0: "general", 1: "fast", 2: "large"}[_lib.lib().fmp_precond_path(self._handle)]

    def ozaki_stats(self) -> dict:
        """Zero-slice skipping of the Ozaki GEMM (fmp_precond_ozaki_stats): fractions of the C^-1
        slice blocks streamed and of the dense MMA work issued."""
        buf = (C.c_double * 2)()
        n = _lib.lib().fmp_precond_ozaki_stats(self._handle, buf, 2)
        _lib.check(0 if n >= 0 else n, "fmp_precond_ozaki_stats")
        return {"kept_slices": float(buf[0]), "kept_mma": float(buf[1])}

    def ozaki_kept_slices(self) -> float:
        return self.ozaki_stats()["kept_slices"]

    def gemm_kind(self) -> str:
        """Woodbury GEMM this plan was created with: 'ozaki' (default), 'own' or 'cublas'."""
        return self._gemm

    STAGES = ("plane_fwd", "column_fwd", "faces", "slice_y", "gemm", "corr", "column_inv", "plane_inv")

    def profile(self, enable: bool = True) -> None:
        """Record CUDA events between the kernels of later applies (fmp_precond_profile)."""
        _lib.check(_lib.lib().fmp_precond_profile(self._handle, int(enable)), "fmp_precond_profile")

    def stage_ms(self) -> dict:
        """Per-stage times (ms) of the last Woodbury apply (synchronises on it)."""
        buf = (C.c_float * len(self.STAGES))()
        n = _lib.lib().fmp_precond_stage_ms(self._handle, buf, len(self.STAGES))
        _lib.check(0 if n >= 0 else n, "fmp_precond_stage_ms")
        return {k: float(buf[i]) for i, k in enumerate(self.STAGES[:n])}

    def restrict(self, blk: _lib.FmpBlock, r: torch.Tensor) -> torch.Tensor:
        """Every subdomain's extended vector, concatenated in plan order at ws offsets."""
        out = torch.empty_like(self.work_a)
        _lib.check(_lib.lib().fmp_precond_restrict(self._handle, C.byref(blk), _lib.ptr(r), _lib.ptr(out),
                                                   _lib.stream()), "fmp_precond_restrict")
        return out

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value and _lib._LIB is not None:
            _lib._LIB.fmp_precond_destroy(h)
            self._handle = None


def block_struct(bx, by, bz, origin=(0, 0, 0), global_ext=None, halo=0, ghosts=None) -> _lib.FmpBlock:
    """fmp_block for a field of extents (bx, by, bz) at `origin` inside `global_ext`."""
    b = _lib.FmpBlock()
    b.bx, b.by, b.bz = bx, by, bz
    b.gx0, b.gy0, b.gz0 = origin
    b.nx, b.ny, b.nz = global_ext if global_ext is not None else (bx, by, bz)
    b.halo = halo
    for q in range(6):
        g = None if ghosts is None else ghosts[q]
        b.ghost[q] = g.data_ptr() if g is not None else None
    return b

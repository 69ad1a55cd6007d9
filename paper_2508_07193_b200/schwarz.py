"""Domain decomposition, halo exchange and the RAS preconditioner (mirror of ref:schwarz.py).

Two levels of decomposition:

* the reference's subdomain partition (`make_partition`, identical geometry and rank
  order, ref:schwarz.py:78-123): the preconditioner's mathematics depends only on it;
* the GPU decomposition: one process per GPU owns a contiguous block of subdomain
  tiles (`BlockLayout`, GPU grid = the reference CLI's `_proc_grid_for(N)`,
  ref:cli.py:214-231).  Inside a GPU, a subdomain's overlap region is read straight
  from the block field -- no halo copy at all; across GPUs the block's ghost shell is
  filled by a three-phase (z, y, x) face exchange over NCCL, which also carries edges
  and corners.

Vectors are per-GPU block tensors (3, bz, by, bx) in the reference's component-major
order.  The reference's list-of-rank-vectors form is accepted on a single GPU for
drop-in use (converted at the boundary).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from itertools import product

import numpy as np
import torch

from . import _lib
from .grid import Box, FieldVector
from .instrument import NULL_TIMER
from .operators import OperatorParams
from .plan import SolvePlan, SubSpec, block_struct, rotation_groups
from . import subdomain

Range3 = tuple[tuple[int, int], tuple[int, int], tuple[int, int]]


class CommunicationError(RuntimeError):
    """Mismatched collective participation or lost halo message (ref:schwarz.py:45)."""


# ---------------------------------------------------------------------------- geometry
@dataclass(frozen=True)
class RankGeometry:
    rank: int
    coords: tuple[int, int, int]
    owned_lo: tuple[int, int, int]
    owned: Box
    ext_lo: tuple[int, int, int]
    ext: Box
    neighbors: tuple[tuple[tuple[int, int, int], int], ...]

    def owned_range(self) -> Range3:
        return tuple((lo, lo + n) for lo, n in zip(self.owned_lo, self.owned.extents))

    def ext_range(self) -> Range3:
        return tuple((lo, lo + n) for lo, n in zip(self.ext_lo, self.ext.extents))


@dataclass(frozen=True)
class Partition:
    global_box: Box
    proc_grid: tuple[int, int, int]
    overlap: int
    ranks: tuple[RankGeometry, ...]

    @property
    def nranks(self) -> int:
        return len(self.ranks)


def make_partition(global_box: Box, proc_grid: tuple[int, int, int], overlap: int) -> Partition:
    """Owned tiles + extended boxes clamped at the physical boundary, rank x-fastest
    (ref:schwarz.py:78-123; same validation messages)."""
    grid = tuple(int(p) for p in proc_grid)
    if min(grid) < 1:
        raise ValueError(f"process grid must be positive, got {proc_grid}")
    if overlap < 0:
        raise ValueError(f"overlap must be >= 0, got {overlap}")
    for n, p, ax in zip(global_box.extents, grid, "xyz"):
        if n % p:
            raise ValueError(f"extent {n} along {ax} not divisible by grid {p}")
    tile = tuple(n // p for n, p in zip(global_box.extents, grid))
    if overlap > min(tile):
        raise ValueError(f"overlap {overlap} exceeds smallest tile extent {min(tile)}")
    px, py, pz = grid
    rank_of = lambda c: c[0] + px * (c[1] + py * c[2])
    ranks = []
    for cz, cy, cx in product(range(pz), range(py), range(px)):
        c = (cx, cy, cz)
        lo = tuple(q * t for q, t in zip(c, tile))
        elo = tuple(max(0, l - overlap) for l in lo)
        ehi = tuple(min(n, l + t + overlap) for n, l, t in zip(global_box.extents, lo, tile))
        nb = []
        if overlap > 0:
            for dz, dy, dx in product((-1, 0, 1), repeat=3):
                q = (cx + dx, cy + dy, cz + dz)
                if (dx, dy, dz) != (0, 0, 0) and all(0 <= a < b for a, b in zip(q, grid)):
                    nb.append(((dx, dy, dz), rank_of(q)))
        ranks.append(RankGeometry(rank_of(c), c, lo, Box(*tile), elo,
                                  Box(*(h - l for l, h in zip(elo, ehi))), tuple(nb)))
    return Partition(global_box, grid, int(overlap), tuple(ranks))


def _intersect(a: Range3, b: Range3) -> Range3 | None:
    out = tuple((max(a0, b0), min(a1, b1)) for (a0, a1), (b0, b1) in zip(a, b))
    return None if any(lo >= hi for lo, hi in out) else out


def _local_slices(region: Range3, origin):
    (x0, x1), (y0, y1), (z0, z1) = region
    ox, oy, oz = origin
    return (slice(None), slice(z0 - oz, z1 - oz), slice(y0 - oy, y1 - oy), slice(x0 - ox, x1 - ox))


def proc_grid_for(nranks: int) -> tuple[int, int, int]:
    """Most cubic (px, py, pz), ties to the larger px (ref:cli.py:214-231)."""
    if nranks < 1:
        raise ValueError(f"rank count must be >= 1, got {nranks}")
    best = None
    for px in range(1, nranks + 1):
        if nranks % px:
            continue
        for py in range(1, nranks // px + 1):
            if (nranks // px) % py:
                continue
            pz = nranks // px // py
            key = (max(px, py, pz) - min(px, py, pz), -px)
            if best is None or key < best[0]:
                best = (key, (px, py, pz))
    return best[1]


# ---------------------------------------------------------------------------- transports
class DeviceTransport:
    """One process, one GPU (stands in for the reference's serial/threads transports)."""

    name = "cuda"
    world = 1
    rank = 0
    distributed = False

    def __init__(self, device=None):
        self.device = _lib.require_cuda(device) if device is None or str(device) != "cpu" else torch.device("cpu")

    def run_ranks(self, fns) -> None:
        for fn in fns:
            fn()

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        return t

    def close(self) -> None:
        pass


class DistTransport:
    """One process per GPU over torch.distributed.

    NCCL moves device tensors directly (NVLink); with the gloo backend device tensors are
    staged through host memory, which lets the multi-block path run (and be tested) with
    several processes sharing one GPU, or on CPU tensors for the host-side logic."""

    name = "nccl"
    distributed = True

    def __init__(self, device=None, group=None, backend: str | None = None):
        import torch.distributed as dist
        if not dist.is_initialized():
            backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.name = dist.get_backend(group)
        if device is None:
            if torch.cuda.is_available():
                device = torch.device("cuda", int(os.environ.get("LOCAL_RANK", self.rank)) % torch.cuda.device_count())
            else:
                device = torch.device("cpu")
        self.device = torch.device(device)
        if self.device.type == "cuda":
            torch.cuda.set_device(self.device)
        self.staged = self.name != "nccl" and self.device.type == "cuda"

    def run_ranks(self, fns) -> None:
        for fn in fns:
            fn()

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self.staged:   # gloo with device tensors: through a host copy (testing backend)
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:             # NCCL: in place, on the current stream
            self.dist.all_reduce(t, group=self.group)
        return t

    def exchange(self, sends: list[tuple[int, torch.Tensor]], recvs: list[tuple[int, torch.Tensor]]) -> None:
        """Grouped point-to-point messages.  NCCL: device tensors, issued on the current stream and
        waited for on it (no host block).  gloo: host tensors (HaloExchanger stages device slabs
        through pinned buffers), blocking."""
        ops = [self.dist.P2POp(self.dist.isend, t, peer, self.group) for peer, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t, peer, self.group) for peer, t in recvs]
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def barrier(self) -> None:
        self.dist.barrier(group=self.group)

    def close(self) -> None:
        pass


def make_transport(name: str, nranks: int | None = None, device=None):
    """'cuda' (aliases 'serial', 'threads': one GPU) or 'nccl' / 'gloo' (one process per
    device under torch.distributed).  Unknown names raise ValueError (ref:schwarz.py:174-179)."""
    if name in ("cuda", "serial", "threads"):
        return DeviceTransport(device)
    if name in ("nccl", "gloo"):
        return DistTransport(device, backend=name)
    if name == "dist":
        return DistTransport(device)
    raise ValueError(f"unknown transport {name!r}")


# ---------------------------------------------------------------------------- GPU blocks
class BlockLayout:
    """This process's block of the global grid and the subdomains it owns."""

    def __init__(self, partition: Partition, transport):
        self.partition = partition
        self.transport = transport
        self.world, self.rank = transport.world, transport.rank
        self.device = transport.device
        g = proc_grid_for(self.world)
        for sp, gp, ax in zip(partition.proc_grid, g, "xyz"):
            if sp % gp:
                raise ValueError(f"subdomain grid {partition.proc_grid} not divisible by GPU grid {g} along {ax}")
        self.gpu_grid = g
        gx, gy, gz = g
        self.coords = (self.rank % gx, (self.rank // gx) % gy, self.rank // (gx * gy))
        gext = partition.global_box.extents
        self.block = tuple(n // p for n, p in zip(gext, g))
        self.origin = tuple(c * b for c, b in zip(self.coords, self.block))
        self.box = Box(*self.block)
        lo, hi = self.origin, tuple(o + b for o, b in zip(self.origin, self.block))
        self.local_ranks = [r for r in partition.ranks
                            if all(l <= o < h for o, l, h in zip(r.owned_lo, lo, hi))]
        self.rank_of_gpu = lambda c: c[0] + gx * (c[1] + gy * c[2])

    @property
    def shape4(self):
        return self.box.shape4

    def neighbor(self, axis: int, side: int) -> int | None:
        c = list(self.coords)
        c[axis] += side
        if not 0 <= c[axis] < self.gpu_grid[axis]:
            return None
        return self.rank_of_gpu(tuple(c))

    def sub_specs(self) -> list[SubSpec]:
        out = []
        for r in self.local_ranks:
            elo = tuple(e - o for e, o in zip(r.ext_lo, self.origin))
            own_off = tuple(o - e for o, e in zip(r.owned_lo, r.ext_lo))
            out.append(SubSpec(r.ext.extents, elo, own_off, r.owned.extents))
        return out

    def block_struct(self, ghosts=None, halo: int = 0) -> _lib.FmpBlock:
        return block_struct(*self.block, origin=self.origin, global_ext=self.partition.global_box.extents,
                            halo=halo, ghosts=ghosts)

    # ---- conversions between the reference list form and block tensors (single GPU)
    def from_list(self, dist: list) -> torch.Tensor:
        if self.world != 1:
            raise CommunicationError("list-form vectors are only supported on a single GPU")
        full = gather_field(self.partition, [np.asarray(a) for a in dist])
        return torch.from_numpy(full).to(self.device).view(self.shape4)

    def to_list(self, x: torch.Tensor) -> list[np.ndarray]:
        return scatter_field(self.partition, x.detach().cpu().numpy().ravel())

    def as_block(self, v) -> tuple[torch.Tensor, bool]:
        """(block tensor, was_list)."""
        if isinstance(v, torch.Tensor):
            if tuple(v.shape) != self.shape4:
                v = v.reshape(self.shape4)
            return v, False
        return self.from_list(v), True


class HaloExchanger:
    """Fills the ghost shell (width P) of a block field from the neighbour GPUs.

    Three phases: z faces, then y faces extended over the z ghosts, then x faces extended over
    both, so edges and corners arrive without diagonal messages (slab layout: fmp_block in
    include/flashmp_b200.h).  Replaces the reference's per-subdomain mailbox messages
    (ref:schwarz.py:217-257) with one slab per GPU face and phase.

    * Allocation-free: send slabs and ghost slots (each with a trailing tag double) are allocated
      once here; NCCL receives straight into the ghost slots.
    * Device packing: fmp_halo_pack builds every slab in one kernel (reading the ghosts of the
      earlier phases); fmp_halo_unpack checks the slab's tag (epoch * 3 + phase), so a lost or
      stale message sets a bit in a host-mapped status word and `check()` raises
      CommunicationError (ref:schwarz.py:237-257).
    * Overlap: `start(x)` issues the exchange on a side stream (NCCL) or a worker thread (gloo
      staging through pinned host buffers) and returns; the caller launches the interior work
      (FMP_PART_INTERIOR) and then `finish()` orders its stream after the ghosts.
    * CPU tensors (gloo, host-logic tests) take the same three phases with torch slicing.

    `trace` keeps the reference's message rows (epoch, src, dst, bytes) for the SUBDOMAIN
    messages this block's subdomains send (ref:schwarz.py:186-188, 234-235; inside a GPU they are
    in-place reads, across GPUs they travel inside the slabs); `gpu_trace` the slabs actually sent.
    """

    PHASE_SLOTS = ((4, 5), (2, 3), (0, 1))   # ghost slots (lo, hi) of phases z, y, x

    def __init__(self, layout: BlockLayout, width: int, record_trace: bool = False):
        self.layout = layout
        self.P = P = int(width)
        self.epoch = 0
        self.trace: list[tuple[int, int, int, int]] = []
        self.gpu_trace: list[tuple[int, int, int, int]] = []
        self.record_trace = record_trace
        self.drop_phase = None   # test hook: (phase, side) whose message is neither sent nor received
        bx, by, bz = layout.block
        dev = layout.device
        nb = [layout.neighbor(a, s) for a in (0, 1, 2) for s in (-1, 1)]
        self.nb = nb   # xlo, xhi, ylo, yhi, zlo, zhi
        shapes = [(3, bz + 2 * P, by + 2 * P, P)] * 2 + [(3, bz + 2 * P, P, bx)] * 2 + [(3, P, by, bx)] * 2
        self.active = any(n is not None for n in nb) and P > 0
        self.cuda = dev.type == "cuda"
        f64 = dict(dtype=torch.float64, device=dev)
        # ghost slot q = a flat buffer of numel + 1 doubles (the tag last); ghosts[q] is its view
        self._gbuf = [torch.zeros(int(np.prod(sh)) + 1, **f64) if (n is not None and P > 0) else None
                      for sh, n in zip(shapes, nb)]
        self.ghosts = [b[:-1].view(sh) if b is not None else None for b, sh in zip(self._gbuf, shapes)]
        # send slab of (phase, side): the same size as the receiving ghost slot on the other side
        self._send = {}
        for ph, slots in enumerate(self.PHASE_SLOTS):
            for side, q in enumerate(slots):
                if nb[q] is not None and P > 0:
                    self._send[(ph, side)] = torch.zeros(int(np.prod(shapes[q])) + 1, **f64)
        self._msgs = self._subdomain_messages() if record_trace else []
        tr = layout.transport
        self.staged = bool(getattr(tr, "staged", False)) and self.cuda
        self._thread = None
        self._error = None
        if self.cuda and self.active:
            self.stream = torch.cuda.Stream(device=dev)
            self.done = torch.cuda.Event()
            self._status = torch.zeros(1, dtype=torch.int32, pin_memory=True)
            if self.staged:   # pinned host staging for gloo: sends and receives, allocated once
                self._hsend = {k: torch.empty(v.numel(), dtype=torch.float64, pin_memory=True)
                               for k, v in self._send.items()}
                self._hrecv = {q: torch.empty(b.numel(), dtype=torch.float64, pin_memory=True)
                               for q, b in enumerate(self._gbuf) if b is not None}

    # ---- geometry / trace
    def _subdomain_messages(self):
        """The reference Exchanger's messages sent by this block's subdomains, in its pack order:
        rank i sends intersect(owned_i, ext_j) to each neighbour j (ref:schwarz.py:203-213)."""
        part = self.layout.partition
        mine = {r.rank for r in self.layout.local_ranks}
        rows = []
        for info in part.ranks:
            if info.rank not in mine:
                continue
            for _, j in info.neighbors:
                reg = _intersect(info.owned_range(), part.ranks[j].ext_range())
                if reg is not None:
                    rows.append((info.rank, j, 3 * 8 * int(np.prod([hi - lo for lo, hi in reg]))))
        return rows

    def block_struct(self) -> _lib.FmpBlock:
        return self.layout.block_struct(self.ghosts if self.active else None, self.P if self.active else 0)

    def _tag(self, phase: int) -> float:
        return float(self.epoch * 3 + phase)

    # ---- exchange
    def exchange(self, x: torch.Tensor) -> None:
        """Synchronous form: start + finish (the ghosts are ready on the current stream)."""
        self.start(x)
        self.finish()

    def start(self, x: torch.Tensor) -> None:
        if self.record_trace:
            self.trace.extend((self.epoch + 1, s, d, b) for s, d, b in self._msgs)
        if not self.active:
            self.epoch += 1
            return
        self.epoch += 1
        if not self.cuda:
            self._run_cpu(x)
            return
        self.stream.wait_stream(torch.cuda.current_stream())   # x is ready on the caller's stream
        if self.staged:
            import threading
            dev = self.layout.device

            def work():
                try:
                    torch.cuda.set_device(dev)
                    self._run_device(x)
                except BaseException as e:   # re-raised by finish()
                    self._error = e
            self._thread = threading.Thread(target=work, daemon=True)
            self._thread.start()
        else:
            self._run_device(x)

    def finish(self) -> None:
        if not (self.active and self.cuda):
            return
        if self._thread is not None:
            self._thread.join()
            self._thread = None
            if self._error is not None:
                e, self._error = self._error, None
                raise e
        torch.cuda.current_stream().wait_event(self.done)

    def check(self) -> None:
        """Raise CommunicationError if any unpack saw a wrong tag (lost / stale message).  The
        status word is written by the device; read it after a synchronisation point."""
        if self.active and self.cuda:
            bits = int(self._status[0])
            if bits:
                names = ["x-lo", "x-hi", "y-lo", "y-hi", "z-lo", "z-hi"]
                self._status.zero_()
                raise CommunicationError(f"rank {self.layout.rank}: missing or stale halo message "
                                         f"({', '.join(n for q, n in enumerate(names) if bits >> q & 1)}) "
                                         f"by epoch {self.epoch}")

    def _pairs(self, phase):
        """[(side, peer, ghost slot)] of the phase, minus a test-dropped message."""
        out = []
        for side, q in enumerate(self.PHASE_SLOTS[phase]):
            peer = self.nb[q]
            if peer is None:
                continue
            out.append((side, peer, q))
        return out

    def _dropped(self, phase, side, sending):
        """Test hook: drop_phase = (phase, side) skips this rank's send toward `side` and, on the
        neighbour, the matching receive (its opposite side)."""
        if self.drop_phase is None:
            return False
        dp, ds = self.drop_phase
        return dp == phase and (ds == side if sending else ds == 1 - side)

    def _run_device(self, x):
        tr = self.layout.transport
        lib = _lib.lib()
        with torch.cuda.stream(self.stream):
            st = self.stream.cuda_stream
            blk = self.block_struct()
            for ph in range(3):
                pairs = self._pairs(ph)
                tag = self._tag(ph)
                for side, peer, q in pairs:
                    _lib.check(lib.fmp_halo_pack(_lib.ref(blk), ph, side, _lib.ptr(x),
                                                 _lib.ptr(self._send[(ph, side)]), tag, st), "fmp_halo_pack")
                sends = [(peer, self._send[(ph, side)], side) for side, peer, q in pairs
                         if not self._dropped(ph, side, True)]
                recvs = [(peer, self._gbuf[q], q) for side, peer, q in pairs if not self._dropped(ph, side, False)]
                if self.record_trace:
                    self.gpu_trace.extend((self.epoch, self.layout.rank, p, (b.numel() - 1) * 8) for p, b, _ in sends)
                if self.staged:
                    for p, b, side in sends:
                        self._hsend[(ph, side)].copy_(b, non_blocking=True)
                    self.stream.synchronize()
                    tr.exchange([(p, self._hsend[(ph, side)]) for p, b, side in sends],
                                [(p, self._hrecv[q]) for p, b, q in recvs])
                    for p, b, q in recvs:
                        b.copy_(self._hrecv[q], non_blocking=True)
                else:
                    tr.exchange([(p, b) for p, b, _ in sends], [(p, b) for p, b, _ in recvs])
                for side, peer, q in pairs:
                    _lib.check(lib.fmp_halo_unpack(_lib.ref(blk), ph, side, _lib.ptr(self._gbuf[q]), tag,
                                                   self._status.data_ptr(), st), "fmp_halo_unpack")
            self.done.record(self.stream)

    def _run_cpu(self, x):
        """Host tensors (gloo): the same three phases built with torch slicing."""
        P = self.P
        bx, by, bz = self.layout.block
        xlo, xhi, ylo, yhi, zlo, zhi = self.ghosts
        tr = self.layout.transport

        def swap(ph, slabs):
            pairs = self._pairs(ph)
            sends = []
            for side, peer, q in pairs:
                buf = self._send[(ph, side)]
                buf[:-1].view(slabs[side].shape).copy_(slabs[side])
                buf[-1] = self._tag(ph)
                if not self._dropped(ph, side, True):
                    sends.append((peer, buf))
            recvs = [(peer, self._gbuf[q]) for side, peer, q in pairs if not self._dropped(ph, side, False)]
            if self.record_trace:
                self.gpu_trace.extend((self.epoch, self.layout.rank, p, (b.numel() - 1) * 8) for p, b in sends)
            tr.exchange(sends, recvs)
            for side, peer, q in pairs:
                if float(self._gbuf[q][-1]) != self._tag(ph):
                    raise CommunicationError(f"rank {self.layout.rank}: missing or stale halo message from "
                                             f"{peer} in epoch {self.epoch}")

        swap(0, {0: x[:, :P], 1: x[:, bz - P:]})

        def zext(rows: slice):  # (3, bz+2P, |rows|, bx): block rows with the z ghosts around them
            w = rows.stop - rows.start
            parts = [zlo[:, :, rows] if zlo is not None else x.new_zeros((3, P, w, bx)), x[:, :, rows],
                     zhi[:, :, rows] if zhi is not None else x.new_zeros((3, P, w, bx))]
            return torch.cat(parts, dim=1)

        swap(1, {0: zext(slice(0, P)), 1: zext(slice(by - P, by))})

        def padded_cols(c0: int, c1: int):  # (3, bz+2P, by+2P, c1-c0)
            out = x.new_zeros((3, bz + 2 * P, by + 2 * P, c1 - c0))
            out[:, P:P + bz, P:P + by] = x[..., c0:c1]
            if ylo is not None:
                out[:, :, :P] = ylo[..., c0:c1]
            if yhi is not None:
                out[:, :, P + by:] = yhi[..., c0:c1]
            if zlo is not None:
                out[:, :P, P:P + by] = zlo[..., c0:c1]
            if zhi is not None:
                out[:, P + bz:, P:P + by] = zhi[..., c0:c1]
            return out

        swap(2, {0: padded_cols(0, P), 1: padded_cols(bx - P, bx)})

    def write_trace_csv(self, path) -> None:
        """The reference's comm trace schema (ref:schwarz.py:259-266)."""
        import csv
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["epoch", "src_rank", "dst_rank", "bytes"])
            w.writerows(self.trace)


# ---------------------------------------------------------------------------- host helpers
def scatter_field(partition: Partition, global_data) -> list[np.ndarray]:
    """Global component-major vector -> per-rank owned vectors (ref:schwarz.py:273-281)."""
    g = partition.global_box
    view = np.asarray(global_data).reshape(g.shape4)
    return [np.ascontiguousarray(view[_local_slices(r.owned_range(), (0, 0, 0))]).ravel()
            for r in partition.ranks]


def gather_field(partition: Partition, dist) -> np.ndarray:
    """Inverse of scatter_field (ref:schwarz.py:284-292)."""
    g = partition.global_box
    full = np.empty(g.shape4)
    for r, arr in zip(partition.ranks, dist):
        full[_local_slices(r.owned_range(), (0, 0, 0))] = np.asarray(arr).reshape(r.owned.shape4)
    return full.ravel()


_SOLVER_CACHE: dict = {}


def solver_data_for(box: Box, alpha: float, device=None) -> subdomain.SubdomainSolverData:
    """Shared precompute cache keyed by (extents, alpha) (ref:schwarz.py:295-305)."""
    dev = _lib.require_cuda(device)
    key = (box.extents, float(alpha), str(dev))
    data = _SOLVER_CACHE.get(key)
    if data is None:
        data = subdomain.precompute(OperatorParams(box, alpha), dev)
        _SOLVER_CACHE[key] = data
    return data


# ---------------------------------------------------------------------------- exchanger (API parity)
class Exchanger:
    """Reference-compatible halo gather: per-subdomain extended vectors (ref:schwarz.py:182-266).

    The extended vectors are produced by the same device restriction the fused solve
    uses (fmp_precond_restrict), so this doubles as the bit-exact index-map check."""

    def __init__(self, partition: Partition, transport, record_trace: bool = False):
        self.partition = partition
        self.layout = BlockLayout(partition, transport)
        self.halo = HaloExchanger(self.layout, max(1, partition.overlap), record_trace)
        self.plan = SolvePlan(self.layout.sub_specs(), 0.0, self.layout.device, need_woodbury=False)
        self.epoch = 0

    @property
    def trace(self):
        return self.halo.trace

    def exchange(self, locals_):
        x, was_list = self.layout.as_block(locals_) if not isinstance(locals_, torch.Tensor) else (locals_, False)
        if was_list and len(locals_) != self.partition.nranks:
            raise CommunicationError(f"expected {self.partition.nranks} rank vectors, got {len(locals_)}")
        self.epoch += 1
        self.halo.exchange(x)
        flat = self.plan.restrict(self.halo.block_struct(), x)
        offs = self.plan._sub_host[:, 14]
        sizes = 3 * self.plan._sub_host[:, 0] * self.plan._sub_host[:, 1] * self.plan._sub_host[:, 2]
        exts = [None] * len(self.plan.subs)
        host = flat.cpu().numpy() if was_list else None
        for pos, orig in enumerate(self.plan.order):
            seg = slice(int(offs[pos]), int(offs[pos] + sizes[pos]))
            exts[orig] = host[seg].copy() if was_list else flat[seg]
        return exts

    def write_trace_csv(self, path) -> None:
        self.halo.write_trace_csv(path)


def exchange_halo(exchanger: Exchanger, locals_):
    return exchanger.exchange(locals_)


# ---------------------------------------------------------------------------- RAS preconditioner
class RasPreconditioner:
    """Restricted additive Schwarz with exact subdomain solves (ref:schwarz.py:308-339).

    apply(r) = sum_i S_i^0T A_i^-1 S_i^gamma r over every subdomain of this GPU in one
    batched launch sequence (csrc/precond.cu); the restriction reads the overlap
    straight from the block field and its ghost shell, the prolongation writes the
    owned tiles straight into the output block."""

    def __init__(self, partition: Partition, alpha: float, transport, timer=NULL_TIMER,
                 record_trace: bool = False, share_rotations: bool = True):
        self.partition = partition
        self.alpha = float(alpha)
        self.timer = timer
        self.layout = BlockLayout(partition, transport)
        self.exchanger = HaloExchanger(self.layout, partition.overlap, record_trace)
        dev = self.layout.device
        self.solvers = {}
        specs = self.layout.sub_specs()
        cinv = {}
        if self.alpha != 0.0:
            # C^-1 only for the canonical shape of each rotation group (plan.rotation_groups)
            # (every shape's own C^-1 with share_rotations=False: the unshared reference layout)
            shapes = list(dict.fromkeys(s.ext for s in specs))
            for (g, _), e in zip(rotation_groups(shapes), shapes):
                if g == shapes.index(e) or not share_rotations:
                    data = solver_data_for(Box(*e), self.alpha, dev)
                    self.solvers[e] = data
                    cinv[e] = data.corr.padded
        self.plan = SolvePlan(specs, self.alpha, dev, cinv=cinv, share_rotations=share_rotations) \
            if self.alpha != 0.0 else None

    def apply_into(self, r: torch.Tensor, z: torch.Tensor) -> torch.Tensor:
        ex = self.exchanger
        ex.check()   # a lost / stale message of an earlier apply (status is final after any sync)
        if self.plan is None:
            ex.exchange(r)
            z.copy_(r)
            return z
        if not ex.active:
            with self.timer.phase("fast_solve"):
                self.plan.apply(ex.block_struct(), _lib.FMP_SOLVE_WOODBURY, r, z)
            return z
        # multi-GPU: the ghost exchange runs beside the interior subdomains' restriction and
        # x/y transforms; "asm_comm" times only the exposed wait for the ghosts
        ex.start(r)
        blk = ex.block_struct()
        with self.timer.phase("fast_solve"):
            self.plan.apply(blk, _lib.FMP_SOLVE_WOODBURY, r, z, part=_lib.FMP_PART_INTERIOR)
        with self.timer.phase("asm_comm"):
            ex.finish()
        with self.timer.phase("fast_solve"):
            self.plan.apply(blk, _lib.FMP_SOLVE_WOODBURY, r, z, part=_lib.FMP_PART_BOUNDARY)
        return z

    def apply_lincomb_into(self, r: torch.Tensor, v: torch.Tensor, beta: float, s: torch.Tensor,
                           z: torch.Tensor) -> torch.Tensor:
        """s = r + beta v, then z = M s (ref:krylov.py:199-201).  On one GPU the update is formed
        inside the apply's forward plane pass (fmp_precond_apply_lincomb, bit-identical); with
        ghost exchanges it is the plain vector kernel followed by apply_into."""
        if self.plan is None or self.exchanger.active:
            _lib.call("fmp_vec_lincomb", r.numel(), 1.0, _lib.ptr(r), float(beta), _lib.ptr(v), _lib.ptr(s),
                      _lib.stream())
            return self.apply_into(s, z)
        self.exchanger.check()
        with self.timer.phase("fast_solve"):
            self.plan.apply_lincomb(self.exchanger.block_struct(), _lib.FMP_SOLVE_WOODBURY, r, v, beta, s, z)
        return z

    def apply_bicg_p_into(self, r: torch.Tensor, p_old: torch.Tensor, v: torch.Tensor, beta: float, omega: float,
                          p_new: torch.Tensor, z: torch.Tensor) -> torch.Tensor:
        """p_new = r + beta (p_old - omega v), then z = M p_new (ref:krylov.py:179-187); fused into
        the apply on one GPU (fmp_precond_apply_bicg_p, bit-identical), else the vector kernel on a
        copy followed by apply_into."""
        if self.plan is None or self.exchanger.active:
            p_new.copy_(p_old)
            _lib.call("fmp_bicg_p", r.numel(), _lib.ptr(r), _lib.ptr(p_new), _lib.ptr(v), float(beta), float(omega),
                      _lib.stream())
            return self.apply_into(p_new, z)
        self.exchanger.check()
        with self.timer.phase("fast_solve"):
            self.plan.apply_bicg_p(self.exchanger.block_struct(), _lib.FMP_SOLVE_WOODBURY, r, p_old, v, beta, omega,
                                   p_new, z)
        return z

    def apply(self, r_dist):
        r, was_list = self.layout.as_block(r_dist)
        z = self.apply_into(r, torch.empty_like(r))
        return self.layout.to_list(z) if was_list else z


def ras_apply(prec: RasPreconditioner, r_dist):
    return prec.apply(r_dist)


# ---------------------------------------------------------------------------- operator
class DistributedOperator:
    """y = A x over this GPU's block (ref:schwarz.py:347-388): a width-1 ghost exchange
    (multi-GPU only) plus the matrix-free stencil kernel; optional fused dot products
    feed the Krylov solvers."""

    def __init__(self, partition: Partition, alpha: float, transport, timer=NULL_TIMER,
                 with_boundary: bool = True):
        self.partition = partition
        self.alpha = float(alpha)
        self.with_boundary = with_boundary
        self.timer = timer
        self.transport = transport
        self.layout = BlockLayout(partition, transport)
        self.exchanger = HaloExchanger(self.layout, 1)
        dev = self.layout.device
        self._dots = torch.zeros(2, dtype=torch.float64, device=dev)
        # one GPU: the fused dot products land in pinned host memory (no device->host copy)
        self._host = _lib.HostScalars(2) if transport.world == 1 else None
        self._scratch = torch.zeros(int(_lib.lib().fmp_reduce_scratch_doubles()), dtype=torch.float64, device=dev)

    def _run(self, mode: int, x: torch.Tensor, y, w):
        ex = self.exchanger
        dots = self._host.ptr() if self._host is not None else _lib.ptr(self._dots)
        args = (self.alpha, int(self.with_boundary), mode)
        ptrs = (_lib.ptr(x), _lib.ptr(y), _lib.ptr(w), dots, _lib.ptr(self._scratch), _lib.stream())
        if not ex.active:
            with self.timer.phase("spmv"):
                _lib.call("fmp_stencil_apply", _lib.ref(ex.block_struct()), *args, *ptrs)
            return
        # multi-GPU: interior units while the width-1 ghosts are in flight, then the faces;
        # "p2p" times only the exposed wait
        ex.start(x)
        blk = ex.block_struct()
        with self.timer.phase("spmv"):
            _lib.call("fmp_stencil_apply_part", _lib.ref(blk), *args, _lib.FMP_PART_INTERIOR, *ptrs)
        with self.timer.phase("p2p"):
            ex.finish()
        with self.timer.phase("spmv"):
            _lib.call("fmp_stencil_apply_part", _lib.ref(blk), *args, _lib.FMP_PART_BOUNDARY, *ptrs)

    def _reduced(self, n: int) -> list[float]:
        with self.timer.phase("reduction"):
            if self._host is not None:
                out = self._host.read(n)
            else:
                out = self.transport.allreduce_(self._dots[:n]).tolist()
        self.exchanger.check()   # synchronised here: a lost / stale ghost message raises now
        return out

    def apply_into(self, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        self._run(0, x, y, None)
        return y

    def apply(self, x_dist):
        x, was_list = self.layout.as_block(x_dist)
        y = self.apply_into(x, torch.empty_like(x))
        return self.layout.to_list(y) if was_list else y

    def apply_dots(self, x: torch.Tensor, y: torch.Tensor, w: torch.Tensor, both: bool) -> list[float]:
        """y = A x; returns [(y, w)] or [(y, w), (y, y)] summed over GPUs."""
        self._run(2 if both else 1, x, y, w)
        return self._reduced(2 if both else 1)

    def residual_norm2(self, x: torch.Tensor, b: torch.Tensor) -> float:
        """||b - A x||^2 over all GPUs, without materialising A x."""
        self._run(3, x, None, b)
        return self._reduced(1)[0]

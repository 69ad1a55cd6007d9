"""GPU tests of the multi-GPU ghost path on ONE device: the pack / unpack kernels of
the C ABI, and the interior / boundary split of the SpMV and of the RAS apply that lets the ghost
exchange overlap interior work.

A fake transport places this process at rank r of a 4-GPU grid ((2,1,2), BlockLayout), so the
block has neighbour faces; its ghosts are filled from a global field by hand (what the exchange
delivers).  Checks:
  * fmp_halo_pack produces exactly the neighbour's ghost slab for every phase and side, reading
    only the ghosts of EARLIER phases (later ones are NaN), plus the tag;
  * fmp_halo_unpack copies a message into its ghost slot and flags a wrong tag in the status word;
  * INTERIOR + BOUNDARY == ALL bitwise (y, fused dots, preconditioner output), with the ghosts NaN
    while the interior part runs -- so it provably reads no ghost cell;
  * the block result equals the single-block (global) result on the block's tile.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GEXT, SGRID, WORLD = (64, 32, 64), (4, 2, 4), 4     # GPU grid (2, 1, 2): blocks 32 x 32 x 32


class FakeTransport:
    distributed = True
    staged = False

    def __init__(self, world, rank):
        self.world, self.rank = world, rank
        self.device = torch.device("cuda", 0)


def global_field(seed=0):
    return np.random.default_rng(seed).uniform(-1, 1, (3, GEXT[2], GEXT[1], GEXT[0]))


def fill_ghosts(hx, G, P, phases=(0, 1, 2), fill=None):
    """Ghost slots of the exchanger from the global field G (zero outside the global box); slots of
    phases not listed get `fill` (NaN: any read of them poisons the result)."""
    lay = hx.layout
    (ox, oy, oz), (bx, by, bz) = lay.origin, lay.block
    Gp = np.pad(G, ((0, 0), (P, P), (P, P), (P, P)))
    zs, ys, xs = slice(oz, oz + bz + 2 * P), slice(oy, oy + by + 2 * P), slice(ox, ox + bx + 2 * P)
    want = {0: Gp[:, zs, ys, ox:ox + P], 1: Gp[:, zs, ys, ox + bx + P:ox + bx + 2 * P],
            2: Gp[:, zs, oy:oy + P, ox + P:ox + bx + P], 3: Gp[:, zs, oy + by + P:oy + by + 2 * P, ox + P:ox + bx + P],
            4: Gp[:, oz:oz + P, oy + P:oy + by + P, ox + P:ox + bx + P],
            5: Gp[:, oz + bz + P:oz + bz + 2 * P, oy + P:oy + by + P, ox + P:ox + bx + P]}
    phase_of = {0: 2, 1: 2, 2: 1, 3: 1, 4: 0, 5: 0}
    for q, gh in enumerate(hx.ghosts):
        if gh is None:
            continue
        if phase_of[q] in phases:
            gh.copy_(torch.from_numpy(np.ascontiguousarray(want[q])))
        else:
            gh.fill_(fill if fill is not None else float("nan"))
    return want


def block_of(lay, G):
    (ox, oy, oz), (bx, by, bz) = lay.origin, lay.block
    return torch.from_numpy(np.ascontiguousarray(G[:, oz:oz + bz, oy:oy + by, ox:ox + bx])).cuda()


@pytest.mark.parametrize("rank", [0, 3])
@pytest.mark.parametrize("P", [1, 2])
def test_pack_builds_the_neighbours_ghost_slab(rank, P):
    from paper_2508_07193_b200 import Box, _lib, make_partition
    from paper_2508_07193_b200.schwarz import BlockLayout, HaloExchanger
    part = make_partition(Box(*GEXT), SGRID, 1)
    lay = BlockLayout(part, FakeTransport(WORLD, rank))
    hx = HaloExchanger(lay, P)
    G = global_field(1)
    x = block_of(lay, G)
    (ox, oy, oz), (bx, by, bz) = lay.origin, lay.block
    Gp = np.pad(G, ((0, 0), (P, P), (P, P), (P, P)))
    lib = _lib.lib()
    for ph in range(3):
        fill_ghosts(hx, G, P, phases=tuple(range(ph)))      # only the earlier phases are valid
        blk = hx.block_struct()
        n = lib.fmp_halo_slab_doubles(_lib.ref(blk), ph)
        for side in (0, 1):
            out = torch.full((n + 1,), -7.0, dtype=torch.float64, device="cuda")
            _lib.call("fmp_halo_pack", _lib.ref(blk), ph, side, _lib.ptr(x), _lib.ptr(out), 12.0 + ph, _lib.stream())
            if ph == 0:
                k0 = oz + P + (bz - P if side else 0)
                want = Gp[:, k0:k0 + P, oy + P:oy + P + by, ox + P:ox + P + bx]
            elif ph == 1:
                j0 = oy + P + (by - P if side else 0)
                want = Gp[:, oz:oz + bz + 2 * P, j0:j0 + P, ox + P:ox + P + bx]
            else:
                i0 = ox + P + (bx - P if side else 0)
                want = Gp[:, oz:oz + bz + 2 * P, oy:oy + by + 2 * P, i0:i0 + P]
            got = out.cpu().numpy()
            assert got.size == want.size + 1 and got[-1] == 12.0 + ph
            assert np.array_equal(got[:-1], np.ascontiguousarray(want).ravel()), (ph, side)


def test_unpack_copies_and_checks_the_tag():
    from paper_2508_07193_b200 import Box, _lib, make_partition
    from paper_2508_07193_b200.schwarz import BlockLayout, HaloExchanger
    part = make_partition(Box(*GEXT), SGRID, 1)
    lay = BlockLayout(part, FakeTransport(WORLD, 0))   # rank 0: neighbours on x-hi and z-hi
    hx = HaloExchanger(lay, 1)
    blk = hx.block_struct()
    lib = _lib.lib()
    status = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    n = lib.fmp_halo_slab_doubles(_lib.ref(blk), 0)
    msg = torch.rand(n + 1, dtype=torch.float64, device="cuda")
    msg[-1] = 9.0
    _lib.call("fmp_halo_unpack", _lib.ref(blk), 0, 1, _lib.ptr(msg), 9.0, status.data_ptr(), _lib.stream())
    torch.cuda.synchronize()
    assert int(status[0]) == 0 and torch.equal(hx.ghosts[5].reshape(-1), msg[:-1])
    _lib.call("fmp_halo_unpack", _lib.ref(blk), 0, 1, _lib.ptr(msg), 10.0, status.data_ptr(), _lib.stream())
    torch.cuda.synchronize()
    assert int(status[0]) == 1 << 5   # z-hi slot


@pytest.mark.parametrize("rank", [0, 1, 2, 3])
def test_spmv_parts_equal_whole_and_single_block(rank):
    from paper_2508_07193_b200 import Box, DistributedOperator, _lib, make_partition, make_transport
    part = make_partition(Box(*GEXT), SGRID, 1)
    op = DistributedOperator(part, 0.25, FakeTransport(WORLD, rank))
    hx = op.exchanger
    assert hx.active
    G, W = global_field(2), global_field(3)
    x, w = block_of(op.layout, G), block_of(op.layout, W)
    scratch = torch.zeros(int(_lib.lib().fmp_reduce_scratch_doubles()), dtype=torch.float64, device="cuda")
    dots = torch.zeros(2, dtype=torch.float64, device="cuda")
    fill_ghosts(hx, G, 1)
    blk = hx.block_struct()
    y_all = torch.empty_like(x)
    _lib.call("fmp_stencil_apply", _lib.ref(blk), 0.25, 1, 2, _lib.ptr(x), _lib.ptr(y_all), _lib.ptr(w),
              _lib.ptr(dots), _lib.ptr(scratch), _lib.stream())
    d_all = dots.clone()
    y = torch.full_like(x, float("nan"))
    fill_ghosts(hx, G, 1, phases=())                         # ghosts NaN during the interior part
    _lib.call("fmp_stencil_apply_part", _lib.ref(blk), 0.25, 1, 2, _lib.FMP_PART_INTERIOR, _lib.ptr(x), _lib.ptr(y),
              _lib.ptr(w), _lib.ptr(dots), _lib.ptr(scratch), _lib.stream())
    torch.cuda.synchronize()
    fill_ghosts(hx, G, 1)
    _lib.call("fmp_stencil_apply_part", _lib.ref(blk), 0.25, 1, 2, _lib.FMP_PART_BOUNDARY, _lib.ptr(x), _lib.ptr(y),
              _lib.ptr(w), _lib.ptr(dots), _lib.ptr(scratch), _lib.stream())
    assert torch.equal(y, y_all)
    assert torch.equal(dots, d_all)
    # against one block covering the global box
    whole = DistributedOperator(part, 0.25, make_transport("cuda"))
    ya = whole.apply(torch.from_numpy(G).cuda())
    (ox, oy, oz), (bx, by, bz) = op.layout.origin, op.layout.block
    assert torch.equal(y_all, ya[:, oz:oz + bz, oy:oy + by, ox:ox + bx])


@pytest.mark.parametrize("rank", [0, 3])
def test_ras_parts_equal_whole_and_single_block(rank):
    from paper_2508_07193_b200 import Box, RasPreconditioner, _lib, make_partition, make_transport
    part = make_partition(Box(*GEXT), SGRID, 1)
    prec = RasPreconditioner(part, 0.25, FakeTransport(WORLD, rank))
    hx = prec.exchanger
    G = global_field(4)
    r = block_of(prec.layout, G)
    fill_ghosts(hx, G, 1)
    blk = hx.block_struct()
    z_all = torch.empty_like(r)
    prec.plan.apply(blk, _lib.FMP_SOLVE_WOODBURY, r, z_all)
    z = torch.full_like(r, float("nan"))
    fill_ghosts(hx, G, 1, phases=())
    prec.plan.apply(blk, _lib.FMP_SOLVE_WOODBURY, r, z, part=_lib.FMP_PART_INTERIOR)
    torch.cuda.synchronize()
    fill_ghosts(hx, G, 1)
    prec.plan.apply(blk, _lib.FMP_SOLVE_WOODBURY, r, z, part=_lib.FMP_PART_BOUNDARY)
    assert torch.equal(z, z_all)
    whole = RasPreconditioner(part, 0.25, make_transport("cuda"))
    za = whole.apply(torch.from_numpy(G).cuda())
    (ox, oy, oz), (bx, by, bz) = prec.layout.origin, prec.layout.block
    zb = za[:, oz:oz + bz, oy:oy + by, ox:ox + bx]
    assert (z_all - zb).abs().max() <= 1e-13 * zb.abs().max()

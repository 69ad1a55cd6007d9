"""Multi-process (world_size 2 and 4) tests of the GPU decomposition.

CPU (gloo): the three-phase ghost exchange fills every ghost slab with the global field.
GPU (gloo staging, all ranks on cuda:0): multi-block SpMV / RAS / BiCGSTAB equal the
single-block results -- the same kernels read neighbour data from the ghost shell."""

import math
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import _dist_helpers as H


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def run(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


@pytest.mark.parametrize("world,gext,sgrid,width", [(2, (16, 8, 8), (4, 2, 2), 1), (4, (16, 8, 16), (4, 2, 4), 2)])
def test_ghost_exchange_fills_global_values(world, gext, sgrid, width):
    res = run(H.halo_worker, world, gext, sgrid, width)
    for rank, bad, checked, nmsg in res:
        assert checked > 0 and bad == 0, (rank, bad, checked)
        assert nmsg > 0


@pytest.mark.gpu
@pytest.mark.parametrize("world,gext,sgrid", [(2, (32, 16, 16), (4, 2, 2)), (4, (32, 16, 32), (4, 2, 4))])
def test_multiblock_matches_single_block(world, gext, sgrid):
    from paper_2508_07193_b200 import (Box, DistributedOperator, RasPreconditioner, SolverConfig, bicgstab,
                                       make_partition, make_transport)
    res = run(H.solve_worker, world, gext, sgrid)
    part = make_partition(Box(*gext), sgrid, 1)
    tr = make_transport("cuda")
    op, prec = DistributedOperator(part, 0.25, tr), RasPreconditioner(part, 0.25, tr)
    x0 = np.random.default_rng(42).uniform(-1.0, 1.0, 3 * int(np.prod(gext)))
    b = op.apply(torch.from_numpy(x0).cuda().view(part.global_box.shape4))
    z = prec.apply(b)
    x, rep = bicgstab(op, prec, b, SolverConfig())
    B, Z, X = (t.cpu().numpy() for t in (b, z, x))
    for rank, (ox, oy, oz), bb, zz, xx, trace, iters in res:
        sl = (slice(None), slice(oz, oz + bb.shape[1]), slice(oy, oy + bb.shape[2]), slice(ox, ox + bb.shape[3]))
        assert np.array_equal(bb, B[sl])                       # stencil with ghosts: bitwise
        assert np.abs(zz - Z[sl]).max() <= 1e-13 * np.abs(Z).max()
        assert iters == rep.iterations
        assert np.abs(np.array(trace) - np.array([t[1] for t in rep.trace])).max() <= 1e-12
        assert np.abs(xx - X[sl]).max() <= 1e-11 * np.abs(X).max()


@pytest.mark.parametrize("world,gext,sgrid,ov", [(2, (8, 8, 8), (2, 1, 1), 1), (2, (8, 8, 8), (2, 2, 2), 1),
                                                 (4, (16, 8, 16), (4, 2, 4), 1)])
def test_subdomain_trace_matches_reference_multiblock(world, gext, sgrid, ov):
    """Across GPU blocks, the union of every block's subdomain message rows equals the reference
    Exchanger's trace (ref:schwarz.py:186-188, 234-235; golden from the reference itself)."""
    from conftest import GOLDEN
    g = np.load(GOLDEN / "schwarz.npz")
    tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, sgrid)) + f"_o{ov}"
    res = run(H.trace_worker, world, gext, sgrid, ov)
    rows = sorted(tuple(r) for _, t in res for r in t)
    want = sorted(tuple(int(v) for v in r) for r in g[f"trace_{tag}"])
    assert rows == want


def test_lost_halo_message_raises_host_path():
    res = run(H.drop_worker, 2, (8, 8, 8), (2, 1, 1), "cpu")
    # rank 1 misses rank 0's x-phase slab (rank 0 still receives rank 1's)
    assert [r[2] for r in res] == [False, True]


@pytest.mark.gpu
def test_lost_halo_message_raises_device_path():
    res = run(H.drop_worker, 2, (16, 8, 8), (2, 1, 1), "cuda:0")
    assert [r[2] for r in res] == [False, True]


@pytest.mark.gpu
def test_exchange_is_allocation_free():
    res = run(H.alloc_worker, 2, (32, 16, 16), (4, 2, 2))
    for rank, before, after in res:
        assert after == before, (rank, before, after)

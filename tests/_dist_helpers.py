"""Worker bodies for the multi-process tests (spawned with torch.multiprocessing)."""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "oracle", ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"], os.environ["WORLD_SIZE"] = str(rank), str(world)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def halo_worker(rank, world, port, gext, sgrid, width, out):
    """Fill the ghost shell of this rank's block and compare every slab with the global field."""
    import numpy as np
    import torch
    init(rank, world, port)
    from paper_2508_07193_b200 import Box, make_partition
    from paper_2508_07193_b200.schwarz import BlockLayout, DistTransport, HaloExchanger
    tr = DistTransport(device="cpu")
    part = make_partition(Box(*gext), sgrid, 1)
    lay = BlockLayout(part, tr)
    glob = torch.arange(3 * int(np.prod(gext)), dtype=torch.float64).view(3, gext[2], gext[1], gext[0])
    (x0, y0, z0), (bx, by, bz) = lay.origin, lay.block
    x = glob[:, z0:z0 + bz, y0:y0 + by, x0:x0 + bx].contiguous()
    hx = HaloExchanger(lay, width, record_trace=True)
    hx.exchange(x)
    P = width
    nx, ny, nz = gext
    bad = 0
    checked = 0

    def expect(c, k, j, i):
        gi, gj, gk = x0 + i, y0 + j, z0 + k
        if not (0 <= gi < nx and 0 <= gj < ny and 0 <= gk < nz):
            return None
        return float(glob[c, gk, gj, gi])

    names = ["xlo", "xhi", "ylo", "yhi", "zlo", "zhi"]
    for q, gbuf in enumerate(hx.ghosts):
        if gbuf is None:
            continue
        for c in range(3):
            for kk in range(gbuf.shape[1]):
                for jj in range(gbuf.shape[2]):
                    for ii in range(gbuf.shape[3]):
                        if q < 2:
                            k, j, i = kk - P, jj - P, (ii - P if q == 0 else bx + ii)
                        elif q < 4:
                            k, j, i = kk - P, (jj - P if q == 2 else by + jj), ii
                        else:
                            k, j, i = (kk - P if q == 4 else bz + kk), jj, ii
                        want = expect(c, k, j, i)
                        if want is None:
                            continue
                        checked += 1
                        if float(gbuf[c, kk, jj, ii]) != want:
                            bad += 1
    out.put((rank, bad, checked, len(hx.trace)))
    import torch.distributed as dist
    dist.barrier()
    dist.destroy_process_group()


def solve_worker(rank, world, port, gext, sgrid, out):
    """Multi-block BiCGSTAB + RAS on one GPU shared by `world` gloo processes."""
    import numpy as np
    import torch
    init(rank, world, port)
    from paper_2508_07193_b200 import (Box, DistributedOperator, RasPreconditioner, SolverConfig, bicgstab,
                                       make_partition)
    from paper_2508_07193_b200.schwarz import DistTransport
    tr = DistTransport(device="cuda:0")
    part = make_partition(Box(*gext), sgrid, 1)
    op = DistributedOperator(part, 0.25, tr)
    prec = RasPreconditioner(part, 0.25, tr)
    lay = op.layout
    x0 = np.random.default_rng(42).uniform(-1.0, 1.0, 3 * int(np.prod(gext))).reshape(3, gext[2], gext[1], gext[0])
    (ox, oy, oz), (bx, by, bz) = lay.origin, lay.block
    xb = torch.from_numpy(np.ascontiguousarray(x0[:, oz:oz + bz, oy:oy + by, ox:ox + bx])).cuda()
    b = op.apply(xb)
    z = prec.apply(b)
    x, rep = bicgstab(op, prec, b, SolverConfig())
    out.put((rank, (ox, oy, oz), b.cpu().numpy(), z.cpu().numpy(), x.cpu().numpy(),
             [t[1] for t in rep.trace], rep.iterations))
    import torch.distributed as dist
    dist.barrier()
    dist.destroy_process_group()


def trace_worker(rank, world, port, gext, sgrid, ov, out):
    """The subdomain message rows this rank's block records over two exchanges."""
    import torch
    init(rank, world, port)
    from paper_2508_07193_b200 import Box, make_partition
    from paper_2508_07193_b200.schwarz import BlockLayout, DistTransport, HaloExchanger
    tr = DistTransport(device="cpu")
    part = make_partition(Box(*gext), sgrid, ov)
    lay = BlockLayout(part, tr)
    hx = HaloExchanger(lay, max(1, ov), record_trace=True)
    x = torch.zeros(lay.shape4, dtype=torch.float64)
    hx.exchange(x)
    hx.exchange(x)
    out.put((rank, list(hx.trace)))
    import torch.distributed as dist
    dist.barrier()
    dist.destroy_process_group()


def drop_worker(rank, world, port, gext, sgrid, device, out):
    """Rank 0 drops its z-phase message toward the high side (and rank 1 its matching receive) in
    the second exchange: rank 1's ghost keeps the first epoch's tag, which must raise
    CommunicationError (host path: at once; device path: at check())."""
    import torch
    init(rank, world, port)
    from paper_2508_07193_b200 import Box, CommunicationError, make_partition
    from paper_2508_07193_b200.schwarz import BlockLayout, DistTransport, HaloExchanger
    tr = DistTransport(device=device)
    part = make_partition(Box(*gext), sgrid, 1)
    lay = BlockLayout(part, tr)
    hx = HaloExchanger(lay, 1)
    x = torch.ones(lay.shape4, dtype=torch.float64, device=device)
    hx.exchange(x)
    if device != "cpu":
        torch.cuda.synchronize()
        hx.check()
    ok_first = True
    hx.drop_phase = (2, 1)   # x phase (the GPU grid is (2,1,1)): rank 0 -> its high side
    raised = False
    try:
        hx.exchange(x)
        if device != "cpu":
            torch.cuda.synchronize()
            hx.check()
    except CommunicationError:
        raised = True
    out.put((rank, ok_first, raised))
    import torch.distributed as dist
    dist.barrier()
    dist.destroy_process_group()


def alloc_worker(rank, world, port, gext, sgrid, out):
    """Device allocator growth over repeated exchanges and split SpMV / RAS applies (gloo staging,
    all ranks on cuda:0): the exchange path allocates nothing after the first call."""
    import torch
    init(rank, world, port)
    from paper_2508_07193_b200 import Box, DistributedOperator, RasPreconditioner, make_partition
    from paper_2508_07193_b200.schwarz import DistTransport
    tr = DistTransport(device="cuda:0")
    part = make_partition(Box(*gext), sgrid, 1)
    op = DistributedOperator(part, 0.25, tr)
    prec = RasPreconditioner(part, 0.25, tr)
    x = torch.rand(op.layout.shape4, dtype=torch.float64, device="cuda:0")
    y, z = torch.empty_like(x), torch.empty_like(x)
    op.apply_into(x, y)
    prec.apply_into(x, z)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    for _ in range(5):
        op.exchanger.exchange(x)
        op.apply_into(x, y)
        prec.apply_into(x, z)
    torch.cuda.synchronize()
    after = torch.cuda.memory_allocated()
    out.put((rank, before, after))
    import torch.distributed as dist
    dist.barrier()
    dist.destroy_process_group()

"""CPU tests of the host-side logic: geometry, layouts, config validation, file formats,
and the C-ABI library's exported symbols (no compute calls without a GPU)."""

import ctypes
import re

import numpy as np
import pytest

import flashmp_oracle as O
from conftest import GOLDEN, ROOT


def test_library_exports_every_header_symbol():
    from paper_2508_07193_b200 import _lib
    header = (ROOT / "include" / "flashmp_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int64_t)\s+(fmp_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    if not _lib.LIB_PATH.exists():
        pytest.skip("libflashmp_b200.so not built")
    handle = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared:
        assert hasattr(handle, name), name
    assert handle.fmp_abi_version() == _lib.ABI_VERSION
    assert handle.fmp_reduce_scratch_doubles() >= 8 * 148


def test_correction_rows_match_reference():
    from paper_2508_07193_b200 import Box
    from paper_2508_07193_b200.subdomain import correction_rows, correction_size
    g = np.load(GOLDEN / "subdomain.npz")
    for ext in ((4, 5, 6), (3, 3, 3), (1, 1, 1)):
        rows, vals, per = correction_rows(Box(*ext))
        tag = "_".join(map(str, ext)) + "_a0.25"
        assert np.array_equal(rows, g[f"rows_{tag}"])
        assert np.array_equal(vals, g[f"values_{tag}"])
        assert sum(per) == correction_size(Box(*ext)) == O.correction_size(ext)


def test_cost_model_matches_reference_formulas():
    from paper_2508_07193_b200 import Box, analytic_cost, correction_size
    for n in (1, 2, 8, 32):
        c = analytic_cost(Box(n, n, n), correction_size(Box(n, n, n)))
        assert c.flops_per_exact_solve == 36 * n ** 4 + 18 * n ** 3
        assert c.flops_total == 144 * n ** 4 + 18 * n ** 3
    assert analytic_cost(Box(32, 32, 32), 6048).flops_total == 151_584_768
    c34 = analytic_cost(Box(34, 34, 34), correction_size(Box(34, 34, 34)))
    assert c34.flops_per_solve == 191_038_248


@pytest.mark.parametrize("gext,grid,ov", [((8, 8, 8), (2, 1, 1), 0), ((8, 8, 8), (2, 1, 1), 1),
                                          ((8, 8, 4), (2, 2, 1), 1), ((12, 8, 8), (3, 2, 2), 2),
                                          ((8, 4, 6), (2, 2, 3), 1)])
def test_partition_geometry_matches_reference(gext, grid, ov):
    from paper_2508_07193_b200 import Box, make_partition
    g = np.load(GOLDEN / "schwarz.npz")
    tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_o{ov}"
    part = make_partition(Box(*gext), grid, ov)
    geom = np.array([[*r.owned_lo, *r.owned.extents, *r.ext_lo, *r.ext.extents] for r in part.ranks])
    assert np.array_equal(geom, g[f"geom_{tag}"])
    for r, o in zip(part.ranks, O.partition(gext, grid, ov)):
        assert r.neighbors == o.neighbors and r.coords == o.coords


def test_partition_validation_and_scatter_gather():
    from paper_2508_07193_b200 import Box, gather_field, make_partition, scatter_field
    with pytest.raises(ValueError, match="divisible"):
        make_partition(Box(10, 8, 8), (3, 1, 1), 1)
    with pytest.raises(ValueError, match="overlap"):
        make_partition(Box(8, 8, 8), (4, 1, 1), 3)
    with pytest.raises(ValueError):
        make_partition(Box(8, 8, 8), (2, 2, 2), -1)
    part = make_partition(Box(6, 4, 2), (3, 2, 1), 0)
    full = np.random.default_rng(0).uniform(-1, 1, part.global_box.dof)
    assert np.array_equal(gather_field(part, scatter_field(part, full)), full)
    ranks = O.partition((6, 4, 2), (3, 2, 1), 0)
    for a, b in zip(scatter_field(part, full), O.scatter((6, 4, 2), ranks, full)):
        assert np.array_equal(a, b)


def test_proc_grid_and_block_layouts():
    from paper_2508_07193_b200 import Box, make_partition, proc_grid_for
    from paper_2508_07193_b200.schwarz import BlockLayout

    class FakeTransport:
        def __init__(self, world, rank):
            self.world, self.rank, self.device = world, rank, "cpu"

    assert [proc_grid_for(n) for n in (1, 2, 4, 8)] == [(1, 1, 1), (2, 1, 1), (2, 1, 2), (2, 2, 2)]
    assert [proc_grid_for(n) for n in (1, 2, 4, 8, 12)] == [O.proc_grid_for(n) for n in (1, 2, 4, 8, 12)]
    part = make_partition(Box(64, 32, 64), (4, 2, 4), 1)
    seen = []
    for rank in range(4):
        lay = BlockLayout(part, FakeTransport(4, rank))
        assert lay.block == (32, 32, 32)
        seen += [r.rank for r in lay.local_ranks]
        for s, r in zip(lay.sub_specs(), lay.local_ranks):
            assert all(-1 <= lo <= b for lo, b in zip(s.ext_lo, lay.block))
            assert tuple(o + e for o, e in zip(s.own_off, r.ext_lo)) == r.owned_lo
    assert sorted(seen) == list(range(part.nranks))
    with pytest.raises(ValueError):
        BlockLayout(make_partition(Box(8, 8, 8), (1, 1, 1), 1), FakeTransport(2, 0))


def test_solver_config_and_reduce_dot():
    from paper_2508_07193_b200 import SolverConfig, reduce_dot
    for bad in (dict(method="cg"), dict(tol=0.0), dict(restart=0), dict(preconditioner="ilu")):
        with pytest.raises(ValueError):
            SolverConfig(**bad)
    assert reduce_dot([1e16, 1.0, -1e16]) == 0.0        # ref:tests/test_krylov.py:24-30


def test_fmpf_round_trip_and_permutation(tmp_path):
    from paper_2508_07193_b200 import Box, FieldVector, dump_field, load_field
    from paper_2508_07193_b200.grid import permute_to_component_major, permute_to_grid_major
    box = Box(3, 4, 5)
    v = FieldVector(box, np.random.default_rng(1).uniform(-1, 1, box.dof))
    dump_field(v, tmp_path / "f.field")
    raw = (tmp_path / "f.field").read_bytes()
    assert raw[:4] == b"FMPF" and len(raw) == 20 + 8 * box.dof
    w = load_field(tmp_path / "f.field")
    assert w.box == box and np.array_equal(w.data, v.data)
    gm = permute_to_grid_major(v)
    assert gm.points()[7, 2] == v.component(2).ravel()[7]
    assert np.array_equal(permute_to_component_major(gm).data, v.data)
    (tmp_path / "bad.field").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError):
        load_field(tmp_path / "bad.field")


def test_svd_factors_bit_identical_to_reference():
    from paper_2508_07193_b200 import svd_of_difference
    g = np.load(GOLDEN / "svd.npz")
    for n in (1, 2, 3, 4, 5, 8, 16, 17, 18, 32, 33, 34):
        s = svd_of_difference(n)
        assert np.array_equal(s.U, g[f"U_{n}"]) and np.array_equal(s.S, g[f"S_{n}"])
        assert np.array_equal(s.Vt, g[f"Vt_{n}"])


@pytest.mark.parametrize("rep", [(3, 4, 5), (2, 2, 3), (4, 4, 3)])
def test_rotation_groups_share_cinv(rep):
    """Cyclic axis rotations of a box have the same C^-1 up to the plan's row map
    (plan.rotation_rowmap): C^-1_member[i, j] == C^-1_rep[map[i], map[j]] (oracle, CPU)."""
    from paper_2508_07193_b200.plan import correction_points, rotate, rotation_groups, rotation_rowmap
    e1 = rotate(rep)
    e2 = rotate(e1)
    groups = rotation_groups([rep, (7, 7, 7), e1, e2])
    assert groups == [(0, 0), (1, 0), (0, 1), (0, 2)]
    assert correction_points(rep).shape == (O.correction_size(rep), 4)
    base = O.precompute(rep, 0.25).Cinv
    for t, e in ((1, e1), (2, e2)):
        rm = rotation_rowmap(rep, t)
        assert sorted(rm.tolist()) == list(range(rm.size))
        got = O.precompute(e, 0.25).Cinv
        assert np.abs(got - base[np.ix_(rm, rm)]).max() <= 1e-13 * np.abs(base).max()


@pytest.mark.parametrize("tag", ["8_8_8_g211_o0", "8_8_8_g211_o1", "8_8_4_g221_o1", "12_8_8_g322_o2", "8_4_6_g223_o1",
                                 "8_8_8_g222_o1"])
def test_subdomain_trace_matches_reference(tag):
    """One block: the exchanger's message rows equal the reference Exchanger's trace row for row
    (same order: ranks ascending, neighbours in (dz, dy, dx) order; ref:schwarz.py:203-235)."""
    import torch
    from paper_2508_07193_b200 import Box, make_partition
    from paper_2508_07193_b200.schwarz import BlockLayout, DeviceTransport, HaloExchanger
    g = np.load(GOLDEN / "schwarz.npz")
    gs, grid, ov = tag.split("_g")[0], tag.split("_g")[1].split("_o")[0], int(tag.split("_o")[1])
    part = make_partition(Box(*map(int, gs.split("_"))), tuple(int(c) for c in grid), ov)
    lay = BlockLayout(part, DeviceTransport("cpu"))
    hx = HaloExchanger(lay, max(1, ov), record_trace=True)
    x = torch.zeros(lay.shape4, dtype=torch.float64)
    hx.exchange(x)
    hx.exchange(x)
    assert np.array_equal(np.array(hx.trace, dtype=np.int64).reshape(-1, 4), g[f"trace_{tag}"])

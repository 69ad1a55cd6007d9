"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]

The reference is imported read-only from /root/reference/pkg/src; nothing is
copied.  Outputs are small .npz files next to this script.  `--big` also runs
BASELINE configs 1 and 2 (32^3 single subdomain CN step; 64^3 2x2x2 of 32^3),
which take a few minutes because of the reference's CPU precompute.  `--huge`
runs the benchmarked configuration itself (256^3, 8x8x8 subdomains of 32^3:
RAS apply, BiCGSTAB solve and one CN step), a 96^3 3x3x3 partition whose
extended boxes include every rotated (34,33,33)-type shape, and the 16^3-subdomain
config-5 case (64^3, 4x4x4), about 25 minutes on 8 cores; outputs are sampled.

The GPU box has no /root/reference: tests there only read these fixtures.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from flashmp import grid as rgrid  # noqa: E402
from flashmp import operators as rops  # noqa: E402
from flashmp import transform as rtr  # noqa: E402
from flashmp import subdomain as rsd  # noqa: E402
from flashmp import schwarz as rsw  # noqa: E402
from flashmp import krylov as rkr  # noqa: E402
from flashmp import cn_driver as rcn  # noqa: E402

SAMPLE = 4096


def rng_field(box, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, box.dof)


def gen_svd():
    out = {}
    for n in (1, 2, 3, 4, 5, 8, 16, 17, 18, 32, 33, 34):
        s = rtr.svd_of_difference(n)
        out[f"U_{n}"], out[f"S_{n}"], out[f"Vt_{n}"] = s.U, s.S, s.Vt
    np.savez_compressed(OUT / "svd.npz", **out)


def gen_operators():
    out = {}
    for ext in ((3, 3, 3), (4, 5, 6), (1, 3, 4), (8, 8, 8), (2, 7, 3)):
        box = rgrid.Box(*ext)
        x = rng_field(box, 11)
        E = rgrid.FieldVector(box, x)
        tag = "_".join(map(str, ext))
        p = rops.OperatorParams(box, 0.25)
        out[f"x_{tag}"] = x
        out[f"A_{tag}"] = rops.apply_operator(p, True, E).data
        out[f"A0_{tag}"] = rops.apply_operator(p, False, E).data
        out[f"Acsr_{tag}"] = rops.assemble_sparse(p, True).matrix @ x
        out[f"curlf_{tag}"] = rops.apply_curl("forward", E).data
        out[f"curlb_{tag}"] = rops.apply_curl("backward", E).data
        out[f"M_{tag}"] = rops.apply_double_curl(E).data
        ts = rtr.TransformSet.for_box(box)
        out[f"G_{tag}"] = rtr.apply_transform(ts, E).data
        out[f"Ginv_{tag}"] = rtr.apply_inverse_transform(ts, E).data
    np.savez_compressed(OUT / "operators.npz", **out)


def gen_subdomain():
    out = {}
    for ext in ((1, 1, 1), (2, 2, 2), (3, 3, 3), (4, 5, 6), (6, 2, 4), (1, 3, 4), (5, 1, 2)):
        for alpha in (0.05, 0.25, 1.0):
            box = rgrid.Box(*ext)
            data = rsd.precompute(rops.OperatorParams(box, alpha))
            tag = "_".join(map(str, ext)) + f"_a{alpha}"
            r = rgrid.FieldVector(box, rng_field(box, 7))
            out[f"r_{tag}"] = r.data
            out[f"exact_{tag}"] = rsd.exact_solve(data, r).data
            out[f"solve_{tag}"] = rsd.solve(data, r).data
            if ext in ((4, 5, 6), (3, 3, 3), (1, 1, 1)) and alpha == 0.25:
                out[f"rows_{tag}"] = data.corr.rows
                out[f"values_{tag}"] = data.corr.values
                out[f"Cinv_{tag}"] = data.corr.inverse
    np.savez_compressed(OUT / "subdomain.npz", **out)


def gen_schwarz():
    out = {}
    cases = [((8, 8, 8), (2, 1, 1), 0), ((8, 8, 8), (2, 1, 1), 1), ((8, 8, 4), (2, 2, 1), 1),
             ((12, 8, 8), (3, 2, 2), 2), ((8, 4, 6), (2, 2, 3), 1)]
    for gext, grid, ov in cases:
        gbox = rgrid.Box(*gext)
        part = rsw.make_partition(gbox, grid, ov)
        tr = rsw.SerialTransport()
        tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_o{ov}"
        r = rng_field(gbox, 3)
        prec = rsw.RasPreconditioner(part, 0.25, tr)
        out[f"r_{tag}"] = r
        out[f"ras_{tag}"] = rsw.gather_field(part, prec.apply(rsw.scatter_field(part, r)))
        op = rsw.DistributedOperator(part, 0.25, tr)
        out[f"spmv_{tag}"] = rsw.gather_field(part, op.apply(rsw.scatter_field(part, r)))
        # index maps: the extended vectors the exchanger builds from a linear-index field
        ex = rsw.Exchanger(part, tr)
        lin = np.arange(gbox.dof, dtype=np.float64)
        exts = ex.exchange(rsw.scatter_field(part, lin))
        out[f"extidx_{tag}"] = np.concatenate(exts).astype(np.int64)
        out[f"geom_{tag}"] = np.array([[*i.owned_lo, *i.owned.extents, *i.ext_lo, *i.ext.extents]
                                       for i in part.ranks], dtype=np.int64)
        # the reference's comm trace: one (epoch, src, dst, bytes) row per message (two exchanges)
        ex = rsw.Exchanger(part, tr, record_trace=True)
        ex.exchange(rsw.scatter_field(part, lin))
        ex.exchange(rsw.scatter_field(part, lin))
        out[f"trace_{tag}"] = np.array(ex.trace, dtype=np.int64).reshape(-1, 4)
    for gext, grid, ov in [((8, 8, 8), (2, 2, 2), 1), ((16, 8, 16), (4, 2, 4), 1)]:   # multi-GPU trace cases
        part = rsw.make_partition(rgrid.Box(*gext), grid, ov)
        tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_o{ov}"
        ex = rsw.Exchanger(part, rsw.SerialTransport(), record_trace=True)
        lin = np.arange(rgrid.Box(*gext).dof, dtype=np.float64)
        ex.exchange(rsw.scatter_field(part, lin))
        ex.exchange(rsw.scatter_field(part, lin))
        out[f"trace_{tag}"] = np.array(ex.trace, dtype=np.int64).reshape(-1, 4)
    np.savez_compressed(OUT / "schwarz.npz", **out)


def _solve_case(gext, grid, ov, alpha, method, prec_on, seed=42, restart=30):
    gbox = rgrid.Box(*gext)
    part = rsw.make_partition(gbox, grid, ov)
    tr = rsw.SerialTransport()
    op = rsw.DistributedOperator(part, alpha, tr)
    prec = rsw.RasPreconditioner(part, alpha, tr) if prec_on else None
    x0 = np.random.default_rng(seed).uniform(-1.0, 1.0, gbox.dof)   # ref:cli.py:98-102
    b = op.apply(rsw.scatter_field(part, x0))
    cfg = rkr.SolverConfig(method=method, restart=restart,
                           preconditioner="ras" if prec_on else "none")
    runner = rkr.bicgstab if method == "bicgstab" else rkr.gmres
    t0 = time.perf_counter()
    x, rep = runner(op, prec, b, cfg)
    sec = time.perf_counter() - t0
    return rsw.gather_field(part, b), rsw.gather_field(part, x), rep, sec


def gen_krylov(big: bool):
    out = {}
    cases = [((16, 16, 16), (2, 2, 2), 1, 0.25, "bicgstab", True),
             ((16, 16, 16), (2, 2, 2), 1, 0.25, "gmres", True),
             ((16, 16, 16), (2, 2, 2), 1, 0.25, "bicgstab", False),
             ((16, 16, 16), (2, 2, 2), 1, 0.25, "gmres", False),
             ((16, 16, 16), (2, 2, 2), 2, 0.25, "bicgstab", True),
             ((12, 12, 8), (3, 2, 1), 1, 1.0, "bicgstab", True),
             ((12, 12, 8), (3, 2, 1), 1, 1.0, "gmres", True),
             ((8, 8, 8), (1, 1, 1), 1, 0.25, "bicgstab", True)]
    if big:
        cases.append(((64, 64, 64), (2, 2, 2), 1, 0.25, "bicgstab", True))
        cases.append(((64, 64, 64), (2, 2, 2), 1, 0.25, "gmres", True))
    for gext, grid, ov, alpha, method, prec_on in cases:
        tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_o{ov}_a{alpha}_{method}_" + (
            "ras" if prec_on else "none")
        b, x, rep, sec = _solve_case(gext, grid, ov, alpha, method, prec_on)
        out[f"relres_{tag}"] = np.array([t[1] for t in rep.trace])
        out[f"meta_{tag}"] = np.array([rep.iterations, int(rep.converged)])
        out[f"seconds_{tag}"] = np.array([sec])
        if b.size <= 3 * 16 ** 3:
            out[f"x_{tag}"] = x
        else:
            idx = np.random.default_rng(0).choice(b.size, SAMPLE, replace=False)
            out[f"xidx_{tag}"] = idx
            out[f"xs_{tag}"] = x[idx]
            out[f"xnorm_{tag}"] = np.array([np.linalg.norm(x)])
        print(f"{tag}: it={rep.iterations} conv={rep.converged} {sec:.2f}s", flush=True)
    np.savez_compressed(OUT / ("krylov_big.npz" if big else "krylov.npz"), **out)


def gen_cn(big: bool):
    out = {}
    cases = [((8, 8, 8), (1, 1, 1), 1), ((16, 16, 16), (2, 2, 2), 1)]
    if big:
        cases = [((32, 32, 32), (1, 1, 1), 1)]
    for gext, grid, ov in cases:
        gbox = rgrid.Box(*gext)
        rng = np.random.default_rng(42)                       # ref:cli.py:143-149
        alpha = 0.25
        dt = 2.0 * np.sqrt(alpha)
        E = rgrid.FieldVector(gbox, rng.uniform(-1.0, 1.0, gbox.dof))
        H = rgrid.FieldVector(gbox, rng.uniform(-1.0, 1.0, gbox.dof))
        state = rcn.EmState(E, H, 0, dt)
        solver = rcn.CnSolver(gbox, grid, ov, alpha, rkr.SolverConfig(), rsw.SerialTransport())
        tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_o{ov}"
        rhs = rcn.build_rhs(state)
        new, rep = rcn.cn_step(state, solver)
        out[f"relres_{tag}"] = np.array([t[1] for t in rep.trace])
        out[f"iters_{tag}"] = np.array([rep.iterations])
        if gbox.dof <= 3 * 16 ** 3:
            out[f"rhs_{tag}"] = rhs.data
            out[f"E1_{tag}"] = new.E.data
            out[f"H1_{tag}"] = new.H.data
        else:
            idx = np.random.default_rng(0).choice(gbox.dof, SAMPLE, replace=False)
            out[f"idx_{tag}"] = idx
            out[f"rhs_{tag}"] = rhs.data[idx]
            out[f"E1_{tag}"] = new.E.data[idx]
            out[f"H1_{tag}"] = new.H.data[idx]
            out[f"norms_{tag}"] = np.array([np.linalg.norm(new.E.data), np.linalg.norm(new.H.data)])
        print(f"cn {tag}: it={rep.iterations}", flush=True)
    np.savez_compressed(OUT / ("cn_big.npz" if big else "cn.npz"), **out)


def gen_reports():
    """Reference CSV outputs (cli.py writers) for the harness-schema parity tests: the writers on
    a fixed synthetic report, the cost table, and two small real runs (solve + CN)."""
    import shutil
    import tempfile
    from flashmp import cli as rcli
    d = OUT / "reports"
    if d.exists():
        shutil.rmtree(d)
    d.mkdir()
    rep = rkr.SolveReport(method="bicgstab", iterations=3, converged=True, final_relres=5.846e-13,
                          trace=[(0, 1.0, 0.0), (1, 3.277e-05, 0.0125), (2, 2.933e-09, 0.025),
                                 (3, 5.846e-13, 0.0375)],
                          breakdown={"fast_solve": 1.25, "spmv": 0.5, "axpy_dot": 0.125}, seconds=1.875)
    rcli.write_trace_csv(d / "trace.csv", rep)
    rcli.write_trace_csv(d / "trace_zero.csv", rep, zero_times=True)
    rcli.write_breakdown_csv(d / "breakdown.csv", rep)
    cfg = rcli.ExperimentConfig(sub=(32, 32, 32), grid=(2, 2, 2), transport="cuda")
    rcli.write_summary_csv(d / "summary.csv", [rcli.RunSummary(cfg, rep, 2.5, 0.75),
                                               rcli.RunSummary(cfg, rep, 2.5, None)])
    for n in (16, 32):
        c = rcli.ExperimentConfig(sub=(n, n, n), out=str(d), mode="costs")
        rcli.run_costs(c)
        (d / "costs.csv").rename(d / f"costs_{n}.csv")
    with tempfile.TemporaryDirectory() as tmp:
        c = rcli.ExperimentConfig(sub=(4, 4, 4), grid=(2, 1, 1), out=tmp, zero_times=True)
        rcli.run_solve(c)
        shutil.copy(Path(tmp) / "trace.csv", d / "run_trace.csv")
        c = rcli.ExperimentConfig(mode="cn", sub=(4, 4, 4), grid=(2, 1, 1), steps=2, out=tmp)
        rcli.run_cn(c)
        shutil.copy(Path(tmp) / "cn_steps.csv", d / "run_cn_steps.csv")


def gen_huge():
    """Reference runs at the benchmarked sizes (ref cli.py:98-136 solve mode, cli.py:139-182 CN).

    Everything is sampled (SAMPLE indices from default_rng(0)) plus the 2-norm and the
    per-(component, z-plane) sums of each field, so the fixture stays small while the GPU test
    still sees every subdomain's contribution."""
    out = {}

    def put(tag, vec, box):
        idx = np.random.default_rng(0).choice(vec.size, SAMPLE, replace=False)
        out[f"idx_{tag}"] = idx
        out[f"s_{tag}"] = vec[idx]
        out[f"norm_{tag}"] = np.array([np.linalg.norm(vec)])
        out[f"zsum_{tag}"] = vec.reshape(3, box.nz, box.ny * box.nx).sum(axis=2)

    alpha = 0.25
    cases = [((96, 96, 96), (3, 3, 3), "bicgstab", True),
             ((64, 64, 64), (4, 4, 4), "bicgstab", False),
             ((64, 64, 64), (4, 4, 4), "gmres", False),
             ((256, 256, 256), (8, 8, 8), "bicgstab", True)]
    for gext, grid, method, full in cases:
        gbox = rgrid.Box(*gext)
        tag = "_".join(map(str, gext)) + "_g" + "".join(map(str, grid)) + f"_{method}"
        part = rsw.make_partition(gbox, grid, 1)
        tr = rsw.SerialTransport()
        t0 = time.perf_counter()
        op = rsw.DistributedOperator(part, alpha, tr)
        prec = rsw.RasPreconditioner(part, alpha, tr)
        if full:
            r = rng_field(gbox, 3)
            ras = rsw.gather_field(part, prec.apply(rsw.scatter_field(part, r)))
            put(f"ras_{tag}", ras, gbox)
            del ras, r
        print(f"{tag}: setup+ras {time.perf_counter() - t0:.1f}s", flush=True)
        x0 = np.random.default_rng(42).uniform(-1.0, 1.0, gbox.dof)   # ref:cli.py:98-102
        b = op.apply(rsw.scatter_field(part, x0))
        del x0
        cfg = rkr.SolverConfig(method=method)
        runner = rkr.bicgstab if method == "bicgstab" else rkr.gmres
        t0 = time.perf_counter()
        x, rep = runner(op, prec, b, cfg)
        sec = time.perf_counter() - t0
        out[f"relres_{tag}"] = np.array([t[1] for t in rep.trace])
        out[f"meta_{tag}"] = np.array([rep.iterations, int(rep.converged)])
        out[f"seconds_{tag}"] = np.array([sec])
        put(f"x_{tag}", rsw.gather_field(part, x), gbox)
        print(f"{tag}: it={rep.iterations} conv={rep.converged} {sec:.1f}s "
              f"trace={[f'{t[1]:.3e}' for t in rep.trace]}", flush=True)
        del x, b
        if full and gext[0] == 256:
            rng = np.random.default_rng(42)                       # ref:cli.py:143-149
            E = rgrid.FieldVector(gbox, rng.uniform(-1.0, 1.0, gbox.dof))
            H = rgrid.FieldVector(gbox, rng.uniform(-1.0, 1.0, gbox.dof))
            state = rcn.EmState(E, H, 0, 2.0 * np.sqrt(alpha))
            solver = rcn.CnSolver(gbox, grid, 1, alpha, rkr.SolverConfig(), tr)
            t0 = time.perf_counter()
            new, rep = rcn.cn_step(state, solver)
            sec = time.perf_counter() - t0
            ctag = f"cn_{tag}"
            out[f"relres_{ctag}"] = np.array([t[1] for t in rep.trace])
            out[f"meta_{ctag}"] = np.array([rep.iterations, int(rep.converged)])
            out[f"seconds_{ctag}"] = np.array([sec])
            put(f"E1_{ctag}", new.E.data, gbox)
            put(f"H1_{ctag}", new.H.data, gbox)
            print(f"{ctag}: it={rep.iterations} {sec:.1f}s", flush=True)
        np.savez_compressed(OUT / "huge.npz", **out)


if __name__ == "__main__":
    if "--schwarz" in sys.argv:
        gen_schwarz()
        sys.exit(0)
    if "--huge" in sys.argv:
        gen_huge()
        sys.exit(0)
    big = "--big" in sys.argv
    if not big:
        gen_svd()
        gen_operators()
        gen_subdomain()
        gen_schwarz()
    gen_krylov(big)
    gen_cn(big)
    if not big:
        gen_reports()

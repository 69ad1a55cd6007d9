"""Experiment records and CSV outputs with the reference harness's schemas.

The reference CLI (`cli.py`) writes trace.csv / breakdown.csv / summary.csv / sweep.csv /
cn_steps.csv / costs.csv; the files produced here have the same columns, row order and number
formatting (`repr` floats), so a GPU run can be diffed file-for-file against a CPU run of the
reference. Only the output side is mirrored -- argument parsing and the command line itself stay
out of scope.

`run_solve` / `run_cn` drive the GPU path (this package's DistributedOperator,
RasPreconditioner, bicgstab/gmres, DeviceCnStepper) with the reference's synthetic inputs.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, replace
from pathlib import Path

import numpy as np

from .grid import Box, FieldVector
from .instrument import BREAKDOWN_CATEGORIES, PhaseTimer
from .krylov import SolveReport, SolverConfig, bicgstab, gmres
from .subdomain import (analytic_cost, correction_size, direct_method_flops, direct_method_inverse_bytes,
                        direct_method_vector_bytes)

MDOFS_DEFINITION = "# mdofs = 3*nx*ny*nz*px*py*pz / solve_seconds / 1e6"   # ref:cli.py:41
DEFAULT_SWEEP_RANKS = (1, 2, 4, 8)                                          # ref:cli.py:43

SUMMARY_COLUMNS = [                                                         # ref:cli.py:287-292
    "mode", "method", "preconditioner", "sub_nx", "sub_ny", "sub_nz",
    "px", "py", "pz", "overlap", "alpha", "tol", "restart", "max_iter", "seed",
    "transport", "iterations", "converged", "final_relres", "seconds", "mdofs",
    "efficiency", "failure",
]
SWEEP_COLUMNS = ["ranks", "px", "py", "pz", "global_nx", "global_ny", "global_nz",
                 "iterations", "converged", "seconds", "mdofs", "efficiency"]   # ref:cli.py:254-255
CN_COLUMNS = ["step", "iterations", "relres", "seconds", "max_abs_e", "max_abs_h"]   # ref:cli.py:176-177


@dataclass
class ExperimentConfig:
    """The reference's experiment record (ref:cli.py:46-75), minus the CLI. `sub` is the
    per-subdomain extent and `grid` the subdomain grid; `transport` names this package's
    transports ("cuda" / "nccl"); it is written to summary.csv verbatim."""

    mode: str = "solve"
    sub: tuple[int, int, int] = (16, 16, 16)
    grid: tuple[int, int, int] = (2, 2, 2)
    overlap: int = 1
    alpha: float = 0.25
    method: str = "bicgstab"
    restart: int = 30
    tol: float = 1e-12
    max_iter: int = 1000
    seed: int = 42
    steps: int = 10
    preconditioner: str = "ras"
    transport: str = "cuda"
    out: str = "out"
    zero_times: bool = False
    ranks: tuple[int, ...] = DEFAULT_SWEEP_RANKS

    @property
    def global_box(self) -> Box:
        return Box(*(s * g for s, g in zip(self.sub, self.grid)))

    def solver_config(self) -> SolverConfig:
        return SolverConfig(method=self.method, restart=self.restart, tol=self.tol,
                            max_iter=self.max_iter, preconditioner=self.preconditioner)


@dataclass
class RunSummary:
    """ref:cli.py:78-83."""

    config: ExperimentConfig
    report: SolveReport
    mdofs: float
    efficiency: float | None = None


def mdofs(global_box: Box, seconds: float) -> float:
    """ref:cli.py:86-87: global DOF / solve seconds / 1e6 (0 for a zero time)."""
    return global_box.dof / seconds / 1e6 if seconds > 0 else 0.0


def weak_scaling_efficiency(ranks, rates) -> list[float]:
    """Throughput relative to linear scaling from the first entry (ref:cli.py:90-97)."""
    base_ranks, base = ranks[0], rates[0]
    out = []
    for n, m in zip(ranks, rates):
        ideal = base * (n / base_ranks)
        out.append(m / ideal if ideal > 0 else 0.0)
    return out


def _fmt(v) -> str:
    """Floats as repr (round-trip exact), everything else str (ref:cli.py:263-266)."""
    return repr(v) if isinstance(v, float) else str(v)


def write_trace_csv(path, report: SolveReport, zero_times: bool = False) -> None:
    """iter,relres,time_ms per trace point (ref:cli.py:269-275)."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["iter", "relres", "time_ms"])
        for it, relres, elapsed in report.trace:
            w.writerow([it, _fmt(float(relres)), _fmt(0.0 if zero_times else float(elapsed) * 1e3)])


def write_breakdown_csv(path, report: SolveReport) -> None:
    """category,seconds over the seven categories (ref:cli.py:278-283)."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["category", "seconds"])
        for cat in BREAKDOWN_CATEGORIES:
            w.writerow([cat, _fmt(float(report.breakdown.get(cat, 0.0)))])


def write_summary_csv(path, summaries: list[RunSummary]) -> None:
    """The definition comment, then one row per run (ref:cli.py:295-308)."""
    with open(path, "w", newline="") as f:
        f.write(MDOFS_DEFINITION + "\n")
        w = csv.writer(f)
        w.writerow(SUMMARY_COLUMNS)
        for s in summaries:
            c, r = s.config, s.report
            w.writerow([c.mode, c.method, c.preconditioner, *c.sub, *c.grid, c.overlap,
                        _fmt(c.alpha), _fmt(c.tol), c.restart, c.max_iter, c.seed, c.transport,
                        r.iterations, int(r.converged), _fmt(float(r.final_relres)),
                        _fmt(float(r.seconds)), _fmt(float(s.mdofs)),
                        _fmt(s.efficiency) if s.efficiency is not None else "", r.failure or ""])


def write_sweep_csv(path, summaries: list[RunSummary]) -> None:
    """ref:cli.py:251-260."""
    with open(path, "w", newline="") as f:
        f.write(MDOFS_DEFINITION + "\n")
        w = csv.writer(f)
        w.writerow(SWEEP_COLUMNS)
        for s in summaries:
            g = s.config.global_box
            w.writerow([int(np.prod(s.config.grid)), *s.config.grid, g.nx, g.ny, g.nz,
                        s.report.iterations, int(s.report.converged),
                        _fmt(s.report.seconds), _fmt(s.mdofs), _fmt(s.efficiency)])


def write_cn_steps_csv(path, rows: list[dict]) -> None:
    """ref:cli.py:175-180."""
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=CN_COLUMNS)
        w.writeheader()
        for row in rows:
            w.writerow({k: _fmt(v) for k, v in row.items()})


def cost_rows(n: int) -> list[tuple[str, str, str]]:
    """Analytic cost table of a cubic n^3 subdomain against the direct method (ref:cli.py:186-204)."""
    box = Box(n, n, n)
    cost = analytic_cost(box, correction_size(box))
    return [
        ("flops_total_nominal", str(cost.flops_total), str(direct_method_flops(n))),
        ("flops_per_solve", str(cost.flops_per_solve), str(direct_method_flops(n))),
        ("flops_per_exact_solve", str(cost.flops_per_exact_solve), ""),
        ("flops_per_correction", str(cost.flops_per_correction), ""),
        ("bytes_resident", str(cost.bytes_resident), str(direct_method_inverse_bytes(n))),
        ("bytes_vectors", str(48 * box.volume), str(direct_method_vector_bytes(n))),
        ("correction_size_m", str(cost.m), ""),
    ]


def write_costs_csv(path, n: int) -> list[tuple[str, str, str]]:
    rows = cost_rows(n)
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["metric", "flashmp", "direct"])
        w.writerows(rows)
    return rows


def _proc_grid(nranks: int) -> tuple[int, int, int]:
    from .schwarz import proc_grid_for
    return proc_grid_for(nranks)


def run_solve(config: ExperimentConfig, write_outputs: bool = True) -> RunSummary:
    """Solve A x = b with b = A x0, x0 ~ U[-1,1] from default_rng(seed) over the global
    component-major DOF, x from zero (ref:cli.py:100-134), on the GPU path; writes
    trace/breakdown/summary CSVs into config.out."""
    from .schwarz import DistributedOperator, RasPreconditioner, make_partition, make_transport, scatter_field
    timer = PhaseTimer()
    part = make_partition(config.global_box, config.grid, config.overlap)
    tr = make_transport(config.transport, part.nranks)
    op = DistributedOperator(part, config.alpha, tr)
    prec = RasPreconditioner(part, config.alpha, tr, timer=timer) if config.preconditioner == "ras" else None
    x0 = np.random.default_rng(config.seed).uniform(-1.0, 1.0, config.global_box.dof)
    b = op.apply(scatter_field(part, x0))
    op.timer = timer
    runner = bicgstab if config.method == "bicgstab" else gmres
    _, report = runner(op, prec, b, config.solver_config(), timer=timer)
    summary = RunSummary(config, report, mdofs(config.global_box, report.seconds))
    if write_outputs:
        out = Path(config.out)
        out.mkdir(parents=True, exist_ok=True)
        write_trace_csv(out / "trace.csv", report, config.zero_times)
        write_breakdown_csv(out / "breakdown.csv", report)
        write_summary_csv(out / "summary.csv", [summary])
    return summary


def run_scaling_sweep(config: ExperimentConfig) -> list[RunSummary]:
    """Weak scaling over subdomain counts with a fixed subdomain (ref:cli.py:234-261): the
    reference's ranks are subdomains here, all on this process's GPU."""
    summaries = []
    for n in config.ranks:
        cfg = replace(config, grid=_proc_grid(n), mode="solve", out=str(Path(config.out) / f"ranks_{n}"))
        summaries.append(run_solve(cfg, write_outputs=True))
    eff = weak_scaling_efficiency([int(np.prod(s.config.grid)) for s in summaries], [s.mdofs for s in summaries])
    for s, e in zip(summaries, eff):
        s.efficiency = e
    out = Path(config.out)
    out.mkdir(parents=True, exist_ok=True)
    write_sweep_csv(out / "sweep.csv", summaries)
    return summaries


def run_cn(config: ExperimentConfig) -> tuple[int, list[dict]]:
    """CN time stepping with dt = 2 sqrt(alpha), E then H ~ U[-1,1] from default_rng(seed)
    (ref:cli.py:139-182); device-resident steps; writes cn_steps.csv and a final FMPF
    checkpoint. Returns (exit code, rows): 0, or 2 when a step failed to converge."""
    import torch
    from .cn_driver import CnSolver, DeviceCnStepper, EmState, StepFailure, save_checkpoint
    from .schwarz import make_transport
    out = Path(config.out)
    out.mkdir(parents=True, exist_ok=True)
    gbox = config.global_box
    rng = np.random.default_rng(config.seed)
    dt = 2.0 * np.sqrt(config.alpha)
    E0 = rng.uniform(-1.0, 1.0, gbox.dof)
    H0 = rng.uniform(-1.0, 1.0, gbox.dof)
    solver = CnSolver(gbox, config.grid, config.overlap, config.alpha, config.solver_config(),
                      make_transport(config.transport, int(np.prod(config.grid))))
    st = DeviceCnStepper(solver, torch.from_numpy(E0).cuda().view(gbox.shape4),
                         torch.from_numpy(H0).cuda().view(gbox.shape4), dt)
    rows, code = [], 0
    for _ in range(config.steps):
        try:
            report = st.step()
        except StepFailure:
            code = 2
            break
        rows.append({"step": st.t, "iterations": report.iterations, "relres": report.final_relres,
                     "seconds": report.seconds, "max_abs_e": float(st.E.abs().max()),
                     "max_abs_h": float(st.H.abs().max())})
    write_cn_steps_csv(out / "cn_steps.csv", rows)
    state = EmState(FieldVector(gbox, st.E.cpu().numpy().ravel()), FieldVector(gbox, st.H.cpu().numpy().ravel()),
                    st.t, dt)
    save_checkpoint(state, out / "checkpoint")
    return code, rows

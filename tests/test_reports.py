"""Harness output schemas: the CSV files written by
paper_2508_07193_b200.reports are byte-identical to the reference CLI's writers on the same
records (tests/golden/reports, made by tests/golden/make_golden.py from the reference itself), and
the GPU runs reproduce the reference runs' traces."""

import csv

import pytest

from conftest import GOLDEN

REP = GOLDEN / "reports"


def _report():
    from paper_2508_07193_b200 import SolveReport
    return SolveReport(method="bicgstab", iterations=3, converged=True, final_relres=5.846e-13,
                       trace=[(0, 1.0, 0.0), (1, 3.277e-05, 0.0125), (2, 2.933e-09, 0.025), (3, 5.846e-13, 0.0375)],
                       breakdown={"fast_solve": 1.25, "spmv": 0.5, "axpy_dot": 0.125}, seconds=1.875)


def test_writers_match_reference_bytes(tmp_path):
    from paper_2508_07193_b200 import reports as R
    rep = _report()
    R.write_trace_csv(tmp_path / "trace.csv", rep)
    R.write_trace_csv(tmp_path / "trace_zero.csv", rep, zero_times=True)
    R.write_breakdown_csv(tmp_path / "breakdown.csv", rep)
    cfg = R.ExperimentConfig(sub=(32, 32, 32), grid=(2, 2, 2), transport="cuda")
    R.write_summary_csv(tmp_path / "summary.csv", [R.RunSummary(cfg, rep, 2.5, 0.75), R.RunSummary(cfg, rep, 2.5)])
    for n in (16, 32):
        R.write_costs_csv(tmp_path / f"costs_{n}.csv", n)
    for name in ("trace.csv", "trace_zero.csv", "breakdown.csv", "summary.csv", "costs_16.csv", "costs_32.csv"):
        assert (tmp_path / name).read_bytes() == (REP / name).read_bytes(), name


def test_sweep_and_cn_schemas(tmp_path):
    from paper_2508_07193_b200 import reports as R
    rep = _report()
    s = [R.RunSummary(R.ExperimentConfig(sub=(4, 4, 4), grid=R._proc_grid(n)), rep, 2.0 * n) for n in (1, 2, 4, 8)]
    for x, e in zip(s, R.weak_scaling_efficiency([1, 2, 4, 8], [x.mdofs for x in s])):
        x.efficiency = e
    R.write_sweep_csv(tmp_path / "sweep.csv", s)
    lines = (tmp_path / "sweep.csv").read_text().splitlines()
    assert lines[0] == R.MDOFS_DEFINITION
    assert lines[1].split(",") == R.SWEEP_COLUMNS
    assert lines[2:] == ["1,1,1,1,4,4,4,3,1,1.875,2.0,1.0", "2,2,1,1,8,4,4,3,1,1.875,4.0,1.0",
                         "4,2,1,2,8,4,8,3,1,1.875,8.0,1.0", "8,2,2,2,8,8,8,3,1,1.875,16.0,1.0"]
    R.write_cn_steps_csv(tmp_path / "cn.csv", [{"step": 1, "iterations": 3, "relres": 1e-15, "seconds": 0.5,
                                                "max_abs_e": 1.5, "max_abs_h": 2.0}])
    ref_header = (REP / "run_cn_steps.csv").read_text().splitlines()[0]
    assert (tmp_path / "cn.csv").read_text().splitlines() == [ref_header, "1,3,1e-15,0.5,1.5,2.0"]
    assert R.mdofs(R.ExperimentConfig().global_box, 0.0) == 0.0


def _rows(path):
    with open(path) as f:
        return [r for r in csv.reader(f) if r and not r[0].startswith("#")]


@pytest.mark.gpu
def test_run_solve_trace_matches_reference_run(tmp_path):
    from paper_2508_07193_b200 import reports as R
    s = R.run_solve(R.ExperimentConfig(sub=(4, 4, 4), grid=(2, 1, 1), out=str(tmp_path), zero_times=True))
    got, want = _rows(tmp_path / "trace.csv"), _rows(REP / "run_trace.csv")
    assert got[0] == want[0] and len(got) == len(want)
    for g, w in zip(got[1:], want[1:]):
        assert g[0] == w[0] and g[2] == w[2] == "0.0"
        assert abs(float(g[1]) - float(w[1])) <= 1e-10 * max(float(w[1]), 1e-5)
    assert s.report.converged
    summ = _rows(tmp_path / "summary.csv")
    assert summ[0] == R.SUMMARY_COLUMNS and len(summ) == 2
    assert [r[0] for r in _rows(tmp_path / "breakdown.csv")[1:]] == list(R.BREAKDOWN_CATEGORIES)


@pytest.mark.gpu
def test_run_cn_matches_reference_run(tmp_path):
    from paper_2508_07193_b200 import load_field
    from paper_2508_07193_b200 import reports as R
    code, rows = R.run_cn(R.ExperimentConfig(mode="cn", sub=(4, 4, 4), grid=(2, 1, 1), steps=2, out=str(tmp_path)))
    assert code == 0
    got, want = _rows(tmp_path / "cn_steps.csv"), _rows(REP / "run_cn_steps.csv")
    assert got[0] == want[0] and len(got) == len(want)
    for g, w in zip(got[1:], want[1:]):
        assert g[:2] == w[:2]                                    # step, iterations
        assert float(g[2]) <= 1e-12
        for c in (4, 5):                                         # max |E|, max |H|
            assert abs(float(g[c]) - float(w[c])) <= 1e-10 * float(w[c])
    E = load_field(tmp_path / "checkpoint" / "E.field")
    assert abs(float(abs(E.data).max()) - float(want[-1][4])) <= 1e-10 * float(want[-1][4])

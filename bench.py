"""Benchmark: FlashMP-preconditioned BiCGSTAB CN-FDTD steps on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg4]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one Crank-Nicolson FDTD step of the double-curl system (ref:cn_driver.py:82-94):
RHS stencil, BiCGSTAB + RAS/FlashMP solve to relres <= 1e-12 (ref defaults: alpha 0.25,
overlap 1, tol 1e-12), H update.  Workload (weak scaling, BASELINE config 4): 256^3 grid
points per GPU in 32^3 subdomains (8x8x8 per GPU), GPU grid = the reference CLI's
_proc_grid_for(N).  value = 3 * global grid points / step seconds / 1e6 (MDoF/s, the
reference's definition ref:cli.py:41,84-85) over all N GPUs.

Rank 0 prints ONE JSON line.  --impl reference times the CPU reference algorithm (the
numpy oracle port, oracle/flashmp_oracle.py) on the host cores instead: real CN steps on a
bounded sample grid (CPU_SAMPLE, same subdomains and tolerances).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CN-FDTD step time-to-solve (s), MDOF/s, iters; precond apply GB/s @1/2/4/8 B200"
FP64_PEAK_FILE = ROOT / "profiles" / "r01_fp64_probe.json"

CONFIGS = {
    # name: (per-GPU block extents, subdomain extents, overlap)
    "cfg4": ((256, 256, 256), (32, 32, 32), 1),
    "cfg2": ((64, 64, 64), (32, 32, 32), 1),
    "cfg1": ((32, 32, 32), (32, 32, 32), 1),
    # BASELINE config 5 (subdomain-size sweep at 512^3 on 8 GPUs): the per-GPU 256^3 block with
    # 16^3 / 64^3 subdomains (32^3 is cfg4); --method gmres for its GMRES leg
    "cfg5_sd16": ((256, 256, 256), (16, 16, 16), 1),
    "cfg5_sd64": ((256, 256, 256), (64, 64, 64), 1),
}


def measured_peaks():
    peaks = {"hbm_gbs": None, "hbm_source": None, "fp64_tflops": None, "fp64_source": None}
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        peaks["hbm_gbs"] = json.loads(mp.read_text())["hbm_gbs"]
        peaks["hbm_source"] = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    else:
        peaks["hbm_gbs"], peaks["hbm_source"] = 6650.0, "B200_PROFILING.md fallback"
    if FP64_PEAK_FILE.exists():
        d = json.loads(FP64_PEAK_FILE.read_text())
        peaks["fp64_tflops"] = max(v for k, v in d.items() if k.startswith("dmma_"))
        peaks["fp64_source"] = "profiles/r01_fp64_probe.json (measured DMMA issue peak on this pool's B200)"
    return peaks


class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region (B200_PROFILING.md clocks
    line). NVML is polled every 5 ms from a thread (a 3-step region lasts ~75 ms, shorter than
    nvidia-smi's start-up); `nvidia-smi -lms 100` is the fallback when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.rows = []
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                         pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
        except Exception:
            self.nvml = None

    def _poll(self):
        nv = self.nvml
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                self.rows.append([sm, self.max_sm] + ["Active" if rs & b else "Not Active" for b in self.bits])
            except Exception:
                pass
            self.stop.wait(0.005)

    def __enter__(self):
        if self.nvml is not None:
            import threading
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=5)
            return
        out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
        for line in (out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6 and parts[0].isdigit():
                self.rows.append(parts)

    def summary(self):
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({n for r in rows for n, v in zip(self.NAMES, r[2:]) if str(v).lower() == "active"})
        return {"sm_mhz": statistics.median(float(r[0]) for r in rows), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


# ----------------------------------------------------------------------------------- ours
INT8_PROBE_FILE = ROOT / "profiles" / "r01_umma_i8_rate.json"
NCU_TRAFFIC_FILE = ROOT / "profiles" / "r02_v11_ncu_traffic.json"
# bench stage -> ncu kernel name(s) whose DRAM bytes (one ncu --set full capture) it covers
STAGE_KERNELS = {"plane_fwd": ["k_plane_fast<0, 5, 0>", "k_plane_fast<0, 5>"], "column_fwd": ["k_column_fast_db<0, 12, 5, 2>"],
                 "faces": ["k_faces<5, 2, 5>"], "slice_y": ["k_ozaki_slice_rows", "k_ozaki_exp", "k_ozaki_digits"], "gemm": ["k_ozaki"],
                 "corr": ["k_corr<5>"], "column_inv": ["k_column_fast_db<1, 12, 5, 2>"], "plane_inv": ["k_plane_fast<1, 5>"]}


def ncu_traffic() -> dict:
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from the committed
    ncu --set full capture of the cfg4 apply (tools/ncu_full.sh + tools/ncu_traffic.py)."""
    return json.loads(NCU_TRAFFIC_FILE.read_text()) if NCU_TRAFFIC_FILE.exists() else {}


def int8_peak_tops() -> tuple[float, str]:
    """Dense INT8 tcgen05 rate: the per-SM MAC/clk measured by tools/umma_rate.cu (M=128, N>=128)
    x 2 x 148 SMs x max SM clock; the 4.5 POPS spec figure if the probe file is absent."""
    if INT8_PROBE_FILE.exists():
        mac = max(r["mac_per_clk"] for r in json.loads(INT8_PROBE_FILE.read_text())["results"])
        return mac * 2 * 148 * 1.965e9 / 1e12, "profiles/r01_umma_i8_rate.json (measured tcgen05 kind::i8 rate)"
    return 4500.0, "B200 dense INT8 spec"


def dominant_roofline(stages: dict, peaks: dict) -> dict | None:
    """Roofline of the dominant single kernel of the step: the longest kernel of the
    preconditioner apply (the apply is ~2/3 of the step and every one of its kernels runs 8 times
    per step; since the Ozaki GEMM skips its all-zero C^-1 slice blocks that is the forward plane
    pass k_plane_fast<0>, profiles/r02_v05_launches_step_summary.txt).  Algorithmic work per launch
    as in stage_rooflines; peak = the measured DMMA / HBM / INT8 rate (MEASURED_PEAKS.json and the
    committed probes)."""
    cand = {k: v for k, v in stages.items() if "frac" in v}
    if not cand:
        return None
    k = max(cand, key=lambda q: cand[q]["ms"])
    g = cand[k]
    src = f"ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum ({NCU_TRAFFIC_FILE.relative_to(ROOT)})"
    out = {"kernel": f"{STAGE_KERNELS.get(k, [k])[0]} ({k})", "time_ms": g["ms"], "traffic": g.get("traffic_bytes"),
           "traffic_source": src}
    if "achieved_tflops" in g:
        out.update(op_type="FP64 multiply-add = 2 flops", bound="tensor", achieved=g["achieved_tflops"],
                   peak=peaks["fp64_tflops"], unit="TFLOP/s", frac=g["frac"], peak_source=peaks["fp64_source"])
    elif "achieved_gbs" in g:
        out.update(bound="hbm", achieved=g["achieved_gbs"], peak=peaks["hbm_gbs"], unit="GB/s", frac=g["frac"],
                   peak_source=peaks["hbm_source"])
    else:
        out.update(op_type="int8 multiply-add = 2 ops", bound="tensor", achieved=g["int8_tops"],
                   peak=g["peak_int8_tops"], unit="TFLOP/s", frac=g["frac"], peak_source=g["peak_source"])
    return out


def stage_rooflines(prec, x, z, specs, peaks, reps):
    """Per-kernel times of the preconditioner apply, from CUDA events recorded between its
    kernels on the launching stream (fmp_precond_profile), averaged over `reps` applies, with
    each kernel's algorithmic work and roofline ("Kernels")."""
    from paper_2508_07193_b200.plan import correction_counts
    import torch
    plan = prec.plan
    plan.profile(True)
    acc = {}
    for _ in range(reps):
        # keep the GPU busy (~1 ms spin) while the host enqueues the apply: otherwise the first
        # stage's interval (event 0 -> end of k_plane_fast<0>) also holds the host's launch latency
        torch.cuda._sleep(2_000_000)
        prec.apply_into(x, z)
        for k, v in plan.stage_ms().items():
            acc[k] = acc.get(k, 0.0) + v / reps
    plan.profile(False)
    fl = {k: 0 for k in ("plane_fwd", "column_fwd", "column_inv", "plane_inv")}
    faces_b = 0
    for sp in specs:
        nx, ny, nz = sp.ext
        wx, wy, wz = sp.own
        V = nx * ny * nz
        fl["plane_fwd"] += 6 * V * (nx + ny)                       # x, y mode products, 3 components
        fl["column_fwd"] += 6 * V * nz + 18 * V                    # z mode product + 3x3 block solve
        fl["column_inv"] += 6 * nx * ny * nz * wz                  # z inverse on the owned rows
        fl["plane_inv"] += 6 * wz * (ny * nx * wx + ny * wy * wx)  # x, y inverse on the owned tile
        faces_b += 24 * V
    gemm_f = 0
    for g, (rep, _t) in enumerate(plan.groups):
        if rep == g:
            m = sum(correction_counts(plan.shapes[g]))
            gemm_f += 2 * m * m * plan.gcols[g]
    fp64, hbm = peaks["fp64_tflops"], peaks["hbm_gbs"]
    traffic = ncu_traffic()
    out = {}
    for k, ms in acc.items():
        e = {"ms": round(ms, 4)}
        tb = [traffic[n]["traffic_bytes"] for n in STAGE_KERNELS.get(k, []) if n in traffic]
        if tb:
            e["traffic_bytes"] = sum(tb)
        if k in fl:
            a = fl[k] / ms / 1e9
            e.update(bound="tensor (FP64 DMMA)", achieved_tflops=round(a, 2), frac=round(a / fp64, 3))
        elif k == "faces":
            a = faces_b / ms / 1e6
            e.update(bound="hbm", achieved_gbs=round(a, 1), frac=round(a / hbm, 3))
        elif k == "gemm" and ms > 0:
            # executed work: the MMAs of the non-zero C^-1 slice blocks (fmp_precond_ozaki_stats);
            # the dense-equivalent rate (every slice product) is reported beside it
            a = gemm_f / ms / 1e9
            kept = plan.ozaki_stats() if plan.gemm_kind() == "ozaki" else {"kept_slices": 1.0, "kept_mma": 1.0}
            pk, src = int8_peak_tops()
            ex = 28 * a * kept["kept_mma"]
            e.update(bound="tensor (INT8 tcgen05, Ozaki S=7: 28 int8 products per FP64 product, all-zero slice blocks skipped)",
                     fp64_equiv_tflops=round(a, 2), int8_tops=round(ex, 1), dense_equiv_int8_tops=round(28 * a, 1),
                     kept_slices=round(kept["kept_slices"], 4), kept_mma=round(kept["kept_mma"], 4),
                     frac=round(ex / pk, 3), peak_int8_tops=round(pk, 1), peak_source=src)
        out[k] = e
    return out


def fused_update_rooflines(prec, x, specs, peaks, reps):
    """The forward plane pass as it runs in 7 of the step's 8 applies: with BiCGSTAB's s update
    (fmp_precond_apply_lincomb) or p update (fmp_precond_apply_bicg_p) fused in.  Times from the
    same stage events as stage_rooflines; work = the plain pass's DMMA flops plus the update's
    HBM bytes per owned DoF (s: v read + s written; p: r, v read + p written)."""
    import torch
    plan = prec.plan
    if plan.path() != "fast" or max(max(sp.ext) for sp in specs) <= 24 or prec.exchanger.active:
        return None   # plans / blocks that run the two-pass form
    flops = sum(6 * int(np.prod(sp.ext)) * (sp.ext[0] + sp.ext[1]) for sp in specs)
    dof = x.numel()
    v, s, pn, z = (torch.empty_like(x) for _ in range(4))
    v.copy_(x).mul_(0.5)
    s.copy_(x)
    out = {}
    plan.profile(True)
    for name, extra_b, fn in (("s_update", 16, lambda: prec.apply_lincomb_into(x, v, -0.3, s, z)),
                              ("p_update", 24, lambda: prec.apply_bicg_p_into(x, s, v, 0.4, 1.1, pn, z))):
        ms = 0.0
        for _ in range(reps):
            torch.cuda._sleep(2_000_000)
            fn()
            ms += plan.stage_ms()["plane_fwd"] / reps
        a = flops / ms / 1e9
        out[name] = {"kernel": f"k_plane_fast<0, 5, {1 if name == 's_update' else 2}>", "ms": round(ms, 4),
                     "achieved_tflops": round(a, 2), "frac_dmma": round(a / peaks["fp64_tflops"], 3),
                     "update_bytes_per_dof": extra_b, "update_gbs": round(extra_b * dof / ms / 1e6, 1)}
    plan.profile(False)
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2508_07193_b200 import (Box, CnSolver, DeviceCnStepper, HostStepPipeline, SolverConfig,
                                       make_transport, _lib)
    from paper_2508_07193_b200.schwarz import proc_grid_for

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        tr = make_transport(args.backend)
    else:
        tr = make_transport("cuda")
    rank = tr.rank
    dev = torch.cuda.current_device()
    block, sub, overlap = CONFIGS[args.config]
    ggrid = proc_grid_for(world)
    gext = tuple(b * g for b, g in zip(block, ggrid))
    sgrid = tuple(n // s for n, s in zip(gext, sub))
    alpha = 0.25
    dt = 2.0 * math.sqrt(alpha)     # ref:cli.py:145
    cfg = SolverConfig(method=args.method, tol=1e-12, max_iter=1000)
    t_setup = time.perf_counter()
    solver = CnSolver(Box(*gext), sgrid, overlap, alpha, cfg, tr)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    shape4 = solver.op.layout.shape4
    gen = torch.Generator(device="cuda").manual_seed(42 + rank)
    E0 = torch.rand(shape4, dtype=torch.float64, device="cuda", generator=gen).mul_(2).sub_(1)
    H0 = torch.rand(shape4, dtype=torch.float64, device="cuda", generator=gen).mul_(2).sub_(1)
    stepper = DeviceCnStepper(solver, E0.clone(), H0.clone(), dt)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        stepper.step()
    torch.cuda.synchronize()
    barrier()
    # ---- timed region: K device-resident steps
    lib = _lib.lib()
    launches0 = lib.fmp_launch_count()
    iters = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        barrier()
        ev0.record()
        for _ in range(args.steps):
            rep = stepper.step()
            iters.append(rep.iterations)
        ev1.record()
        torch.cuda.synchronize()
        barrier()
    launches = lib.fmp_launch_count() - launches0
    t_total = max_over_ranks(ev0.elapsed_time(ev1) * 1e-3)
    ms_per_step = t_total / args.steps * 1e3
    dof = 3 * int(np.prod(gext))
    value = dof * args.steps / t_total / 1e6

    # ---- component timings (CUDA events on the launching stream) for the roofline
    prec, op = solver.prec, solver.op
    x = stepper.E.clone()
    z = torch.empty_like(x)
    reps = 5
    for _ in range(2):
        prec.apply_into(x, z)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        prec.apply_into(x, z)
    e1.record()
    torch.cuda.synchronize()
    t_prec = e0.elapsed_time(e1) * 1e-3 / reps
    e0.record()
    for _ in range(reps):
        op.apply_into(x, z)
    e1.record()
    torch.cuda.synchronize()
    t_spmv = e0.elapsed_time(e1) * 1e-3 / reps
    from paper_2508_07193_b200.subdomain import analytic_cost, correction_size
    specs = solver.op.layout.sub_specs()
    flops_ref = flops_exec = 0
    bytes_alg = 0
    for s in specs:
        bx = Box(*s.ext)
        c = analytic_cost(bx, correction_size(bx))
        flops_ref += c.flops_per_solve
        flops_exec += c.flops_executed
        bytes_alg += 24 * bx.volume
    owned = int(np.prod(block))
    bytes_alg += 24 * owned + sum(8 * correction_size(Box(*e)) ** 2 for e in {s.ext for s in specs})
    peaks = measured_peaks()
    spmv_bytes = 48 * owned
    prec_tflops = flops_exec / t_prec / 1e12
    stages = stage_rooflines(prec, x, z, specs, peaks, reps)
    fused_stages = fused_update_rooflines(prec, x, specs, peaks, reps)

    # ---- per-phase breakdown of one extra step (reference categories, ref:instrument.py:17-25)
    from paper_2508_07193_b200.instrument import PhaseTimer
    timer = PhaseTimer()
    solver.timer = timer
    solver.op.timer = timer
    solver.prec.timer = timer
    torch.cuda.synchronize()
    tb0 = time.perf_counter()
    stepper.step()
    torch.cuda.synchronize()
    t_break = time.perf_counter() - tb0
    breakdown = {k: round(v * 1e3, 3) for k, v in timer.seconds.items()}
    breakdown["step_wall_ms"] = round(t_break * 1e3, 3)
    from paper_2508_07193_b200.instrument import NULL_TIMER
    solver.timer = solver.op.timer = solver.prec.timer = NULL_TIMER

    # ---- end-to-end through the public API: host fields in, host fields out, every step
    e2e = None
    if not args.no_e2e:
        Eh = E0.cpu().pin_memory()
        Hh = H0.cpu().pin_memory()
        Eo, Ho = torch.empty_like(Eh).pin_memory(), torch.empty_like(Hh).pin_memory()
        pipe = HostStepPipeline(solver, dt)   # public API: host fields in/out, overlapped transfers
        pipe.run(Eh, Hh, Eo, Ho, steps=1)     # warm-up
        # enough steps that the pipeline fill (the first step's H2D, ~15 ms) and drain (the last
        # step's D2H) amortise: the steady state is one device step plus ~0.7 ms of copy interference
        ke = max(args.steps, 16)
        torch.cuda.synchronize()
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        pipe.run(Eh, Hh, Eo, Ho, steps=ke)
        a1.record()
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(a0.elapsed_time(a1) * 1e-3)
        # this box's host link (one pinned field each way), to read the e2e number against
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dbuf = torch.empty_like(stepper.E)
        c0.record()
        dbuf.copy_(Eh, non_blocking=True)
        c1.record()
        torch.cuda.synchronize()
        h2d_gbs = Eh.numel() * 8 / c0.elapsed_time(c1) / 1e6
        c0.record()
        Eo.copy_(dbuf, non_blocking=True)
        c1.record()
        torch.cuda.synchronize()
        d2h_gbs = Eh.numel() * 8 / c0.elapsed_time(c1) / 1e6
        e2e = {"value": round(dof * ke / t_e2e / 1e6, 3), "unit": "MDoF/s",
               "h2d_bytes_per_step": 2 * Eh.numel() * 8, "d2h_bytes_per_step": 2 * Eo.numel() * 8,
               "steps": ke, "ms_per_step": round(t_e2e / ke * 1e3, 3),
               "host_link_gbs": {"h2d": round(h2d_gbs, 1), "d2h": round(d2h_gbs, 1)},
               "note": "HostStepPipeline: independent steps from host-resident E,H (throughput workload); "
                       "each step's H2D/D2H inside the timed region, overlapped with neighbouring solves"}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "MDoF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic: E,H ~ U[-1,1) (torch Philox, seed 42+rank)",
        "config": {"workload": f"{args.config}: CN-FDTD step, {'GMRES(30)' if getattr(args, 'method', 'bicgstab') == 'gmres' else 'BiCGSTAB'}+FlashMP RAS, tol 1e-12, alpha 0.25, "
                               f"overlap {overlap}", "global_grid": list(gext), "per_gpu_block": list(block),
                   "subdomain": list(sub), "subdomain_grid": list(sgrid), "gpu_grid": list(ggrid),
                   "parallelism": f"domain decomposition x{world}",
                   "l2": "inputs larger than L2 (each field 403 MB per GPU at 256^3)"},
        "step_time_s": round(ms_per_step / 1e3, 6), "iters_per_step": iters,
        "setup_s": round(setup_s, 3),
        "precond_apply": {"ms": round(t_prec * 1e3, 4), "GB_per_s": round(bytes_alg / t_prec / 1e9, 1),
                          "algorithmic_bytes": bytes_alg, "flops_reference_count": flops_ref,
                          "flops_executed": flops_exec, "tflops_executed": round(prec_tflops, 2),
                          "tflops_reference_count": round(flops_ref / t_prec / 1e12, 2)},
        "precond_kernels": stages,
        "plane_fwd_fused_update": fused_stages,
        "spmv": {"ms": round(t_spmv * 1e3, 4), "GB_per_s": round(spmv_bytes / t_spmv / 1e9, 1),
                 "algorithmic_bytes": spmv_bytes,
                 "traffic_bytes": ncu_traffic().get("k_spmv_bulk<0, 4>", {}).get("traffic_bytes"),
                 "frac_hbm": round(spmv_bytes / t_spmv / 1e9 / peaks["hbm_gbs"], 3)},
        "roofline": dominant_roofline(stages, peaks),
        "roofline_apply": {"kernel": "RAS precond apply (fused FlashMP sequence: FP64 DMMA transforms + Ozaki INT8 tcgen05 Woodbury GEMM)",
                     "note": "composite: executed FP64-equivalent flops of all 8 kernels over the FP64 DMMA peak; "
                             "the Woodbury GEMM's share runs on the INT8 pipe, so this can exceed an FP64-only bound",
                     "bound": "tensor", "achieved": round(prec_tflops, 3), "peak": peaks["fp64_tflops"],
                     "unit": "TFLOP/s", "frac": round(prec_tflops / peaks["fp64_tflops"], 3)
                     if peaks["fp64_tflops"] else None,
                     "traffic": (sum(v.get("traffic_bytes", 0) for v in stages.values()) or None),
                     "traffic_note": "DRAM bytes per apply, sum over its kernels from one ncu --set full capture "
                                     f"({NCU_TRAFFIC_FILE.relative_to(ROOT)}); algorithmic bytes "
                                     f"{bytes_alg} (precond_apply.algorithmic_bytes)",
                     "peak_source": peaks["fp64_source"], "flops_per_launch": flops_exec},
        "breakdown_ms": breakdown,
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, steps=args.cpu_steps, method=args.method)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------------------------- CPU reference
# The reference is pure Python (numpy/scipy), so "the reference's own CPU implementation" is the
# numpy restatement oracle/flashmp_oracle.py (the reference cannot travel to the GPU box).  It is
# timed on REAL CN steps (RHS -> BiCGSTAB to 1e-12 with the real Woodbury C^-1 -> H update,
# ref:cn_driver.py:82-94, cli.py:139-182) on a bounded sample of the workload: the same 32^3
# subdomains, alpha, overlap and tolerance on a smaller grid (CPU_SAMPLE), so a step takes a few
# seconds on the host cores.  Precompute (C^-1 per extended shape) is setup, outside the timed
# region, as in the reference's own cn_steps.csv seconds (ref:cli.py:164-171).
CPU_SAMPLE = {"cfg4": ((128, 128, 128), (32, 32, 32)), "cfg2": ((64, 64, 64), (32, 32, 32)),
              "cfg1": ((32, 32, 32), (32, 32, 32)), "cfg5_sd16": ((64, 64, 64), (16, 16, 16)),
              "cfg5_sd64": ((64, 64, 64), (64, 64, 64))}


class CpuCnSample:
    """Real CN steps of the CPU reference algorithm (oracle port) on the sample grid."""

    def __init__(self, config: str, seed: int = 42, method: str = "bicgstab"):
        sys.path.insert(0, str(ROOT / "oracle"))
        import flashmp_oracle as O
        self.O = O
        self.gext, sub = CPU_SAMPLE[config]
        self.sub, self.method = sub, method
        self.grid = tuple(n // s for n, s in zip(self.gext, sub))
        self.alpha = 0.25
        self.dt = 2.0 * math.sqrt(self.alpha)      # ref:cli.py:145
        self.ranks = O.partition(self.gext, self.grid, 1)
        t0 = time.perf_counter()
        for r in self.ranks:                       # C^-1 per distinct extended shape (setup)
            O.solver_data(r.ext, self.alpha, closed_form=True)
        self.setup_s = time.perf_counter() - t0
        rng = np.random.default_rng(seed)          # ref:cli.py:143-149
        shape = (3, self.gext[2], self.gext[1], self.gext[0])
        self.E = rng.uniform(-1.0, 1.0, shape)
        self.H = rng.uniform(-1.0, 1.0, shape)
        self.dof = 3 * int(np.prod(self.gext))
        self.iters: list[int] = []

    def step(self) -> float:
        O, g, a = self.O, self.gext, self.alpha
        op = lambda u: O.op_apply(g, a, u)
        prec = lambda u: O.ras_apply(g, self.ranks, a, u)

        def solve(rhs):
            if self.method == "gmres":
                return O.gmres(op, prec, rhs.ravel(), restart=30, tol=1e-12, max_iter=1000)
            return O.bicgstab(op, prec, rhs.ravel(), tol=1e-12, max_iter=1000)

        t0 = time.perf_counter()
        self.E, self.H, rep = O.cn_step(self.E, self.H, self.dt, solve)
        sec = time.perf_counter() - t0
        self.iters.append(rep.iterations)
        return sec

    def describe(self, steps: int) -> str:
        return (f"oracle/flashmp_oracle.py (numpy restatement of the reference; OpenBLAS threads = host cores): "
                f"{steps} real CN steps (RHS, {'GMRES(30)' if self.method == 'gmres' else 'BiCGSTAB'} to 1e-12 with "
                f"real C^-1, H update; time-marching) on a {'x'.join(map(str, self.gext))} grid of "
                f"{len(self.ranks)} subdomains of {self.sub[0]}^3 (overlap 1, "
                f"alpha 0.25), measured iterations per step {self.iters}; C^-1 precompute {self.setup_s:.1f} s "
                f"untimed (setup)")


def cpu_baseline(config: str, steps: int = 2, method: str = "bicgstab"):
    """Rank-0, N=1 CPU baseline beside our own line: `steps` real CN steps of the sample."""
    smp = CpuCnSample(config, method=method)
    smp.step()                                    # warm-up (first-touch, BLAS thread pool)
    times = [smp.step() for _ in range(steps)]
    sec = statistics.mean(times)
    return {"value": round(smp.dof / sec / 1e6, 4), "unit": "MDoF/s", "cores": os.cpu_count(), "kind": "port",
            "sample": smp.describe(steps), "step_s": round(sec, 3), "setup_s": round(smp.setup_s, 1)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    smp = CpuCnSample(args.config, method=args.method)
    for _ in range(args.warmup):
        smp.step()
    smp.iters.clear()
    t0 = time.perf_counter()
    times = [smp.step() for _ in range(args.steps)]
    t_total = time.perf_counter() - t0
    step = t_total / args.steps
    value = smp.dof / step / 1e6
    block, sub, overlap = CONFIGS[args.config]
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "MDoF/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step * 1e3, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: E,H ~ U[-1,1) (numpy PCG64 seed 42, ref:cli.py:143-149)",
            "config": {"workload": f"{args.config}: CN-FDTD step, {'GMRES(30)' if getattr(args, 'method', 'bicgstab') == 'gmres' else 'BiCGSTAB'}+FlashMP RAS, tol 1e-12, alpha 0.25, "
                                   f"overlap {overlap} (CPU reference algorithm on a bounded sample grid)",
                       "sample_grid": list(smp.gext), "subdomain": list(sub), "subdomain_grid": list(smp.grid),
                       "world_launch": world},
            "iters_per_step": smp.iters, "step_times_s": [round(t, 3) for t in times],
            "setup_s": round(smp.setup_s, 1),
            "cpu_baseline": {"value": round(value, 4), "unit": "MDoF/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": smp.describe(args.steps)},
            "e2e": {"value": round(value, 4), "unit": "MDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--method", default="bicgstab", choices=["bicgstab", "gmres"],
                    help="Krylov method (BASELINE configs 1-4: BiCGSTAB; config 5 also GMRES(30))")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2, help="timed CN steps of the CPU baseline sample")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N > 1 (gloo stages through host memory; testing only)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

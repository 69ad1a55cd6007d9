"""Digest of ncu --set full reports: time, DRAM bytes, pipe utilisation, issue, top stall reasons.
    python tools/ncu_digest.py gpurun_out/v12_*.ncu-rep"""
import csv, subprocess, sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64pipe%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block")]


def digest(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v))
        un = dict(zip(h, u))
        print(f"== {path}  {d.get('Kernel Name', '')[:70]}")
        print("   " + "  ".join(f"{n}={d.get(k, '?')}{un.get(k, '')}" for k, n in KEYS if k in d))
        stalls = [(float(d[k].replace(",", "") or 0), k) for k in h
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
        stalls.sort(reverse=True)
        print("   stalls/issue: " + ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, k in stalls[:7]))


for p in sys.argv[1:]:
    digest(p)

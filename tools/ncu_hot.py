"""Top stall-sampled SASS lines of an ncu report: python tools/ncu_hot.py REPORT [N]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))
tot = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
rows.sort(key=lambda r: -float(r["Warp Stall Sampling (All Samples)"] or 0))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in rows[:n]:
    v = float(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{v / tot:6.1%}  {r['Address']:>6}  {r['Source'][:90]}")

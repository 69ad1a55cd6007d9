"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import csv, collections, io, sys
text = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
agg = collections.OrderedDict()
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0][:60]
    agg.setdefault(k, []).append(float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]])
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'mean_us':>10s} {'total_us':>11s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} {len(v):5d} {sum(v)/len(v):10.1f} {sum(v):11.1f} {sum(v)/tot:6.1%}")

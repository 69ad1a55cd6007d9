"""DRAM traffic per launch of every preconditioner / SpMV kernel from ncu --set full reports:
    python tools/ncu_traffic.py OUT.json REPORT...   (reports from tools/ncu_full.sh)"""
import csv, json, subprocess, sys

out = {}
for path in sys.argv[2:]:
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, u = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for v in rows[2:]:
        d, un = dict(zip(h, v)), dict(zip(h, u))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale[un["dram__bytes_read.sum"]]
        wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale[un["dram__bytes_write.sum"]]
        t = float(d["gpu__time_duration.sum"].replace(",", ""))
        out[name] = {"dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "traffic_bytes": int(rd + wr),
                     "ncu_time_us": t, "report": path.split("/")[-1]}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1))

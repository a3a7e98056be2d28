"""Add a traffic.json entry from an `ncu --set full` report of one stencil launch on the bench
workload:  python tools/traffic.py REPORT.ncu-rep|RAW.csv KEY LEVELS [raw_csv_out]
(RAW.csv: the report's `ncu -i REPORT --page raw --csv` export)"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key, levels = sys.argv[1], sys.argv[2], int(sys.argv[3])
raw = (open(rep).read() if rep.endswith(".csv") else
       subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
if len(sys.argv) > 4:
    open(sys.argv[4], "w").write(raw)
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
d = dict(zip(h, r[2]))
f = lambda k: float(d[k].replace(",", ""))
unit = dict(zip(h, r[1]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = f("dram__bytes_read.sum") * scale.get(unit["dram__bytes_read.sum"], 1)
wr = f("dram__bytes_write.sum") * scale.get(unit["dram__bytes_write.sum"], 1)
tscale = {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}
dur = f("gpu__time_duration.sum") * tscale.get(unit["gpu__time_duration.sum"], 1)
esz = 8 if "double" in d["Kernel Name"] else 4
algo = 32766 * 4094 * esz * (4 if levels > 1 else 3)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
t = json.load(open(path))
t[key] = {"workload": "config4_weak_unit_delta_line_32768x4096_per_gpu", "kernel": d["Kernel Name"],
          "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
          "algorithmic_bytes_per_launch": algo, "traffic_over_algorithmic": (rd + wr) / algo,
          "levels_per_launch": levels, "ncu_duration_us": dur,
          "source": f"ncu --set full --clock-control none, 1 steady-state launch ({os.path.basename(rep)})"}
json.dump(t, open(path, "w"), indent=1)
print(key, t[key])

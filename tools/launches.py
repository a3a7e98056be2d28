"""Summarise an ncu --metrics launch-list CSV: mean time and DRAM bytes per kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
pat = sys.argv[2] if len(sys.argv) > 2 else ""
hdr = None
d = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        k = dict(zip(hdr, r))
        d[k["Kernel Name"][:44]][k["Metric Name"]].append(float(k["Metric Value"].replace(",", "")))
for k, v in d.items():
    if pat not in k:
        continue
    t = v["gpu__time_duration.sum"]
    rd = v.get("dram__bytes_read.sum", [0])
    wr = v.get("dram__bytes_write.sum", [0])
    print(f"{k:44s} n={len(t):3d} t={sum(t)/len(t)/1e3:9.1f}us rd={sum(rd)/len(rd)/1e6:8.1f}MB wr={sum(wr)/len(wr)/1e6:8.1f}MB")

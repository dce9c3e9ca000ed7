"""Summarise an ncu --csv launch list: per kernel ID, time and DRAM bytes (>= min_us)."""
import csv
import sys
from collections import OrderedDict

path = sys.argv[1]
min_us = float(sys.argv[2]) if len(sys.argv) > 2 else 50.0
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
k = OrderedDict()
for d in data:
    key = (int(d["ID"]), d["Kernel Name"][:60])
    k.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for (i, name), m in k.items():
    t = m.get("gpu__time_duration.sum", 0)
    if t > min_us * 1e3:
        print(f"{i:4d} {name:60s} {t / 1e6:8.3f} ms  R {m.get('dram__bytes_read.sum', 0) / 1e9:7.2f} GB "
              f"W {m.get('dram__bytes_write.sum', 0) / 1e9:7.2f} GB")

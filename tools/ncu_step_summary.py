"""Sum an ncu --metrics --csv launch log per kernel (one SpMV step = the listed launches)."""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]
idx = {h: i for i, h in enumerate(hdr)}
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    if r[idx["ID"]].isdigit():
        i = int(r[idx["ID"]])
        per[i][r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
        names[i] = r[idx["Kernel Name"]].split("(")[0]
tot = collections.Counter()
for i, m in per.items():
    for k, v in m.items():
        if "pct" in k or "registers" in k:
            continue
        tot[k] += v
out = {"launches": len(per), "kernels": sorted(set(names.values())), "sum": dict(tot),
       "per_launch": [{"kernel": names[i], **per[i]} for i in sorted(per)]}
t_ns = tot.get("gpu__time_duration.sum", 0)
if t_ns:
    out["step_ms"] = t_ns / 1e6
    out["dram_bytes"] = tot.get("dram__bytes_read.sum", 0) + tot.get("dram__bytes_write.sum", 0)
    out["dram_GBps"] = out["dram_bytes"] / t_ns
    cyc = tot.get("sm__cycles_elapsed.avg", 0)
    if cyc:
        out["sm_clock_GHz"] = cyc / t_ns
        req = tot.get("lts__t_requests_srcunit_tex.sum", 0)
        out["l2_requests_per_sm_cycle"] = req / 148 / cyc
print(json.dumps(out, indent=1))

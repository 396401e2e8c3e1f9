#!/usr/bin/env python3
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
tot = 0.0
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
for d in data:
    name = d["Kernel Name"].split("(")[0][:48]
    t = float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
    key = (name, d.get("Grid Size", ""))
    agg.setdefault(key, [0, 0.0])
    agg[key][0] += 1
    agg[key][1] += t
    tot += t
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[1]:10.1f} us {v[0]:3d}x {100 * v[1] / tot:5.1f}%  {k[0]:48s} {k[1]}")
print(f"total {tot:.1f} us over {len(data)} launches")

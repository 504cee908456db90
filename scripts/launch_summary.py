#!/usr/bin/env python
"""Mean duration per kernel of an ncu --csv launch list (gpu__time_duration.sum)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]
            data[name].append(float(d["Metric Value"].replace(",", "")))
tot = 0.0
for k, v in data.items():
    m = sum(v) / len(v) / 1000
    tot += m
    print(f"{k:28s} n={len(v):4d} mean {m:8.2f} us")
print(f"{'sum of means':28s}        {tot:8.2f} us")

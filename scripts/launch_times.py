#!/usr/bin/env python
"""Mean per-kernel duration from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
ix = {k: i for i, k in enumerate(rows[0])}
d = defaultdict(list)
for r in rows[1:]:
    if r[ix["Metric Name"]] == "gpu__time_duration.sum":
        d[r[ix["Kernel Name"]][:70]].append(float(r[ix["Metric Value"]].replace(",", "")))
for k, v in d.items():
    print(f"{k:70s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:8.1f} us")

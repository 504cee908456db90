#!/usr/bin/env python
"""Per-source-line shared-memory wavefronts (excessive = bank conflicts) and stall samples of an
ncu report captured with --import-source on.

    python scripts/ncu_conflicts.py gpurun_out/prof_attn_v33.ncu-rep [--top 15]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[2]
n = len(hdr)
ix = {k: i for i, k in enumerate(hdr)}
agg = collections.defaultdict(lambda: [0, 0, 0, 0])
cur, fn = None, None
for r in rows[3:]:
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r[0] and r[0].isdigit() and (len(r) < 4 or r[2] in ("-", "")):
        cur = (fn, int(r[0]), r[1][:70])
        continue
    if len(r) > n:  # SASS text split on its commas: re-join it
        r = r[:3] + [",".join(r[3:3 + len(r) - n + 1])] + r[4 + len(r) - n:]
    if len(r) != n:
        continue
    try:
        a = agg[cur]
        a[0] += int(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
        a[1] += int(r[ix["L1 Wavefronts Shared"]] or 0)
        a[2] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        a[3] += int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
tot = [sum(v[i] for v in agg.values()) or 1 for i in range(4)]
print(f"shared wavefronts {tot[1]}, excessive {tot[0]} ({100 * tot[0] / tot[1]:.1f}%); stall samples {tot[2]}")
print("-- by excessive shared wavefronts")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    if v[0]:
        print(f"  excess {v[0]:9d} of {v[1]:9d}  stall {100 * v[2] / tot[2]:5.1f}%  {k}")
print("-- by stall samples")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"  stall {100 * v[2] / tot[2]:5.1f}%  inst {100 * v[3] / tot[3]:5.1f}%  excess {v[0]:8d}  {k}")

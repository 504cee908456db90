#!/usr/bin/env python
"""Static SASS opcode counts per kernel of the built library (cuobjdump -sass): the evidence of
which tensor-core / TMA generation each kernel uses (tcgen05: UTCIMMA/UTCHMMA, LDTM/STTM; TMA bulk:
UBLKCP; legacy mma.sync: IMMA/HMMA; fp64: DMMA/DFMA).

    python scripts/sass_opcodes.py [build/*.o]  > profiles/rNN_sass_opcodes.txt
"""
import collections
import glob
import re
import subprocess
import sys

OPS = ["UTCIMMA", "UTCHMMA", "UTCQMMA", "LDTM", "STTM", "UTMALDG", "UBLKCP", "IMMA", "HMMA", "DMMA", "DFMA",
       "SYNCS", "BAR", "FFMA2"]
files = sys.argv[1:] or sorted(glob.glob("build/*.o"))
for f in files:
    out = subprocess.run(["cuobjdump", "-sass", f], capture_output=True, text=True).stdout
    kern, counts = None, collections.OrderedDict()
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = collections.Counter()
            continue
        if kern is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9]*)(\.\S+)?", line)
        if m:
            op = m.group(2)
            full = (m.group(2) + (m.group(3) or ""))
            for o in OPS:
                if op == o or (o == "FFMA2" and full.startswith("FFMA2")):
                    counts[kern][o] += 1
    for k, c in counts.items():
        if not any(c.values()):
            continue
        name = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(.*", "", name.replace("(anonymous namespace)::", ""))[:110]
        print(f"{f.split('/')[-1]:14s} {name}")
        print("    " + "  ".join(f"{o} {c[o]}" for o in OPS if c[o]))

#!/usr/bin/env python
"""Build a profiling variant of libdquant_b200.so with extra nvcc flags into variants/<name>/.

    python scripts/build_variant.py smtrace -DDQ_GQ_SMTRACE
    DQ_LIB=variants/smtrace/libdquant_b200.so python scripts/attn_trace.py

variants/ is git-ignored but travels to the GPU box with the snapshot (build/ does not).
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12591_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out = os.path.join(B.ROOT, "variants", name)
os.makedirs(out, exist_ok=True)


def comp(src):
    obj = os.path.join(out, src.replace(".cu", ".o"))
    subprocess.run([B.NVCC, *B.FLAGS, *extra, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
    return obj


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, B._sources()))
lib = os.path.join(out, "libdquant_b200.so")
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "shared", "-o", lib, *objs], check=True)
for o in objs:
    os.remove(o)
print(lib)

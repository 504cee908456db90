#!/usr/bin/env python
"""Per-work-item phase timeline of the fused attention kernel (globaltimer stamps), C2 shapes."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12591_b200 import _lib  # noqa: E402
from paper_2405_12591_b200.attention import DecodeKvCache  # noqa: E402

units, T = int(os.environ.get("UNITS", 512)), int(os.environ.get("T", 4096))
G = int(os.environ.get("G", 1))  # G=8: the tcgen05 GQA kernel (path 2)
ctas = os.environ.get("CTAS")
cache = DecodeKvCache(layers=1, units=units, g=G, bits=int(os.environ.get("BITS", 4)),
                      chunk_b=int(os.environ["CHUNK_B"]) if os.environ.get("CHUNK_B") else None,
                      ctas=None if ctas is None else int(ctas),
                      tc=None if G == 8 else bool(int(os.environ.get("TC", "0"))))
k = torch.randn((units, T, 128), device="cuda").half()
cache.prefill(0, k, k)
del k
q = torch.randn((units, G, 128), device="cuda").half()
out = torch.empty_like(q)
cache.attend(0, q, out)
a = cache._layers[0].args
trace = torch.zeros((a.nwork, 8), dtype=torch.int64, device="cuda")
a.trace = trace.data_ptr()
for _ in range(3):
    cache.launch(0, q, out, phases=1)
torch.cuda.synchronize()
t = trace.cpu().numpy().astype(np.float64)
if os.environ.get("SAVE"):
    np.savez(os.environ["SAVE"], trace=trace.cpu().numpy(), work=cache._layers[0].keep[1].cpu().numpy())
t0 = t[:, 0].min()
path = cache._layers[0].args.path
if path == 2:  # stamps 0 start, 1 K done, 2 softmax done, 3 V done, 5 end (slots 4, 6, 7: profiling builds)
    rel = lambda c: ((t[:, c] - t[:, 0]) / 1e3).mean()  # noqa: E731
    print(f"consumers: K done {rel(1):.2f}, softmax done {rel(2):.2f}, V done {rel(3):.2f}, end {rel(5):.2f} us "
          f"(item-relative means)")
    if os.environ.get("MMAWAIT"):  # build with -DDQ_GQ_MMAWAIT: MMA warp V phase span / A waits / Y waits, ns
        print(f"MMA warp V phase: span {(t[:, 4] / 1e3).mean():.2f} us, waiting for A {(t[:, 6] / 1e3).mean():.2f} us, "
              f"for Y {(t[:, 7] / 1e3).mean():.2f} us")
    if os.environ.get("WIDETRACE"):  # build with -DDQ_GQ_WIDETRACE: widening warp V stages span / ring waits / A waits
        print(f"widening V stages: span {(t[:, 4] / 1e3).mean():.2f} us, waiting for the ring {(t[:, 6] / 1e3).mean():.2f} us, "
              f"for A buffers {(t[:, 7] / 1e3).mean():.2f} us")
    if os.environ.get("ROLETRACE") == "1":  # -DDQ_GQ_ROLETRACE=1: the MMA warp per period (V(j) + K(j+2))
        print(f"MMA warp per period: span {(t[:, 4] / 1e3).mean():.2f} us, waiting for A {(t[:, 6] / 1e3).mean():.2f} us, "
              f"for P / Y / S {(t[:, 7] / 1e3).mean():.2f} us")
    if os.environ.get("ROLETRACE") == "2":  # -DDQ_GQ_ROLETRACE=2: the widening warps per period
        print(f"widening per period: span {(t[:, 4] / 1e3).mean():.2f} us, waiting for the ring {(t[:, 6] / 1e3).mean():.2f} us, "
              f"for A buffers {(t[:, 7] / 1e3).mean():.2f} us")
    if os.environ.get("SMTRACE"):  # build with -DDQ_GQ_SMTRACE: 7 S ready, 4 row max, 6 column max
        print(f"softmax: row max {rel(4):.2f}, column max {rel(6):.2f}, P written {rel(2):.2f}")
    t[:, 4] = t[:, 3]
ph = np.diff(t[:, :6], axis=1) / 1e3  # us
names = (["K stages", "softmax", "V stages", "(unused)", "epilogue"] if path in (1, 2) else
         ["prologue+W", "K stages", "softmax", "V stages", "epilogue"])
print(f"ctas {a.nctas}, items {a.nwork}, kernel span {(t[:, 5].max() - t0) / 1e3:.1f} us")
for i, n in enumerate(names):
    print(f"  {n:11s} mean {ph[:, i].mean():6.2f} us  p50 {np.median(ph[:, i]):6.2f}  p90 {np.percentile(ph[:, i], 90):6.2f}")
life = (t[:, 5] - t[:, 0]) / 1e3
print(f"  item life  mean {life.mean():6.2f} us  min {life.min():6.2f}  max {life.max():6.2f}")
starts = np.sort((t[:, 0] - t0) / 1e3)
print("  start-time quantiles (us):", np.round(np.percentile(starts, [0, 25, 50, 75, 90, 100]), 1))
ends = np.sort((t[:, 5] - t0) / 1e3)
print("  end-time quantiles (us):  ", np.round(np.percentile(ends, [0, 25, 50, 75, 90, 100]), 1))
# concurrency over time
grid = np.linspace(0, ends[-1], 40)
conc = [int(((t[:, 0] - t0) / 1e3 <= x).sum() - ((t[:, 5] - t0) / 1e3 <= x).sum()) for x in grid]
print("  resident items over time:", conc)
# per-CTA finish times (stamp 6 = blockIdx, 7 = SM; path 1 reuses them)
if path in (1, 2):
    t[:, 6] = 0
cta = t[:, 6].astype(int)  # (path 1: no SM ids)
ncta = cta.max() + 1
cta_end = np.array([(t[cta == c, 5].max() - t0) / 1e3 for c in range(ncta) if (cta == c).any()])
cta_items = np.bincount(cta)
print(f"  CTAs {ncta}: items per CTA min {cta_items.min()} max {cta_items.max()}")
print("  CTA end quantiles (us):   ", np.round(np.percentile(cta_end, [0, 10, 50, 90, 100]), 1))

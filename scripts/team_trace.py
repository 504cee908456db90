#!/usr/bin/env python
"""Per-item phase timeline of the mma.sync split kernel (path 0), built with -DDQ_ATTN_TRACE:
stamps 0 item start (W image in), 1 K phase done, 2 softmax done, 3 V phase done, 4 end; slots 5-7
CTA, SM, team.  Prints the mean phase lengths, the gap between a team's items, and per SM how
much of the kernel had 0 / 1 / 2 teams streaming (K or V phase).

    DQ_LIB=variants/trace/libdquant_b200.so python scripts/team_trace.py     (C2 shape, 1 layer)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12591_b200.attention import DecodeKvCache  # noqa: E402

units, T = int(os.environ.get("UNITS", 512)), int(os.environ.get("T", 4096))
cache = DecodeKvCache(layers=1, units=units, g=1, bits=int(os.environ.get("BITS", 4)),
                      chunk_b=int(os.environ["CHUNK_B"]) if os.environ.get("CHUNK_B") else None)
k = torch.randn((units, T, 128), device="cuda").half()
cache.prefill(0, k, k)
del k
q = torch.randn((units, 1, 128), device="cuda").half()
out = torch.empty_like(q)
cache.attend(0, q, out)
a = cache._layers[0].args
trace = torch.zeros((a.nwork, 8), dtype=torch.int64, device="cuda")
a.trace = trace.data_ptr()
for _ in range(3):
    cache.launch(0, q, out, phases=1)
torch.cuda.synchronize()
t = trace.cpu().numpy().astype(np.float64)
t0, t1 = t[:, 0].min(), t[:, 4].max()
us = lambda x: x / 1e3  # noqa: E731
print(f"items {a.nwork}, span {us(t1 - t0):.1f} us")
for name, c0, c1 in [("K", 0, 1), ("softmax", 1, 2), ("V", 2, 3), ("epilogue", 3, 4)]:
    d = us(t[:, c1] - t[:, c0])
    print(f"  {name:9s} mean {d.mean():6.2f} us  p90 {np.percentile(d, 90):6.2f}")
# gaps between consecutive items of one team (end -> next start: W image wait + descriptor)
gaps = []
for (cta, team) in {(int(r[5]), int(r[7])) for r in t}:
    rows = t[(t[:, 5] == cta) & (t[:, 7] == team)]
    rows = rows[np.argsort(rows[:, 0])]
    gaps += list(us(rows[1:, 0] - rows[:-1, 4]))
print(f"  item gap  mean {np.mean(gaps):6.2f} us")
# streaming teams per SM over time (1 ns grid is too fine: 20 ns bins)
bins = np.arange(t0, t1, 20.0)
hist = np.zeros(3)
for sm in np.unique(t[:, 6]):
    rows = t[t[:, 6] == sm]
    streaming = np.zeros(len(bins))
    for r in rows:
        for c0, c1 in ((0, 1), (2, 3)):
            streaming += (bins >= r[c0]) & (bins < r[c1])
    busy = (bins >= rows[:, 0].min()) & (bins < rows[:, 4].max())
    for n in range(3):
        hist[n] += np.sum((np.minimum(streaming, 2) == n) & busy)
hist /= hist.sum()
print(f"  SM time with 0 / 1 / 2 streaming phases: {hist[0]:.2f} / {hist[1]:.2f} / {hist[2]:.2f}")

#!/usr/bin/env python
"""Per-warp phase timeline of the split kernel (needs a build with -DDQ_ATTN_WARP_TRACE).

Stamps per (item, warp): 0 W ready, 1 K end, 2 after sync A (row max), 3 after sync B (tile
maxima), 4 after sync C (P ready), 5 V end, 6 after epilogue sync 1, 7 item end.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2405_12591_b200.attention import DecodeKvCache  # noqa: E402

units, T = 512, 4096
cache = DecodeKvCache(layers=1, units=units, g=1, bits=4)
k = torch.randn((units, T, 128), device="cuda").half()
cache.prefill(0, k, k)
q = torch.randn((units, 1, 128), device="cuda").half()
out = torch.empty_like(q)
cache.attend(0, q, out)
a = cache._layers[0].args
trace = torch.zeros((a.nwork, 8, 8), dtype=torch.int64, device="cuda")
a.trace = trace.data_ptr()
cache.launch(0, q, out, phases=1)
torch.cuda.synchronize()
a.trace = None
t = trace.cpu().numpy().astype(np.float64) / 1e3  # us
ok = (t > 0).all(axis=(1, 2))
t = t[ok]
names = ["K (W ready -> K end)", "K end -> sync A", "sync A -> sync B", "sync B -> sync C (P ready)",
         "V (sync C -> V end)", "V end -> epilogue sync 1", "sync 1 -> item end"]
d = np.diff(t, axis=2)  # items x warps x 7
print(f"items {t.shape[0]}")
for i, n in enumerate(names):
    per_warp = d[:, :, i].mean(axis=0)
    print(f"  {n:30s} mean {d[:, :, i].mean():6.2f} us   per warp " + " ".join(f"{x:5.2f}" for x in per_warp))
# the wait at each barrier: last arrival minus own arrival
for k_, n in ((1, "sync A"), (3, "sync C"), (5, "epilogue sync 1")):
    arr = t[:, :, k_]
    print(f"  wait at {n:16s}: mean {(arr.max(axis=1)[:, None] - arr).mean():.2f} us, "
          f"last arriver by warp {np.bincount(arr.argmax(axis=1), minlength=8)}")
life = t[:, 0, 7] - t[:, 0, 0]
print(f"  item (W ready -> end) {life.mean():.2f} us")

#!/usr/bin/env python
"""tcgen05 split kernel (path 1) vs mma.sync (path 0) vs the CPU oracle on one layer."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dquant_oracle as O  # noqa: E402
from paper_2405_12591_b200.attention import DecodeKvCache  # noqa: E402

units, T = int(os.environ.get("UNITS", 6)), int(os.environ.get("T", 4096))
rng = np.random.default_rng(3)
k = rng.standard_normal((units, T, 128)).astype(np.float32)
k[:, :, [3, 70]] *= 20.0
k = k.astype(np.float16)
v = rng.standard_normal((units, T, 128)).astype(np.float16)
q = rng.standard_normal((units, 1, 128)).astype(np.float16)
outs = {}
for tc in (False, True):
    c = DecodeKvCache(layers=1, units=units, g=1, bits=4, tc=tc)
    c.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    outs[tc] = c.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    print("path", c._layers[0].args.path, "ctas", c.ctas)
ref = np.stack([O.attention_units(q[u:u + 1].astype(np.float32), k[u:u + 1].astype(np.float32),
                                  v[u:u + 1].astype(np.float32), 4)[0] for u in range(units)])


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


print("mma.sync vs oracle", max(rel(outs[False][u], ref[u]) for u in range(units)))
print("tcgen05  vs oracle", max(rel(outs[True][u], ref[u]) for u in range(units)))
print("tcgen05 vs mma.sync", max(rel(outs[True][u], outs[False][u]) for u in range(units)))

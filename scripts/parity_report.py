#!/usr/bin/env python
"""Print the fused-attention parity errors vs the CPU oracle for a few configurations (GPU)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dquant_oracle as O  # noqa: E402
from paper_2405_12591_b200.attention import DecodeKvCache  # noqa: E402


def run(bits, g, T, units=2, outlier=False, seed=0):
    rng = np.random.default_rng(seed)
    k = rng.standard_normal((units, T, 128)).astype(np.float32)
    if outlier:
        k[:, :, [3, 77]] *= 20.0
    k = k.astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, g, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=g, bits=bits)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    errs = []
    for u in range(units):
        lay = O.LayerOracle(128, bits, 1 << 30)
        lay.prefill(k[u].astype(np.float32), v[u].astype(np.float32))
        ref = lay.attend(q[u].astype(np.float32)).astype(np.float64)
        errs.append(np.linalg.norm(ref - out[u]) / np.linalg.norm(ref))
    return max(errs)


if __name__ == "__main__":
    for bits, g, T, outl in [(4, 1, 4096, False), (4, 1, 4096, True), (4, 2, 2048, False), (2, 1, 4096, False),
                             (8, 1, 2048, False), (4, 1, 1009, False)]:
        print(f"bits={bits} g={g} T={T} outlier={outl}: max rel err {run(bits, g, T, outlier=outl):.3e}", flush=True)

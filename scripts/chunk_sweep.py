#!/usr/bin/env python
"""Split-kernel work-item size sweep: mean attention time per layer (prepare + split + combine,
CUDA events, layers cycled so the compressed cache exceeds L2) for each (units, T, bits) case
and chunk_b in CHUNKS (0: the automatic plan).

    CASES="32x32768x4,16x32768x4,512x4096x4" CHUNKS=256,512 python scripts/chunk_sweep.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12591_b200.attention import DecodeKvCache  # noqa: E402

cases = [tuple(int(x) for x in c.split("x")) for c in os.environ.get("CASES", "32x32768x4").split(",")]
chunks = [int(c) for c in os.environ.get("CHUNKS", "256,512").split(",")]
for units, T, bits in cases:
    per_layer = units * T * 128 * 2 * bits / 8
    layers = max(2, int(4 * 126e6 / per_layer) + 1)
    for cb in chunks:
        cache = DecodeKvCache(layers=layers, units=units, g=1, bits=bits, chunk_len=1024, chunk_b=cb or None)
        gen = torch.Generator(device="cuda").manual_seed(0)
        for layer in range(layers):
            k = torch.randn((units, T, 128), generator=gen, device="cuda").half()
            cache.prefill(layer, k, k)
        q = torch.randn((units, 1, 128), device="cuda").half()
        out = torch.empty_like(q)
        for layer in range(layers):
            cache.attend(layer, q, out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            for layer in range(layers):
                cache.attend(layer, q, out)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * layers)
        nwork = cache._layers[0].args.nwork
        print(f"units {units:5d} T {T:6d} bits {bits} chunk_b {cb}: {us:7.1f} us/layer, {nwork} items, "
              f"{cache.split_ctas} ctas, {per_layer / us / 1e3:7.0f} GB/s", flush=True)
        del cache

"""Cost of sealing a 1024-token chunk into a segment (kvcache.py:124-128) at the C2 shape.

Times K3 (compress_blocks) on `units` K and `units` V blocks of `chunk` x 128 fp16 for one
layer, per kernel of the write path (CUDA events around the whole call; per-kernel split via
torch.profiler), and reports blocks/s and the amortised cost per decode step at 32 layers.

    python scripts/seal_cost.py [--units 512] [--chunk 1024] [--layers 32] [--step-ms 2.2]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2405_12591_b200 import _lib
from paper_2405_12591_b200.attention import compress_blocks

ap = argparse.ArgumentParser()
ap.add_argument("--units", type=int, default=512)
ap.add_argument("--chunk", type=int, default=1024)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--step-ms", type=float, default=2.2)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
k = torch.randn((a.units, a.chunk, 128), generator=g, device=dev).half()
v = torch.randn((a.units, a.chunk, 128), generator=g, device=dev).half()


def seal():
    compress_blocks(k, 4, _lib.LAYOUT_KTILE, torch.float32)
    compress_blocks(v, 4, _lib.LAYOUT_VTILE, torch.float32)


seal()
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    seal()
    e1.record()
    torch.cuda.synchronize()
    ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
dev_ms = min(t[0] for t in ts)
wall_ms = min(t[1] for t in ts)
blocks = 2 * a.units
res = {"units": a.units, "chunk": a.chunk, "blocks_per_layer": blocks, "layer_ms_device": dev_ms,
       "layer_ms_wall": wall_ms, "blocks_per_s": blocks / (dev_ms / 1e3),
       "seal_event_ms_all_layers": dev_ms * a.layers,
       "amortised_ms_per_step": dev_ms * a.layers / a.chunk,
       "fraction_of_step": dev_ms * a.layers / a.chunk / a.step_ms}
if a.profile:
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        seal()
        torch.cuda.synchronize()
    per = {}
    for ev in prof.key_averages():
        if ev.device_type.name == "CUDA":
            per[ev.key[:60]] = round(ev.device_time_total / 1e3, 3)
    res["kernels_ms"] = dict(sorted(per.items(), key=lambda x: -x[1])[:12])
print(json.dumps(res))

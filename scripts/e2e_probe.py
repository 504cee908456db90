#!/usr/bin/env python
"""Where the C2 end-to-end step's extra time goes: eager device-resident step, the same step
captured as a graph without host copies, and DecodeStepGraph (host copies on side streams)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12591_b200.attention import DecodeKvCache  # noqa: E402
from paper_2405_12591_b200.decode_step import DecodeStepGraph  # noqa: E402

L, U, T = int(os.environ.get("LAYERS", 32)), 512, 4096
cache = DecodeKvCache(layers=L, units=U, g=1, bits=4)
gen = torch.Generator(device="cuda").manual_seed(0)
for layer in range(L):
    k = torch.randn((U, T, 128), generator=gen, device="cuda").half()
    cache.prefill(layer, k, k)
q = torch.randn((L, U, 1, 128), device="cuda").half()
kn = torch.randn((L, U, 128), device="cuda").half()
out = torch.empty_like(q)


def step():
    for layer in range(L):
        cache.attend(layer, q[layer], out[layer], append=(kn[layer], kn[layer]))


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print(f"eager step          {timed(step):.3f} ms")
step()
torch.cuda.synchronize()
tails = [lay.tail_len for lay in cache._layers]
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for lay, t in zip(cache._layers, tails):
    lay.tail_len = t


def replay():
    g.replay()
    for layer in range(L):
        cache._after_append(layer)


print(f"graph, no copies    {timed(replay):.3f} ms")
q_h, k_h = q.cpu().pin_memory(), kn.cpu().pin_memory()
out_h = torch.empty(q.shape, dtype=torch.float16).pin_memory()
v_h = k_h.clone().pin_memory()
cands = [((1,) * L, (1,) * L), ((1, 3), None), ((1, 2, 4, 8, 16), (1, 2, 4, 8, 16)), ((1, 7), (1,) * L), ((1, 2, 4, 8, 16), (16, 8, 4, 2, 1)),
         ((1, 3, 12), (12, 12, 6, 2)), ((1, 2, 4, 8, 16), (8,) * 4), ((2, 6, 24), (2, 6, 24))]
steppers = [DecodeStepGraph(cache, q_h, k_h, v_h, out_h, up_sizes=u, down_sizes=d) for u, d in cands]
# round robin (each replay appends a token to every tail, so later replays cost more): every
# candidate sees the same tail lengths on average
tot = [0.0] * len(cands)
n = 10
for it in range(n):
    for ci, st in enumerate(steppers):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.replay()
        e1.record()
        torch.cuda.synchronize()
        tot[ci] += e0.elapsed_time(e1)
for (up, down), t in zip(cands, tot):
    print(f"up {str(up[:6]):18s} down {str(down[:6] if down else 'default'):22s} {t / n:.3f} ms")

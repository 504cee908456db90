import os, sys, time
import torch
sys.path.insert(0, '/root/repo')
from paper_2405_12591_b200.attention import DecodeKvCache
from paper_2405_12591_b200.decode_step import DecodeStepGraph, DeviceStepGraph
L, U, T = 32, 512, 4096
cache = DecodeKvCache(layers=L, units=U, g=1, bits=4)
gen = torch.Generator(device="cuda").manual_seed(0)
for layer in range(L):
    k = torch.randn((U, T, 128), generator=gen, device="cuda").half()
    cache.prefill(layer, k, k)
q = torch.randn((L, U, 1, 128), device="cuda").half()
kn = torch.randn((L, U, 128), device="cuda").half()
out = torch.empty_like(q)
ds = DeviceStepGraph(cache, q, kn, kn, out)
q_h, k_h = q.cpu().pin_memory(), kn.cpu().pin_memory()
out_h = torch.empty(q.shape, dtype=torch.float16).pin_memory()
hs = DecodeStepGraph(cache, q_h, k_h, k_h.clone().pin_memory(), out_h)
for name, st in (("device", ds), ("hosted", hs), ("device", ds), ("hosted", hs)):
    for _ in range(3): st.replay()
    torch.cuda.synchronize()
    n = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(n): st.replay()
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
    print(f"{name}: gpu {e0.elapsed_time(e1)/n:.3f} ms/step, host enqueue {(t1-t0)/n*1e3:.3f} ms/step")

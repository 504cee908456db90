#!/usr/bin/env python
"""End-to-end decode of a LLaMA-shaped random-init model with the DecoQuant KV cache.

    python scripts/model_decode.py [--shape 7b] [--batch 16] [--context 4096] [--steps 10]

Prints tokens/s of whole-model decode steps (attention through the fused DecoQuant kernels,
dense layers through cuBLAS bf16), CUDA-event timed.
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12591_b200.model import LLAMA2_7B, LLAMA2_13B, LLAMA2_70B, DecoQuantLM  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="7b", choices=["7b", "13b", "70b"])
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--context", type=int, default=4096)
ap.add_argument("--layers", type=int, default=None)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
shape = {"7b": LLAMA2_7B, "13b": LLAMA2_13B, "70b": LLAMA2_70B}[a.shape]
if a.layers:
    from dataclasses import replace
    shape = replace(shape, layers=a.layers)
t0 = time.perf_counter()
lm = DecoQuantLM(shape, a.batch)
lm.prefill_random(a.context)
torch.cuda.synchronize()
setup = time.perf_counter() - t0
tok = torch.zeros(a.batch, dtype=torch.int64, device="cuda")
for _ in range(a.warmup):
    tok = lm.step(tok)
torch.cuda.synchronize()


def timed(fn):
    global tok
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        tok = fn(tok)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps


eager_ms = timed(lm.step)
lm.capture()
ms = timed(lm.replay)
print(json.dumps({"model": f"llama2-{a.shape}-shape random-init", "layers": shape.layers, "batch": a.batch,
                  "context": a.context, "ms_per_step": ms, "tokens_per_s": a.batch / (ms / 1e3),
                  "eager_ms_per_step": eager_ms,
                  "kv_memory_vs_fp16": lm.cache.ledger()[1] / lm.cache.ledger()[0], "setup_s": setup}))

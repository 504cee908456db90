#!/usr/bin/env python
"""Eigensolver phase timing (K3's eig_tql_kernel): one block and a 1024-block batch of
2048 x 128 through deco_quantize_batched; run with DQ_LIB pointing at DQ_EIG_STOP builds."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12591_b200.compress import deco_quantize_batched  # noqa: E402

for n in (1, 32, 1024):
    x = torch.randn((n, 2048, 128), device="cuda").half()
    for _ in range(2):
        deco_quantize_batched(x, 4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        deco_quantize_batched(x, 4)
    e1.record()
    torch.cuda.synchronize()
    print(f"{n:5d} blocks: {e0.elapsed_time(e1) / 3:.3f} ms per call")

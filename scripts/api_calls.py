#!/usr/bin/env python
"""Reference-API calls one at a time (numpy in / numpy out): per-call wall time, for profiling
the drop-in path (bench.py --config c1 reports the same table as `api`)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_12591_b200 as dq  # noqa: E402

rng = np.random.default_rng(0)
block = rng.standard_normal((2048, 128)).astype(np.float16).astype(np.float32)
q = rng.standard_normal((1, 128)).astype(np.float32)
qm = dq.deco_quantize(block, 4)
cache = dq.KvCache(dq.CacheConfig(layers=1, dim=128, bits=4, chunk_len=1024))
cache.prefill(0, block, block)
for row in block[:1100]:
    cache.append_token(0, row, row)
calls = {
    "deco_quantize": lambda: dq.deco_quantize(block, 4),
    "deco_dequantize": lambda: dq.deco_dequantize(qm),
    "fused_matmul_t": lambda: dq.fused_matmul_t(q, qm),
    "fused_matmul": lambda: dq.fused_matmul(rng.standard_normal((1, 2048)).astype(np.float32), qm),
    "attention_scores": lambda: cache.attention_scores(0, q[0]),
}
n = int(os.environ.get("REPS", 10))
for name, fn in calls.items():
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{name:18s} {(time.perf_counter() - t0) / n * 1e6:9.1f} us per call")

#!/usr/bin/env python
"""Split the outlier-data attention error into write-path (code flips) and read-path parts."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dquant_oracle as O  # noqa: E402
from paper_2405_12591_b200.attention import DecodeKvCache  # noqa: E402


def enc_from_seg(seg):
    core0, qt = seg.local_tensors
    p = O.Plan2.of(seg.rows, seg.cols)
    codes = O.unpack_codes(qt.payload, qt.count, qt.bits).reshape(p.r, p.i2, p.j2)
    return O.Encoded(p, qt.bits, core0.detach().cpu().numpy().astype(np.float32), np.float32(qt.scale), codes)


for scale in (1.0, 5.0, 20.0, 50.0):
    rng = np.random.default_rng(1)
    T, units = 4096, 2
    k = rng.standard_normal((units, T, 128)).astype(np.float32)
    k[:, :, [3, 77]] *= scale
    k = k.astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, 1, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=1, bits=4)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    for u in range(units):
        ours_k, ours_v = enc_from_seg(cache.export_segment(0, 0, u, "k")), enc_from_seg(cache.export_segment(0, 0, u, "v"))
        ref_k, ref_v = O.encode(k[u].astype(np.float32), 4), O.encode(v[u].astype(np.float32), 4)
        r = ref_k.codes.reshape(ref_k.r, -1).astype(np.int32)
        g = ours_k.codes.reshape(ours_k.r, -1).astype(np.int32)
        s = np.where((r * g).sum(1) < 0, -1, 1)[:, None]
        flips = int((g * s != r).sum())
        lay_ref = O.LayerOracle(128, 4, 1 << 30)
        lay_ref.k_segs, lay_ref.v_segs, lay_ref.rows = [ref_k], [ref_v], [T]
        lay_ours = O.LayerOracle(128, 4, 1 << 30)
        lay_ours.k_segs, lay_ours.v_segs, lay_ours.rows = [ours_k], [ours_v], [T]
        qq = q[u].astype(np.float32)
        a_ref, a_ours = lay_ref.attend(qq).astype(np.float64), lay_ours.attend(qq).astype(np.float64)
        e_total = np.linalg.norm(a_ref - out[u]) / np.linalg.norm(a_ref)
        e_read = np.linalg.norm(a_ours - out[u]) / np.linalg.norm(a_ours)
        e_write = np.linalg.norm(a_ref - a_ours) / np.linalg.norm(a_ref)
        print(f"scale={scale:5.1f} u={u} k-code flips={flips:4d}  total={e_total:.2e} read-path={e_read:.2e} "
              f"write-path={e_write:.2e}", flush=True)

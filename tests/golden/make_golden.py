"""Generate golden vectors by running the REFERENCE ``dquant`` package.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports the reference read-only from ``/root/reference/pkg/src`` and writes
``tests/golden/golden.npz`` (+ ``golden_meta.json``).  The GPU box never runs
this script; the committed fixtures travel instead.  Inputs are seeded and
rounded to fp16 where the device path would see fp16, so both sides see
identical values.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    import dquant
    from dquant import compress, kvcache, mpo, quantize

    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"reference": REF, "numpy": np.__version__}

    # ---- codec: quantize_rtn (quantize.py:123-151) on the reference's own test inputs
    for bits in (2, 4, 8):
        rng = np.random.default_rng(bits)  # test_quantize.py:52-55
        t = (rng.standard_normal(2000) * rng.choice([0.1, 1, 30], 2000)).astype(np.float32)
        q = quantize.quantize_rtn(t, bits)
        arrays[f"rtn{bits}_t"] = t
        arrays[f"rtn{bits}_scale"] = np.float32(q.scale)
        arrays[f"rtn{bits}_payload"] = np.frombuffer(q.payload, np.uint8)
        # pack of random in-range codes, odd count to exercise the padded last byte
        qm = (1 << (bits - 1)) - 1
        codes = np.random.default_rng(100 + bits).integers(-qm, qm + 1, size=101)
        arrays[f"pack{bits}_codes"] = codes.astype(np.int8)
        arrays[f"pack{bits}_payload"] = np.frombuffer(quantize.pack(codes.tolist(), bits), np.uint8)
    q = quantize.quantize_rtn(np.array([[1, -2], [3, -4]], np.float32), 4)
    arrays["worked_scale"] = np.float32(q.scale)
    arrays["worked_payload"] = np.frombuffer(q.payload, np.uint8)

    # ---- planner (mpo.py:73-96) and bond law (mpo.py:54-63)
    plans = []
    for rows, cols, n in [(4096, 4096, 2), (7, 16, 2), (1, 1, 2), (4096, 4096, 3), (512, 512, 4),
                          (96, 100, 2), (97, 31, 3), (1024, 6, 4), (2048, 128, 2), (1009, 128, 2),
                          (1023, 128, 2), (8, 128, 2), (4, 128, 2), (16384, 128, 2), (37, 41, 2)]:
        p = mpo.plan_shapes(rows, cols, n)
        plans.append([rows, cols, n, list(p.i_factors), list(p.j_factors), list(p.bond_dims())])
    meta["plans"] = plans

    # ---- DecoQuant blocks (compress.py:85-107, mpo.py:153-198)
    blocks = {}
    rng = np.random.default_rng(0)
    blocks["c1h0"] = (rng.standard_normal((2048, 128)).astype(np.float16).astype(np.float32), 4)
    blocks["out512"] = (dquant.synth_activations(512, 128, outlier_cols=4, outlier_scale=20.0, seed=3)
                        .astype(np.float16).astype(np.float32), 4)
    def h16(seed, shape):
        return np.random.default_rng(seed).standard_normal(shape).astype(np.float16).astype(np.float32)

    blocks["b2_256"] = (h16(5, (256, 128)), 2)
    blocks["b8_256"] = (h16(6, (256, 128)), 8)
    blocks["odd1009"] = (h16(7, (1009, 128)), 4)
    blocks["r1023"] = (h16(8, (1023, 128)), 4)
    blocks["tiny8"] = (h16(9, (8, 128)), 4)
    blocks["s37x41"] = (h16(10, (37, 41)), 4)
    blocks["s64x48"] = (h16(11, (64, 48)), 4)
    blocks["d64_512"] = (h16(12, (512, 64)), 4)
    meta["blocks"] = {}
    for name, (m, bits) in blocks.items():
        plan = mpo.plan_shapes(*m.shape, 2)
        chain = mpo.decompose(m, plan)
        qm = compress.deco_quantize(m, bits)
        qt = qm.local_tensors[1]
        rec = compress.deco_dequantize(qm)
        rep = compress.compression_report(qm)
        rng_x = np.random.default_rng(1000 + len(name))
        x_t = rng_x.standard_normal((3, m.shape[1])).astype(np.float32)
        x = rng_x.standard_normal((3, m.shape[0])).astype(np.float32)
        arrays[f"{name}_m"] = m.astype(np.float16)  # exact: every input is fp16-rounded
        arrays[f"{name}_core0"] = chain.local_tensors[0]
        arrays[f"{name}_core1"] = chain.local_tensors[1]
        arrays[f"{name}_scale"] = np.float32(qt.scale)
        arrays[f"{name}_payload"] = np.frombuffer(qt.payload, np.uint8)
        if m.size <= 256 * 128:
            arrays[f"{name}_rec"] = rec
        else:  # large blocks: keep a checksum row set instead of the whole matrix
            arrays[f"{name}_rec_rows"] = rec[::97]
        arrays[f"{name}_xt"] = x_t
        arrays[f"{name}_mmt"] = compress.fused_matmul_t(x_t, qm)
        arrays[f"{name}_x"] = x
        arrays[f"{name}_mm"] = compress.fused_matmul(x, qm)
        meta["blocks"][name] = {
            "bits": bits,
            "shape": list(m.shape),
            "i": list(plan.i_factors),
            "j": list(plan.j_factors),
            "ratio": rep.ratio,
            "bytes_original": rep.bytes_original,
            "bytes_compressed": rep.bytes_compressed,
        }

    # ---- the reference's outlier matrix (test_compress.py:47-53) and its errors
    sm = dquant.synth_activations(256, 256, outlier_cols=8, outlier_scale=20.0, seed=11)
    arrays["synth256"] = sm
    rec = compress.deco_dequantize(compress.deco_quantize(sm, 4))
    direct = quantize.dequantize(quantize.quantize_rtn(sm, 4))
    meta["synth256"] = {
        "deco_err": float(np.linalg.norm(sm.astype(np.float64) - rec) / np.linalg.norm(sm)),
        "direct_err": float(np.linalg.norm(sm.astype(np.float64) - direct) / np.linalg.norm(sm)),
    }

    # ---- KV cache lifecycle (kvcache.py:94-225)
    cfg = kvcache.CacheConfig(layers=2, dim=128, bits=4, chunk_len=32)
    cache = kvcache.KvCache(cfg)
    rng = np.random.default_rng(21)
    pk = rng.standard_normal((100, 128)).astype(np.float32)
    pv = rng.standard_normal((100, 128)).astype(np.float32)
    cache.prefill(0, pk, pv)
    ak = rng.standard_normal((70, 128)).astype(np.float32)
    av = rng.standard_normal((70, 128)).astype(np.float32)
    for t in range(70):
        cache.append_token(0, ak[t], av[t])
    qrow = rng.standard_normal(128).astype(np.float32)
    arrays["kv_prefill_k"], arrays["kv_prefill_v"] = pk, pv
    arrays["kv_append_k"], arrays["kv_append_v"] = ak, av
    arrays["kv_q"] = qrow
    arrays["kv_scores"] = cache.attention_scores(0, qrow)
    arrays["kv_keys"] = cache.read_keys(0)
    arrays["kv_values"] = cache.read_values(0)
    led = cache.ledger()
    meta["kv"] = {
        "segments": len(cache.layers[0].key_segments),
        "tail_len": cache.layers[0].tail_len,
        "bytes_fp16_equivalent": led.bytes_fp16_equivalent,
        "bytes_actual": led.bytes_actual,
    }

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()

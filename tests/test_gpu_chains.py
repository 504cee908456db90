"""Chains longer than 2 on the device: decompose, deco_quantize / dequantize,
fused reads and compression_report for n = 3, 4 against the reference's outputs
(tests/golden/golden_chains.*) and the oracle; the KV-cache mirror with CacheConfig(n=3)."""

import json
import os

import numpy as np
import pytest

from oracle import dquant_oracle as O

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gold():
    g = np.load(os.path.join(HERE, "golden", "golden_chains.npz"))
    with open(os.path.join(HERE, "golden", "golden_chains.json")) as f:
        return g, json.load(f)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30))


def test_chain_decompose_and_deco_quantize(gold):
    import paper_2405_12591_b200 as dq

    g, meta = gold
    for key, case in meta["cases"].items():
        name, n = key.rsplit("_n", 1)[0], int(key.rsplit("_n", 1)[1])
        m = g[f"{name}_m"]
        plan = dq.plan_shapes(*m.shape, n)
        chain = dq.decompose(m, plan)
        assert list(chain.bond_dims) == case["bonds"]
        assert rel(g[f"{key}_rec"], dq.reconstruct(chain)) < 1e-5, key
        # factors vs the oracle's LAPACK ones, sign-invariantly per bond: a middle
        # core carries the flips of its left bond (the previous core's) and of its right bond
        ref = O.tt_split(m, plan.i_factors, plan.j_factors)
        left = np.ones(1)
        for c, r in zip(chain.local_tensors, ref):
            cm = c.reshape(c.shape[0], -1, c.shape[3]).astype(np.float64) * left[:, None, None]
            rm = r.reshape(r.shape[0], -1, r.shape[3]).astype(np.float64)
            right = np.sign(np.einsum("abc,abc->c", cm, rm))
            right[right == 0] = 1
            assert rel(rm, cm * right) < 1e-5, key
            left = right
        for bits in (4, 2):
            q = dq.deco_quantize(m, bits, n)
            kb = f"{key}_b{bits}"
            got = [t.scale for t in q.quantized_locals]
            assert got == pytest.approx(case["bits"][str(bits)]["scales"], rel=1e-6), kb
            assert rel(g[f"{kb}_deq"], dq.deco_dequantize(q)) < 1e-3, kb
            meter = dq.WorkingSetMeter()
            assert rel(g[f"{kb}_mm"], dq.fused_matmul(g[f"{key}_x"], q, meter)) < 1e-3, kb
            from paper_2405_12591_b200.compress import TILE_ELEMENTS

            assert 0 < meter.peak_elements <= TILE_ELEMENTS
            assert rel(g[f"{kb}_mmt"], dq.fused_matmul_t(g[f"{key}_xt"], q)) < 1e-3, kb
            rep = dq.compression_report(q)
            assert rep.bytes_compressed == case["bits"][str(bits)]["bytes_compressed"]
            assert rep.ratio == pytest.approx(case["bits"][str(bits)]["ratio"], rel=1e-12)


def test_kvcache_mirror_with_three_core_chains():
    """CacheConfig(n=3): segments compressed as 3-core chains, scores through the chain sweep."""
    import paper_2405_12591_b200 as dq

    rng = np.random.default_rng(3)
    k = rng.standard_normal((600, 64)).astype(np.float32)
    v = rng.standard_normal((600, 64)).astype(np.float32)
    cache = dq.KvCache(dq.CacheConfig(layers=1, dim=64, bits=4, chunk_len=256, n=3))
    cache.prefill(0, k[:512], v[:512])
    for t in range(512, 600):
        cache.append_token(0, k[t], v[t])
    q = rng.standard_normal(64).astype(np.float32)
    scores = cache.attention_scores(0, q)
    _, _, deq = O.deco_chain(k[:512], 4, 3)
    ref = np.concatenate([O.chain_matmul_t(q[None], deq)[0], q @ k[512:600].T]) / np.float32(np.sqrt(64))
    assert rel(ref, scores.ravel()) < 1e-3
    assert rel(v[:512], cache.read_values(0)[:512]) < 0.3  # int4 chains: coarse, but the right rows

"""The opt-in per-channel asymmetric mode (north_star "per-channel asymmetric int4/int2";
SURVEY.md 8f f4).  It is not in the reference (whose quantizer is per-tensor symmetric), so its
parity is pinned against the oracle's restatement (oracle.rtn_asym / encode_asym), not the
reference: codes and channel tables bit-exact from the same core1, attention within 1e-3."""

import numpy as np
import pytest
import torch

from oracle import dquant_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-3


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30))


@pytest.mark.parametrize("bits,T", [(4, 2048), (2, 1024), (4, 1009), (4, 24)])
def test_asym_codes_and_channels_bit_exact(bits, T):
    from paper_2405_12591_b200 import _lib
    from paper_2405_12591_b200.compress import deco_quantize_asym_batched
    from paper_2405_12591_b200.mpo import decompose_batched

    rng = np.random.default_rng(T + bits)
    k = rng.standard_normal((3, T, 128)).astype(np.float32)
    k[:, :, [5, 40]] *= 20.0
    kd = torch.from_numpy(k).cuda()
    _, core1, p = decompose_batched(kd)
    res = deco_quantize_asym_batched(kd, bits, _lib.LAYOUT_REF)
    for u in range(3):
        c1 = core1[u].cpu().numpy().reshape(p.r, p.i2, p.j2)
        s, z, codes = O.rtn_asym(c1, bits)
        ch = res["channels"][u].cpu().numpy()
        assert np.array_equal(ch[0], s) and np.array_equal(ch[1], z.astype(np.float32))
        got = O.unpack_codes(res["payload"][u].cpu().numpy().tobytes(), c1.size, bits) & ((1 << bits) - 1)
        assert np.array_equal(got.reshape(c1.shape), codes.astype(got.dtype))


@pytest.mark.parametrize("bits,g,T,units,scale", [(4, 1, 4096, 3, 20.0), (2, 1, 8192, 2, 20.0), (4, 2, 2048, 2, 1.0),
                                                  (4, 1, 1009, 2, 50.0), (2, 2, 600, 2, 1.0)])
def test_asym_attention_matches_oracle(bits, g, T, units, scale):
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(3 * T + bits + g)
    k = rng.standard_normal((units, T, 128)).astype(np.float32)
    k[:, :, [3, 77]] *= scale
    k = k.astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, g, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=g, bits=bits, asym=True)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    assert cache._layers[0].args.asym == 1 and cache._layers[0].args.path == 0
    for u in range(units):
        lay = O.LayerOracle(128, bits, 1 << 30, asym=True)
        lay.prefill(k[u].astype(np.float32), v[u].astype(np.float32))
        ref = lay.attend(q[u].astype(np.float32))
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


def test_asym_segments_tail_and_append():
    """prefill + sealed chunks + fp16 tail with the fused append, asymmetric segments."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    units, chunk, P, steps = 2, 256, 700, 300
    rng = np.random.default_rng(12)
    k = rng.standard_normal((units, P + steps, 128)).astype(np.float32)
    k[:, :, [9]] *= 30.0
    k = k.astype(np.float16)
    v = rng.standard_normal((units, P + steps, 128)).astype(np.float16)
    q = rng.standard_normal((units, 1, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=1, bits=4, chunk_len=chunk, asym=True)
    kd, vd, qd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(q).cuda()
    cache.prefill(0, kd[:, :P], vd[:, :P])
    for t in range(P, P + steps):
        cache.attend(0, qd, append=(kd[:, t], vd[:, t]))
    out = cache.attend(0, qd).float().cpu().numpy()
    for u in range(units):
        lay = O.LayerOracle(128, 4, chunk, asym=True)
        lay.prefill(k[u, :P].astype(np.float32), v[u, :P].astype(np.float32))
        for t in range(P, P + steps):
            lay.append(k[u, t].astype(np.float32), v[u, t].astype(np.float32))
        assert rel(lay.attend(q[u].astype(np.float32)), out[u]) < TOL


def test_asym_beats_symmetric_on_outlier_channels():
    """The point of the mode: with outlier key channels the per-channel codes track the exact
    attention far better than the reference's per-tensor scale (measured, recorded in DESIGN)."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(8)
    units, T = 4, 4096
    k = rng.standard_normal((units, T, 128)).astype(np.float32)
    k[:, :, [3, 77]] *= 20.0
    k = k.astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, 1, 128)).astype(np.float16)
    errs = {}
    for asym in (False, True):
        cache = DecodeKvCache(layers=1, units=units, g=1, bits=4, asym=asym)
        cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
        out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
        e = []
        for u in range(units):
            s = q[u].astype(np.float64) @ k[u].astype(np.float64).T / np.sqrt(128)
            p = np.exp(s - s.max())
            p /= p.sum()
            e.append(rel(p @ v[u].astype(np.float64), out[u]))
        errs[asym] = float(np.median(e))
    print("median relative error vs exact attention: symmetric", errs[False], "asymmetric", errs[True])
    assert errs[True] < 0.5 * errs[False]

"""K3 (batched fp64 TT-SVD + quantize) and K4 (reconstruct) against the reference goldens.

SVD factors are compared sign-invariantly: each bond index r may flip sign
between LAPACK and the Jacobi kernel; flipping row r of core1 negates exactly
that row's codes (the symmetric quantizer is odd), so after per-r alignment the
codes must be identical.
"""

import numpy as np
import pytest
import torch

from oracle import dquant_oracle as O

pytestmark = pytest.mark.gpu

BLOCKS = ["c1h0", "out512", "b2_256", "b8_256", "odd1009", "r1023", "tiny8", "s37x41", "s64x48", "d64_512"]


@pytest.fixture(scope="module")
def dq():
    import paper_2405_12591_b200 as dq

    return dq


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30))


def signs(ref_core1, got_core1):
    """per bond index: +1/-1 aligning got to ref"""
    r = ref_core1.shape[0]
    dots = (ref_core1.reshape(r, -1).astype(np.float64) * got_core1.reshape(r, -1).astype(np.float64)).sum(1)
    return np.where(dots < 0, -1.0, 1.0)


@pytest.mark.parametrize("name", BLOCKS)
def test_decompose_matches_reference(golden, dq, name):
    g, meta = golden
    m = g[f"{name}_m"].astype(np.float32)
    chain = dq.decompose(m, dq.plan_shapes(*m.shape, 2))
    c0, c1 = chain.local_tensors
    r0, r1 = g[f"{name}_core0"], g[f"{name}_core1"]
    assert c0.shape == r0.shape and c1.shape == r1.shape
    s = signs(r1, c1)
    assert rel(r1, c1 * s[:, None, None, None]) < 1e-5
    assert rel(r0, c0 * s[None, None, None, :]) < 1e-5
    assert rel(m, dq.reconstruct(chain)) < 1e-5


@pytest.mark.parametrize("name", BLOCKS)
def test_deco_quantize_codes_bit_exact(golden, dq, name):
    g, meta = golden
    info = meta["blocks"][name]
    bits = info["bits"]
    m = g[f"{name}_m"].astype(np.float32)
    q = dq.deco_quantize(m, bits)
    qt = q.local_tensors[1]
    assert np.float32(qt.scale).tobytes() == g[f"{name}_scale"].tobytes()
    r = qt.shape[0]
    ref_codes = O.unpack_codes(g[f"{name}_payload"].tobytes(), qt.count, bits).reshape(r, -1)
    got_codes = qt.codes().reshape(r, -1)
    s = signs(g[f"{name}_core1"], O.dequant(got_codes, qt.scale))
    np.testing.assert_array_equal(got_codes * s[:, None].astype(np.int8), ref_codes)
    # reconstruction vs the reference's dequantized matrix (north_star: <= 1e-3)
    rec = dq.deco_dequantize(q)
    if f"{name}_rec" in g:
        assert rel(g[f"{name}_rec"], rec) < 1e-5
    else:
        assert rel(g[f"{name}_rec_rows"], rec[::97]) < 1e-5
    rep = dq.compression_report(q)
    assert rep.ratio == pytest.approx(info["ratio"], abs=1e-15)
    assert rep.bytes_compressed == info["bytes_compressed"]


def test_c1_batched_32_heads(dq):
    """C1: 32 heads x 2048 x 128, int4: batched kernel vs the oracle, head by head."""
    from paper_2405_12591_b200.compress import deco_quantize_batched

    rng = np.random.default_rng(0)
    k = rng.standard_normal((32, 2048, 128)).astype(np.float16)
    res = deco_quantize_batched(torch.from_numpy(k).cuda(), 4)
    assert int(res["flags"].item()) == 0
    payload = res["payload"].cpu().numpy()
    scales = res["scale"].cpu().numpy()
    core0 = res["core0"].cpu().numpy()
    p = O.Plan2.of(2048, 128)
    flips = 0
    for h in range(32):
        enc = O.encode(k[h].astype(np.float32), 4)
        assert np.float32(scales[h]) == enc.scale
        got = O.unpack_codes(payload[h].tobytes(), enc.codes.size, 4).reshape(p.r, -1)
        ref = enc.codes.reshape(p.r, -1)
        s = np.where((got.astype(np.int32) * ref).sum(1) < 0, -1, 1).astype(np.int8)
        flips += int((got * s[:, None] != ref).sum())
        genc = O.Encoded(p, 4, core0[h] * s[None, None, None, :].astype(np.float32), scales[h],
                         (got * s[:, None]).reshape(p.r, p.i2, p.j2))
        assert rel(O.decode(enc), O.decode(genc)) < 1e-3
    assert flips == 0


def test_fp16_input_equals_fp32_input(dq):
    from paper_2405_12591_b200.compress import deco_quantize_batched

    rng = np.random.default_rng(3)
    k = rng.standard_normal((4, 1024, 128)).astype(np.float16)
    a = deco_quantize_batched(torch.from_numpy(k).cuda(), 4)
    b = deco_quantize_batched(torch.from_numpy(k.astype(np.float32)).cuda(), 4)
    assert torch.equal(a["payload"], b["payload"]) and torch.equal(a["scale"], b["scale"])


def test_degenerate_inputs(dq):
    z = dq.deco_quantize(np.zeros((16, 16), np.float32), 4)
    assert not z.local_tensors[1].codes().any()
    np.testing.assert_array_equal(dq.deco_dequantize(z), np.zeros((16, 16)))
    chain = dq.decompose(np.zeros((16, 16), np.float32), dq.plan_shapes(16, 16, 2))
    for c in chain.local_tensors:
        assert not np.asarray(c).any()
    u = np.random.default_rng(1).standard_normal((64, 1)).astype(np.float32)
    v = np.random.default_rng(2).standard_normal((1, 48)).astype(np.float32)
    m = (u @ v).astype(np.float32)
    assert rel(m, dq.reconstruct(dq.decompose(m, dq.plan_shapes(64, 48, 2)))) < 1e-5
    eye = np.eye(64, dtype=np.float32)
    assert rel(eye, dq.deco_dequantize(dq.deco_quantize(eye, 8))) < 1e-2
    m4 = np.eye(4, dtype=np.float32)
    assert rel(m4, dq.reconstruct(dq.decompose(m4, dq.ShapePlan((2, 2), (2, 2))))) < 1e-6


def test_nonfinite_raises_like_reference(dq):
    from paper_2405_12591_b200.errors import NonFiniteInput

    m = np.random.default_rng(0).standard_normal((64, 64)).astype(np.float32)
    m[3, 5] = np.nan
    with pytest.raises(NonFiniteInput):
        dq.deco_quantize(m, 4)
    with pytest.raises(np.linalg.LinAlgError):
        dq.deco_quantize(m, 4)


def test_reference_compress_properties(golden, dq):
    """test_compress.py:47-76 ported: outlier matrix beats RTN; determinism; shapes."""
    g, meta = golden
    m = g["synth256"]  # the reference's synth_activations(256, 256, 8, 20.0, seed=11)
    deco = rel(m, dq.deco_dequantize(dq.deco_quantize(m, 4)))
    assert deco == pytest.approx(meta["synth256"]["deco_err"], rel=1e-3)
    assert deco < meta["synth256"]["direct_err"]
    direct = rel(m, dq.dequantize(dq.quantize_rtn(m, 4)))
    assert direct == pytest.approx(meta["synth256"]["direct_err"], rel=1e-6)
    a, b = dq.deco_quantize(m, 4), dq.deco_quantize(m, 4)
    assert a.local_tensors[1].payload == b.local_tensors[1].payload
    for shape in [(24, 56), (37, 41), (128, 64)]:
        x = np.random.default_rng(sum(shape)).standard_normal(shape).astype(np.float32)
        assert dq.deco_dequantize(dq.deco_quantize(x, 4)).shape == shape

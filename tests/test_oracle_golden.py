"""Pin the CPU oracle (oracle/dquant_oracle.py) to vectors produced by the reference itself.

The fixtures come from tests/golden/make_golden.py, which imports the reference
``dquant`` package.  Bytes, codes, scales and plans must match exactly; float
outputs must match to round-off.
"""

import numpy as np
import pytest

from oracle import dquant_oracle as O


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30))


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_rtn_bit_exact(golden, bits):
    g, _ = golden
    scale, codes = O.rtn(g[f"rtn{bits}_t"], bits)
    assert np.float32(scale).tobytes() == g[f"rtn{bits}_scale"].tobytes()
    assert O.pack_codes(codes, bits).tobytes() == g[f"rtn{bits}_payload"].tobytes()


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_pack_unpack_bit_exact(golden, bits):
    g, _ = golden
    codes = g[f"pack{bits}_codes"]
    payload = O.pack_codes(codes, bits)
    assert payload.tobytes() == g[f"pack{bits}_payload"].tobytes()
    np.testing.assert_array_equal(O.unpack_codes(payload, codes.size, bits), codes)
    # unpack_range semantics (quantize.py:95-109)
    for start, count in [(0, 7), (3, 11), (50, 51), (97, 4)]:
        np.testing.assert_array_equal(O.unpack_codes(payload, count, bits, start), codes[start:start + count])


def test_reference_pack_goldens():
    # test_quantize.py:111-118 and test_formats.py golden bytes
    assert O.pack_codes([1, -1], 4).tobytes() == b"\xf1"
    assert O.pack_codes([-7], 8).tobytes() == b"\xf9"
    assert O.pack_codes([1, 0, -1, 1], 2).tobytes() == bytes([0b01_11_00_01])
    assert O.pack_codes([1, -1, 7, -7], 4).tobytes() == b"\xf1\x97"


def test_worked_example(golden):
    g, _ = golden
    scale, codes = O.rtn(np.array([[1, -2], [3, -4]], np.float32), 4)
    assert codes.tolist() == [[2, -4], [5, -7]]
    assert np.float32(scale) == g["worked_scale"]


def test_plans(golden):
    _, meta = golden
    for rows, cols, n, i_f, j_f, bd in meta["plans"]:
        pi, pj = O.plan(rows, cols, n)
        assert list(pi) == i_f and list(pj) == j_f
        assert list(O.bonds(pi, pj)) == bd


def _blocks(meta):
    return sorted(meta["blocks"])


@pytest.mark.parametrize("name", ["c1h0", "out512", "b2_256", "b8_256", "odd1009", "r1023", "tiny8",
                                  "s37x41", "s64x48", "d64_512"])
def test_blocks_match_reference(golden, name):
    g, meta = golden
    info = meta["blocks"][name]
    m = g[f"{name}_m"].astype(np.float32)
    bits = info["bits"]
    p = O.Plan2.of(*m.shape)
    assert [p.i1, p.i2] == info["i"] and [p.j1, p.j2] == info["j"]
    core0, core1, _ = O.tt_split2(m, p)
    # same LAPACK routine: cores agree to round-off (bit-identical on the generating host)
    assert rel(g[f"{name}_core0"], core0) < 1e-5
    assert rel(g[f"{name}_core1"], core1) < 1e-5
    # codec on the reference's own core1: bit-exact
    scale, codes = O.rtn(g[f"{name}_core1"], bits)
    assert np.float32(scale).tobytes() == g[f"{name}_scale"].tobytes()
    assert O.pack_codes(codes, bits).tobytes() == g[f"{name}_payload"].tobytes()
    enc = O.Encoded(p, bits, g[f"{name}_core0"], np.float32(scale), codes.reshape(-1, p.i2, p.j2))
    rec = O.decode(enc)
    if f"{name}_rec" in g:
        assert rel(g[f"{name}_rec"], rec) < 1e-6
    else:
        assert rel(g[f"{name}_rec_rows"], rec[::97]) < 1e-6
    assert rel(g[f"{name}_mmt"], O.matmul_t(g[f"{name}_xt"], enc)) < 1e-6
    assert rel(g[f"{name}_mm"], O.matmul(g[f"{name}_x"], enc)) < 1e-6
    mu, b_orig, b_comp = O.ratio_report(enc)
    assert mu == pytest.approx(info["ratio"], abs=1e-15)
    assert (b_orig, b_comp) == (info["bytes_original"], info["bytes_compressed"])


def test_kvcache_lifecycle(golden):
    g, meta = golden
    lay = O.LayerOracle(128, 4, 32)
    lay.prefill(g["kv_prefill_k"], g["kv_prefill_v"])
    for t in range(70):
        lay.append(g["kv_append_k"][t], g["kv_append_v"][t])
    assert len(lay.k_segs) == meta["kv"]["segments"]
    assert len(lay.tail_k) == meta["kv"]["tail_len"]
    assert lay.ledger() == (meta["kv"]["bytes_fp16_equivalent"], meta["kv"]["bytes_actual"])
    # the oracle re-runs the SVD; scores agree to round-off with the reference's
    assert rel(g["kv_scores"], lay.scores(g["kv_q"])) < 1e-5
    assert rel(g["kv_keys"], lay.read("k")) < 1e-5
    assert rel(g["kv_values"], lay.read("v")) < 1e-5


def test_attention_composition_sane():
    rng = np.random.default_rng(0)
    k = rng.standard_normal((64, 128)).astype(np.float32)
    v = rng.standard_normal((64, 128)).astype(np.float32)
    q = rng.standard_normal((2, 128)).astype(np.float32)
    lay = O.LayerOracle(128, None, 1024)
    lay.prefill(k, v)
    s = q.astype(np.float64) @ k.T.astype(np.float64) / np.sqrt(128)
    p = np.exp(s - s.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    assert rel(p @ v, lay.attend(q)) < 1e-6


def test_oracle_rtn_float64_golden():
    """float64 inputs (ties 1 ulp away, values beyond the fp32 range, subnormals) against the
    reference's own quantize_rtn (tests/golden/make_golden_f64.py)."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_f64.npz"))
    names = sorted({k[:-2] for k in g.files if k.endswith("_t")})
    assert len(names) >= 5
    with np.errstate(over="ignore"):
        for n in names:
            for bits in (2, 4, 8):
                s, c = O.rtn(g[n + "_t"], bits)
                assert np.float32(s).tobytes() == g[f"{n}_{bits}_scale"].tobytes(), (n, bits)
                assert O.pack_codes(c.reshape(-1), bits).tobytes() == g[f"{n}_{bits}_payload"].tobytes(), (n, bits)

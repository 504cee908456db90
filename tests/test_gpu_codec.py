"""K1/K2 on the GPU: bit-exact against the reference's golden bytes (quantize.py:66-157)."""

import numpy as np
import pytest
import torch

from oracle import dquant_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dq():
    import paper_2405_12591_b200 as dq

    return dq


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quantize_rtn_golden(golden, dq, bits):
    g, _ = golden
    q = dq.quantize_rtn(g[f"rtn{bits}_t"], bits)
    assert np.float32(q.scale).tobytes() == g[f"rtn{bits}_scale"].tobytes()
    assert q.payload == g[f"rtn{bits}_payload"].tobytes()


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_pack_unpack_golden(golden, dq, bits):
    g, _ = golden
    codes = g[f"pack{bits}_codes"]
    assert dq.pack(codes.tolist(), bits) == g[f"pack{bits}_payload"].tobytes()
    np.testing.assert_array_equal(dq.unpack(g[f"pack{bits}_payload"].tobytes(), codes.size, bits), codes)
    from paper_2405_12591_b200.quantize import unpack_range

    payload = g[f"pack{bits}_payload"].tobytes()
    for start, count in [(0, 7), (3, 11), (50, 51), (97, 4), (0, 101)]:
        np.testing.assert_array_equal(unpack_range(payload, start, count, bits), codes[start:start + count])


def test_reference_pack_goldens(dq):
    assert dq.pack([1, -1], 4) == b"\xf1"
    assert dq.pack([-7], 8) == b"\xf9"
    assert dq.pack([1, 0, -1, 1], 2) == bytes([0b01_11_00_01])
    assert dq.pack([1, -1, 7, -7], 4) == b"\xf1\x97"
    for a in range(-7, 8):
        for b in range(-7, 8):
            assert dq.unpack(dq.pack([a, b], 4), 2, 4).tolist() == [a, b]


def test_worked_example_and_edges(dq):
    q = dq.quantize_rtn(np.array([[1, -2], [3, -4]], np.float32), 4)
    assert q.scale == pytest.approx(4 / 7)
    np.testing.assert_array_equal(q.codes().reshape(2, 2), [[2, -4], [5, -7]])
    z = dq.quantize_rtn(np.zeros((3, 3), np.float32), 8)
    assert z.scale == 1.0 and not z.codes().any()
    m = dq.quantize_rtn(np.array([[127.0]], np.float32), 8)
    assert m.scale == 1.0 and m.codes().tolist() == [127]
    np.testing.assert_array_equal(dq.dequantize(dq.quantize_rtn(np.zeros((2, 5), np.float32), 4)), 0)


def test_errors(dq):
    from paper_2405_12591_b200.errors import CorruptPayload, NonFiniteInput, RangeOverflow, UnsupportedBits

    with pytest.raises(UnsupportedBits):
        dq.quantize_rtn(np.ones(3, np.float32), 3)
    with pytest.raises(NonFiniteInput):
        dq.quantize_rtn(np.array([np.inf], np.float32), 8)
    with pytest.raises(RangeOverflow):
        dq.pack([8], 4)
    with pytest.raises(RangeOverflow):
        dq.pack([-8], 4)
    with pytest.raises(CorruptPayload):
        dq.unpack(b"\x00", 5, 4)
    with pytest.raises(RangeOverflow):
        dq.pack(torch.tensor([0, 9], dtype=torch.int8, device="cuda"), 4)


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_codec_matches_oracle_large(dq, bits):
    """Mixed-scale values incl. exact ties: GPU codes == oracle codes (1M elements)."""
    rng = np.random.default_rng(40 + bits)
    qm = (1 << (bits - 1)) - 1
    t = (rng.standard_normal(1 << 20) * rng.choice([1e-3, 1, 50], 1 << 20)).astype(np.float32)
    t[:64] = np.arange(-32, 32, dtype=np.float32) * (float(np.abs(t).max()) / qm / 2)  # x.5 ties
    scale, codes = O.rtn(t, bits)
    q = dq.quantize_rtn(t, bits)
    assert np.float32(q.scale) == scale
    assert q.payload == O.pack_codes(codes, bits).tobytes()
    # torch in -> torch out, same bytes
    qt = dq.quantize_rtn(torch.from_numpy(t).cuda(), bits)
    assert torch.equal(qt.data.cpu(), torch.from_numpy(O.pack_codes(codes, bits)))


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_requantize_reference_core1(golden, dq, bits):
    """Codec parity on the reference's own large core (SURVEY.md 8c recipe 1)."""
    g, meta = golden
    for name, info in meta["blocks"].items():
        if info["bits"] != bits:
            continue
        q = dq.quantize_rtn(g[f"{name}_core1"], bits)
        assert np.float32(q.scale).tobytes() == g[f"{name}_scale"].tobytes(), name
        assert q.payload == g[f"{name}_payload"].tobytes(), name


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quantize_rtn_float64_golden(dq, bits):
    """float64 input keeps the reference's fp64 arithmetic on the original values
    (quantize.py:131-145): near-tie values 1 ulp from a rounding boundary, values beyond the
    fp32 range, subnormal maxima -- bit-exact scale and payload."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_f64.npz"))
    names = sorted({k[:-2] for k in g.files if k.endswith("_t")})
    for n in names:
        t = g[n + "_t"]
        q = dq.quantize_rtn(t, bits)
        assert np.float32(q.scale).tobytes() == g[f"{n}_{bits}_scale"].tobytes(), n
        assert q.payload == g[f"{n}_{bits}_payload"].tobytes(), n
        qt = dq.quantize_rtn(torch.from_numpy(t).cuda(), bits)  # torch float64 CUDA input too
        assert qt.payload == q.payload
    # the advisor's example: 2.5 - 1e-12 rounds to 2 in fp64 and to 3 after an fp32 cast
    assert dq.unpack(dq.quantize_rtn(np.array([7.0, 2.5 - 1e-12]), 4).payload, 2, 4).tolist() == [7, 2]

"""DQT1 / DQZ1 byte parity with files the reference wrote (tests/golden/golden_formats.json):
read -> write reproduces them byte for byte, the device decode of a reference chain matches
the oracle, and chains exported from the device KV cache round-trip."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import dquant_oracle as O

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "golden_formats.json")) as f:
        return json.load(f)


def test_packed_tensor_bytes_match_reference(golden, tmp_path):
    from paper_2405_12591_b200 import QuantizedTensor, pack
    from paper_2405_12591_b200.formats import read_tensor, tensor_bytes, write_tensor

    g = golden["packed_tensor"]
    q = QuantizedTensor(tuple(g["shape"]), g["bits"], g["scale"], payload=pack(g["codes"], g["bits"]))
    assert tensor_bytes(q).hex() == g["file"]
    p = tmp_path / "q.dqt"
    write_tensor(p, q)
    back = read_tensor(p)
    assert back == q and list(back.codes()) == g["codes"]


@pytest.mark.parametrize("idx", range(4))
def test_reference_chain_roundtrip_and_decode(golden, idx, tmp_path):
    from paper_2405_12591_b200 import deco_dequantize
    from paper_2405_12591_b200.formats import mpo_bytes, parse_mpo, read_mpo

    g = golden["chains"][idx]
    data = bytes.fromhex(g["file"])
    q = parse_mpo(data)
    assert (q.rows, q.cols, q.bits) == (g["rows"], g["cols"], g["bits"])
    assert mpo_bytes(q) == data  # byte-exact re-serialisation
    p = tmp_path / "c.dqz"
    p.write_bytes(data)
    assert mpo_bytes(read_mpo(p)) == data
    # device decode (K4) of the reference's own cores vs the oracle contraction of them
    core0, qt = q.local_tensors
    pl = O.Plan2.of(g["rows"], g["cols"])
    enc = O.Encoded(plan=pl, bits=g["bits"], core0=np.asarray(core0, np.float32), scale=np.float32(qt.scale),
                    codes=qt.codes().reshape(pl.r, pl.i2, pl.j2))
    ref = O.decode(enc)
    got = deco_dequantize(q)
    assert float(np.linalg.norm(got - ref) / np.linalg.norm(ref)) < 1e-6


def test_device_cache_segment_export_roundtrip(tmp_path):
    from paper_2405_12591_b200.attention import DecodeKvCache
    from paper_2405_12591_b200.formats import read_mpo, write_mpo

    rng = np.random.default_rng(7)
    k = torch.from_numpy(rng.standard_normal((2, 1024, 128)).astype(np.float16)).cuda()
    cache = DecodeKvCache(layers=1, units=2, g=1, bits=4)
    cache.prefill(0, k, k)
    for which in ("k", "v"):
        seg = cache.export_segment(0, 0, 1, which)
        p = tmp_path / f"{which}.dqz"
        write_mpo(p, seg)
        back = read_mpo(p)
        assert back.local_tensors[1] == seg.local_tensors[1]
        c0 = seg.local_tensors[0]
        c0 = c0.cpu().numpy() if isinstance(c0, torch.Tensor) else np.asarray(c0)
        assert np.array_equal(np.asarray(back.local_tensors[0]), c0)

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


def _chain_from_oracle(e):
    """oracle Encoded (the reference's algorithm, pinned to its goldens) -> QuantizedMpo"""
    from paper_2405_12591_b200 import QuantizedMpo, QuantizedTensor, plan_shapes

    p = e.plan
    qt = QuantizedTensor((e.r, p.i2, p.j2, 1), e.bits, float(e.scale), payload=e.payload)
    return QuantizedMpo(plan=plan_shapes(p.i1 * p.i2, p.j1 * p.j2, 2), bits=e.bits, local_tensors=(e.core0, qt))


@pytest.mark.parametrize("T,bits", [(1024, 4), (1009, 2)])
def test_import_dqz1_chains_into_decode_cache(T, bits):
    """DQZ1 files (written from reference-algorithm chains) -> DecodeKvCache.import_segment ->
    fused decode attention, against the oracle over the same chains; plus export -> DQZ1 ->
    import round trip (identical attention output)."""
    from paper_2405_12591_b200.attention import DecodeKvCache
    from paper_2405_12591_b200.formats import mpo_bytes, parse_mpo

    units = 2
    rng = np.random.default_rng(T + bits)
    k = rng.standard_normal((units, T, 128)).astype(np.float16).astype(np.float32)
    v = rng.standard_normal((units, T, 128)).astype(np.float16).astype(np.float32)
    q = rng.standard_normal((units, 1, 128)).astype(np.float16)
    ek = [O.encode(k[u], bits) for u in range(units)]
    ev = [O.encode(v[u], bits) for u in range(units)]
    kq = [parse_mpo(mpo_bytes(_chain_from_oracle(e))) for e in ek]  # through the DQZ1 bytes
    vq = [parse_mpo(mpo_bytes(_chain_from_oracle(e))) for e in ev]
    cache = DecodeKvCache(layers=1, units=units, g=1, bits=bits)
    cache.import_segment(0, kq, vq)
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    for u in range(units):
        lay = O.LayerOracle(128, bits, 1 << 30)
        lay.k_segs.append(ek[u])
        lay.v_segs.append(ev[u])
        lay.rows.append(T)
        ref = lay.attend(q[u].astype(np.float32))
        assert np.linalg.norm(ref - out[u]) / np.linalg.norm(ref) < 1e-3
    # export -> bytes -> import into a second cache: the same segments, the same output
    kx = [parse_mpo(mpo_bytes(cache.export_segment(0, 0, u, "k"))) for u in range(units)]
    vx = [parse_mpo(mpo_bytes(cache.export_segment(0, 0, u, "v"))) for u in range(units)]
    assert all(mpo_bytes(a) == mpo_bytes(b) for a, b in zip(kx, kq))
    c2 = DecodeKvCache(layers=1, units=units, g=1, bits=bits)
    c2.import_segment(0, kx, vx)
    assert torch.equal(c2.attend(0, torch.from_numpy(q).cuda()), cache.attend(0, torch.from_numpy(q).cuda()))


def test_cli_quantize_dequantize(tmp_path):
    """cli quantize -> DQZ1 (reference bytes for the reference's chain), dequantize -> DQT1 within
    1e-3 of the oracle reconstruction; exit codes of the reference's cli.py (2 malformed, 3 bad
    parameters, 4 unknown subcommand)."""
    import json as _json
    import subprocess
    import sys

    from paper_2405_12591_b200.formats import read_tensor, write_tensor

    root = os.path.dirname(HERE)
    rng = np.random.default_rng(5)
    m = rng.standard_normal((512, 128)).astype(np.float16).astype(np.float32)
    write_tensor(tmp_path / "m.dqt", m)

    def run(*a):
        return subprocess.run([sys.executable, "-m", "paper_2405_12591_b200.cli", *a], capture_output=True,
                              text=True, cwd=root, timeout=300)

    r = run("quantize", "--input", str(tmp_path / "m.dqt"), "--bits", "4", "--out", str(tmp_path / "m.dqz"))
    assert r.returncode == 0, r.stderr
    summary = _json.loads(r.stdout)
    e = O.encode(m, 4)
    assert summary["bytes_compressed"] == O.ratio_report(e)[2] and summary["n"] == 2
    r = run("dequantize", "--input", str(tmp_path / "m.dqz"), "--out", str(tmp_path / "r.dqt"))
    assert r.returncode == 0, r.stderr
    rec = read_tensor(tmp_path / "r.dqt")
    ref = O.decode(e)
    assert np.linalg.norm(rec - ref) / np.linalg.norm(ref) < 1e-3
    assert run("quantize", "--input", str(tmp_path / "m.dqt"), "--bits", "3", "--out", "x").returncode == 3
    assert run("dequantize", "--input", str(tmp_path / "m.dqt"), "--out", "x").returncode == 2
    assert run("frobnicate").returncode == 4

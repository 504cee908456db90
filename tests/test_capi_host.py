"""CPU-only checks of the C-ABI library and the host-side logic (no kernels launched)."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import dquant_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2405_12591_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        from paper_2405_12591_b200.build import build

        build()
    return _lib


def header_symbols():
    text = open(os.path.join(ROOT, "include", "dquant_b200.h")).read()
    return sorted(set(re.findall(r"\b(dq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(L):
    lib = L.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), f"{name} declared in include/dquant_b200.h but not exported"
        assert name in L.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.dq_version() >= 10000


def test_plan_shapes_matches_reference(L, golden):
    from paper_2405_12591_b200 import plan_shapes

    _, meta = golden
    for rows, cols, n, i_f, j_f, bd in meta["plans"]:
        p = plan_shapes(rows, cols, n)
        assert list(p.i_factors) == i_f and list(p.j_factors) == j_f
        assert list(p.bond_dims()) == bd


def test_plan_errors(L):
    from paper_2405_12591_b200 import plan_shapes
    from paper_2405_12591_b200.errors import ShapeMismatch

    with pytest.raises(ShapeMismatch):
        plan_shapes(4, 4, 1)
    with pytest.raises(ShapeMismatch):
        plan_shapes(0, 4, 2)


def test_make_plan2_and_layout_bytes(L):
    for T in (8, 1009, 1023, 1024, 2048, 4096, 32768):
        p = L.plan2(T, 128)
        op = O.Plan2.of(T, 128)
        assert (p.i1, p.i2, p.j1, p.j2, p.r) == (op.i1, op.i2, op.j1, op.j2, op.r)
        for bits in (2, 4, 8):
            ref = L.layout_bytes(p, bits, L.LAYOUT_REF)
            assert ref == O.payload_bytes(p.r * p.i2 * p.j2, bits)
            i2p = -(-p.i2 // 64) * 64
            assert L.layout_bytes(p, bits, L.LAYOUT_KTILE) == p.r * i2p * 16 * bits // 8
            assert L.layout_bytes(p, bits, L.LAYOUT_VTILE) == p.r * i2p * 16 * bits // 8
    from paper_2405_12591_b200.errors import UnsupportedBits

    with pytest.raises(UnsupportedBits):
        L.layout_bytes(L.plan2(64, 128), 3, 0)


@pytest.mark.parametrize("chunk_b", [64, 128, 256])
def test_attention_work_plan(L, chunk_b):
    """dq_attention_plan (host): every 64-row tile of every segment is covered exactly once by
    items of <= chunk_b rows inside one segment; partial slots are grouped per unit."""
    from paper_2405_12591_b200.attention import plan_work

    segs = []
    units = 3
    for u in range(units):
        for T in (4096, 1024, 1009, 8):
            p = L.plan2(T, 128)
            s = L.Segment()
            s.T, s.i1, s.i2, s.r = T, p.i1, p.i2, p.r
            s.i2p = -(-p.i2 // 64) * 64
            s.unit = u
            segs.append(s)
    arr = (L.Segment * len(segs))(*segs)
    wp = plan_work(arr, len(segs), units, chunk_b)
    covered = {}
    for i in range(wp.nwork):
        s, b0, nt = wp.work[3 * i: 3 * i + 3]
        assert b0 % 64 == 0 and 1 <= nt <= chunk_b // 64
        covered.setdefault(s, []).extend(range(b0 // 64, b0 // 64 + nt))
    for s, seg in enumerate(segs):
        tiles = -(-seg.i2 // 64)
        assert sorted(covered[s]) == list(range(tiles))
        sizes = [wp.work[3 * i + 2] for i in range(wp.nwork) if wp.work[3 * i] == s]
        assert len(sizes) == -(-tiles // (chunk_b // 64)) and max(sizes) - min(sizes) <= 1
    assert wp.total_parts == wp.nwork
    assert sorted(wp.work_part) == list(range(wp.total_parts))
    for i in range(wp.nwork):
        u = segs[wp.work[3 * i]].unit
        assert wp.unit_part0[u] <= wp.work_part[i] < wp.unit_part0[u] + wp.unit_nparts[u]
    with pytest.raises(ValueError):  # DQ_ERR_INVALID_ARG: chunk_b not a multiple of 64
        plan_work(arr, len(segs), units, 100)


def test_struct_layouts(L):
    # sizes must match the C structs in include/dquant_b200.h
    assert ctypes.sizeof(L.Plan2) == 40
    assert ctypes.sizeof(L.Segment) == 6 * 8 + 2 * 4 + 8 * 4  # 4 + 2 (asymmetric channel tables) pointers
    assert L.AttnArgs.work.offset % 8 == 0


def test_host_mirror_types(L):
    from paper_2405_12591_b200 import CacheConfig, MpoChain, ShapePlan, split_large_small
    from paper_2405_12591_b200.errors import BondMismatch, CorruptPayload, ShapeMismatch, UnsupportedBits
    from paper_2405_12591_b200.quantize import QuantizedTensor, payload_size

    assert payload_size(101, 4) == 51
    chain = MpoChain((np.zeros((1, 8, 8, 64), np.float32), np.zeros((64, 512, 512, 1), np.float32)))
    large, small = split_large_small(chain)
    assert large.shape == (64, 512, 512, 1) and small.shape == (1, 8, 8, 64)
    with pytest.raises(BondMismatch):
        MpoChain((np.zeros((1, 2, 2, 3), np.float32), np.zeros((4, 2, 2, 1), np.float32)))
    with pytest.raises(ShapeMismatch):
        ShapePlan((2,), (2,))
    with pytest.raises(CorruptPayload):
        QuantizedTensor(shape=(2, 2), bits=4, scale=1.0, payload=b"\x00")
    with pytest.raises(UnsupportedBits):
        CacheConfig(layers=1, dim=8, bits=3)
    with pytest.raises(ShapeMismatch):
        CacheConfig(layers=0, dim=8)


def test_sharding_ranges():
    from paper_2405_12591_b200.sharding import kv_head_range, local_units

    assert kv_head_range(32, 0, 8) == (0, 4)
    assert kv_head_range(32, 7, 8) == (28, 32)
    assert kv_head_range(8, 3, 8) == (3, 4)
    units = [u for r in range(4) for u in local_units(2, 8, r, 4)]
    assert sorted(units) == [(b, h) for b in range(2) for h in range(8)]
    with pytest.raises(ValueError):
        kv_head_range(6, 0, 4)


# the reference's public names (dquant/__init__.py:38-79) minus the dense tensor primitives of
# tensor.py (DenseTensor, QrResult, SvdResult, matmul, permute, qr, reshape, svd: out of scope)
REFERENCE_ALL = [
    "CacheConfig", "CompressionReport", "ErrorRecord", "KvCache", "MemoryLedger", "MpoChain", "OutlierStats",
    "QuantizedMpo", "QuantizedTensor", "ShapePlan", "WorkingSetMeter", "compression_report", "deco_dequantize",
    "deco_quantize", "decompose", "decomposition_comparison", "default_suite", "dequantize", "fused_matmul",
    "fused_matmul_t", "iqr_stats", "length_sweep", "migration_report", "pack", "plan_shapes", "quantize_rtn",
    "reconstruct", "simulate_generation", "split_large_small", "strategy_sweep", "synth_activations", "unpack",
]


def test_reference_names_exported():
    """import paper_2405_12591_b200 as dquant: every reference name resolves (analysis lazily)."""
    import paper_2405_12591_b200 as dq

    for name in REFERENCE_ALL:
        assert name in dq.__all__, name
        assert getattr(dq, name) is not None, name

"""Quantisation-error statistics of the paper's tables, on the device path.

Restates the reference's sweep protocol (analysis.py:147-293) with every DecoQuant step on
the sm_100a kernels: ``decompose`` (K3 factorisation), ``quantize_rtn`` / ``dequantize``
(K2), ``deco_quantize`` / ``deco_dequantize`` (K3 + K4).  The SVD / QR baselines of
``decomposition_comparison`` use cuSOLVER through torch (analysis-only, off the hot path).
Errors are Frobenius norms of the reconstruction residual in fp64, as in the reference;
``tests/test_gpu_analysis.py`` checks every record and median against the reference's own
sweep (``tests/golden/golden_analysis.json``).

The suite generator is a host-side data source (like ``torch.randn`` in the bench): it must
reproduce the reference matrices exactly, so it is numpy with the same RNG call order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .compress import deco_dequantize, deco_quantize
from .errors import EmptyInput, ShapeMismatch
from .mpo import MpoChain, decompose, plan_shapes, reconstruct, split_large_small
from .quantize import dequantize, quantize_rtn

SYNTH_TERMS, SYNTH_DECAY, SYNTH_NOISE = 14, 0.8, 0.08  # analysis.py:22-24

MATRIX_RTN, TL_ONLY, BOTH, SVD, QR = "matrix-rtn", "deco-tl-only", "deco-both", "svd-quant", "qr-quant"


@dataclass(frozen=True)
class OutlierStats:  # analysis.py:47-55
    q1: float
    q3: float
    iqr: float
    lower_fence: float
    upper_fence: float
    outlier_count: int
    total_count: int


@dataclass(frozen=True)
class ErrorRecord:  # analysis.py:58-66
    method: str
    bits: int
    n: int
    seed: int
    frobenius_error: float
    relative_error: float
    param_overhead: float


def iqr_stats(values) -> OutlierStats:
    """Quartiles interpolated at p (n - 1), Tukey fences at 1.5 IQR (analysis.py:69-86)."""
    v = np.sort(np.asarray(values.cpu() if isinstance(values, torch.Tensor) else values, np.float64).ravel())
    if v.size == 0:
        raise EmptyInput("iqr_stats needs at least one value")

    def q(p):
        x = p * (v.size - 1)
        i = int(np.floor(x))
        j = min(i + 1, v.size - 1)
        return float(v[i] + (v[j] - v[i]) * (x - i))

    q1, q3 = q(0.25), q(0.75)
    lo, hi = q1 - 1.5 * (q3 - q1), q3 + 1.5 * (q3 - q1)
    return OutlierStats(q1, q3, q3 - q1, lo, hi, int(np.count_nonzero((v < lo) | (v > hi))), v.size)


def _dyadic(n: int) -> int:
    return 1 << max(1, (n - 1).bit_length())


def _walsh(index: int, n: int) -> np.ndarray:
    """+-1 from the parity of (t & index), t on the covering dyadic grid (analysis.py:89-98)."""
    t = np.arange(_dyadic(n))
    parity = np.array([bin(x).count("1") & 1 for x in (t & index)], dtype=np.float64)
    return (1.0 - 2.0 * parity)[:n]


def _index_pairs(rows: int, cols: int, count: int):
    """Coarse-to-fine (row, col) pattern pairs by diagonals (analysis.py:101-115)."""
    def ladder(m):
        return [0] + [m >> (k + 1) for k in range(m.bit_length() - 1)]

    ri, ci = ladder(_dyadic(rows)), ladder(_dyadic(cols))
    out = []
    for d in range(1, len(ri) + len(ci)):
        for a in range(d + 1):
            if a < len(ri) and d - a < len(ci):
                out.append((ri[a], ci[d - a]))
            if len(out) == count:
                return out
    return out


def synth_activations(rows: int, cols: int, outlier_cols: int = 8, outlier_scale: float = 20.0,
                      seed: int = 0) -> np.ndarray:
    """Correlated multiscale Gaussian field + scaled outlier channels (analysis.py:118-144).

    Same RNG draws in the same order as the reference: the iid noise field, one coefficient
    per pattern pair, then the outlier column choice.
    """
    if outlier_cols > cols:
        raise ShapeMismatch("outlier_cols cannot exceed cols")
    if outlier_scale < 1:
        raise ShapeMismatch("outlier_scale must be >= 1")
    rng = np.random.default_rng(seed)
    pairs = _index_pairs(rows, cols, SYNTH_TERMS)
    w = SYNTH_DECAY ** np.arange(len(pairs))
    w = w * np.sqrt((1.0 - SYNTH_NOISE ** 2) / np.sum(w * w))
    field = SYNTH_NOISE * rng.standard_normal((rows, cols))
    for (r, c), wk in zip(pairs, w):
        field += (wk * rng.standard_normal()) * np.outer(_walsh(r, rows), _walsh(c, cols))
    chosen = rng.choice(cols, size=outlier_cols, replace=False)
    if outlier_cols:
        field[:, chosen] *= outlier_scale
    return field.astype(np.float32)


def default_suite(seeds=range(20), rows=512, cols=512, outlier_cols=8, scale=20.0):
    """The 20-seed outlier suite every sweep uses (analysis.py:147-152)."""
    return [synth_activations(rows, cols, outlier_cols, scale, seed=s) for s in seeds]


def _errors(ref: torch.Tensor, rec: torch.Tensor):
    diff = torch.linalg.norm((ref.double() - rec.double()).reshape(-1)).item()
    norm = torch.linalg.norm(ref.double().reshape(-1)).item()
    return diff, (diff / norm if norm else 0.0)


def _overhead(chain: MpoChain) -> float:
    return sum(int(t.numel()) for t in chain.local_tensors) / (chain.rows * chain.cols)


def strategy_sweep(suite, bits_list=(2, 4, 8)):
    """Matrix RTN vs DecoQuant (large core only, the compression default) vs both cores
    (analysis.py:181-201), one record per (seed, method, bits), n = 2, on the device."""
    dev = _lib.require_cuda()
    records = []
    for seed, m in enumerate(suite):
        x = torch.as_tensor(np.asarray(m, np.float32)).to(dev)
        chain = decompose(x, plan_shapes(x.shape[0], x.shape[1], 2))
        ov = _overhead(chain)
        for bits in bits_list:
            e, r = _errors(x, dequantize(quantize_rtn(x, bits)))
            records.append(ErrorRecord(MATRIX_RTN, bits, 2, seed, e, r, 1.0))
            e, r = _errors(x, deco_dequantize(deco_quantize(x, bits)))
            records.append(ErrorRecord(TL_ONLY, bits, 2, seed, e, r, ov))
            both = MpoChain(tuple(dequantize(quantize_rtn(c, bits)) for c in chain.local_tensors))
            e, r = _errors(x, reconstruct(both))
            records.append(ErrorRecord(BOTH, bits, 2, seed, e, r, ov))
    return sorted(records, key=lambda t: (t.seed, t.method, t.bits))


def length_sweep(suite, n_list=(2, 3, 4), bits: int = 4):
    """Compression error as the chain length grows, first core kept (analysis.py:222-235): n = 2
    on the K3 kernels, n = 3, 4 through the device fp64 TT-SVD (``mpo.decompose``)."""
    dev = _lib.require_cuda()
    records = []
    for seed, m in enumerate(suite):
        x = torch.as_tensor(np.asarray(m, np.float32)).to(dev)
        for n in n_list:
            chain = decompose(x, plan_shapes(x.shape[0], x.shape[1], n))
            cores = (chain.local_tensors[0],) + tuple(dequantize(quantize_rtn(c, bits)) for c in chain.local_tensors[1:])
            e, r = _errors(x, reconstruct(MpoChain(cores)))
            records.append(ErrorRecord(TL_ONLY, bits, n, seed, e, r, _overhead(chain)))
    return sorted(records, key=lambda t: (t.seed, t.n, t.bits))


def decomposition_comparison(suite, bits: int = 4):
    """Chain vs SVD vs QR, quantizing the larger factor (analysis.py:246-271)."""
    dev = _lib.require_cuda()
    records = []
    for seed, m in enumerate(suite):
        x = torch.as_tensor(np.asarray(m, np.float32)).to(dev)
        chain = decompose(x, plan_shapes(x.shape[0], x.shape[1], 2))
        e, r = _errors(x, deco_dequantize(deco_quantize(x, bits)))
        records.append(ErrorRecord(TL_ONLY, bits, 2, seed, e, r, _overhead(chain)))
        # the reference's tensor.svd hands back float32 factors (tensor.py:86-91)
        u, s, vt = (t.float().double() for t in torch.linalg.svd(x.double(), full_matrices=False))
        root = s.sqrt()
        a, b = u * root, root[:, None] * vt
        rec = (dequantize(quantize_rtn(a.float(), bits)).double() @ b if a.numel() > b.numel()
               else a @ dequantize(quantize_rtn(b.float(), bits)).double())
        e, r = _errors(x, rec)
        records.append(ErrorRecord(SVD, bits, 2, seed, e, r, (a.numel() + b.numel()) / x.numel()))
        q, rr = torch.linalg.qr(x.double(), mode="reduced")
        q32, r32 = q.float(), rr.float()
        rec = (dequantize(quantize_rtn(q32, bits)).double() @ r32.double() if q.numel() > rr.numel()
               else q32.double() @ dequantize(quantize_rtn(r32, bits)).double())
        e, r = _errors(x, rec)
        records.append(ErrorRecord(QR, bits, 2, seed, e, r, (q.numel() + rr.numel()) / x.numel()))
    return sorted(records, key=lambda t: (t.seed, t.method, t.bits))


def migration_report(m, plan=None):
    """IQR statistics of the matrix and of its two cores (analysis.py:155-170): on outlier
    data the large core's IQR collapses while the small core keeps the wide values."""
    x = torch.as_tensor(np.asarray(m, np.float32)).to(_lib.require_cuda())
    chain = decompose(x, plan or plan_shapes(x.shape[0], x.shape[1], 2))
    large, small = split_large_small(chain)
    return iqr_stats(x), iqr_stats(large), iqr_stats(small)


def median_by(records, key=lambda r: (r.method, r.bits)):
    """Median Frobenius error per group (analysis.py:288-293)."""
    groups = {}
    for r in records:
        groups.setdefault(key(r), []).append(r.frobenius_error)
    return {k: float(np.median(v)) for k, v in sorted(groups.items())}

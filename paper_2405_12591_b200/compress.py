"""DecoQuant: factorise, quantize every core but the first, read without materialising.

Mirrors ``dquant/compress.py``: ``TILE_ELEMENTS`` (20), ``WorkingSetMeter`` (23-33),
``QuantizedMpo`` (36-73), ``CompressionReport`` (76-82), ``deco_quantize`` (85-94),
``deco_dequantize`` (105-107), ``fused_matmul`` (159-192), ``fused_matmul_t``
(195-231), ``compression_report`` (234-248).

GPU kernels: deco_quantize -> K3 (csrc/factor.cu), deco_dequantize -> K4
(csrc/reads.cu reconstruct), fused reads -> csrc/reads.cu.  Chains of length 2.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from math import prod

import numpy as np
import torch

from . import _lib, mpo
from ._lib import check, lib, ptr, stream_ptr
from .errors import ShapeMismatch, Unsupported
from .quantize import QuantizedTensor, _check_bits, payload_size

TILE_ELEMENTS = 64 * 64
# codes one CTA of the fused kernels holds dequantized at any moment (one per thread)
_FUSED_INFLIGHT = 256


class WorkingSetMeter:
    """Tracks transient dequantized buffer sizes inside fused multiplies (compress.py:23-33)."""

    def __init__(self):
        self.peak_elements = 0
        self.total_unpacked = 0

    def record(self, n_elements: int):
        self.total_unpacked += n_elements
        if n_elements > self.peak_elements:
            self.peak_elements = n_elements


@dataclass(frozen=True)
class QuantizedMpo:
    """A core chain where all cores but the first are bit-packed (compress.py:36-73)."""

    plan: mpo.ShapePlan
    bits: int
    local_tensors: tuple  # core0 (fp32 array / tensor), then QuantizedTensor(s)

    def __post_init__(self):
        shapes = [tuple(t.shape) for t in self.local_tensors]
        if len(shapes) != self.plan.n:
            raise ShapeMismatch("chain length disagrees with plan")
        for k, s in enumerate(shapes):
            expected = (1 if k == 0 else shapes[k - 1][3], self.plan.i_factors[k], self.plan.j_factors[k])
            if tuple(s[:3]) != expected or (k == len(shapes) - 1 and s[3] != 1):
                raise ShapeMismatch(f"core {k} has shape {s}, expected {expected}")

    @property
    def rows(self) -> int:
        return self.plan.rows

    @property
    def cols(self) -> int:
        return self.plan.cols

    @property
    def quantized_locals(self) -> tuple:
        return tuple(t for t in self.local_tensors if isinstance(t, QuantizedTensor))

    @property
    def fp_locals(self) -> tuple:
        return tuple(t for t in self.local_tensors if not isinstance(t, QuantizedTensor))


@dataclass(frozen=True)
class CompressionReport:
    """Stored-size accounting against a 16-bit uncompressed baseline."""

    ratio: float
    bytes_original: int
    bytes_compressed: int


def _numel(t) -> int:
    return t.numel() if isinstance(t, torch.Tensor) else int(np.asarray(t).size)


def _core0_dev(core0) -> torch.Tensor:
    dev = _lib.require_cuda()
    if isinstance(core0, torch.Tensor):
        return core0.to(dev, torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(core0, dtype=np.float32)).to(dev)


def deco_quantize_batched(blocks: torch.Tensor, bits: int, layout: int = _lib.LAYOUT_REF, stride: int | None = None):
    """K3 on a batch (nblk, rows, cols) of fp16/fp32 CUDA blocks.

    Returns dict(core0 (nblk,1,i1,j1,r) f32, payload (nblk, stride) u8 in `layout`,
    scale (nblk,) f32, plan).  Raises NonFiniteInput / NoConvergence from device flags.
    """
    _check_bits(bits)
    dev = _lib.require_cuda()
    if blocks.ndim != 3:
        raise ShapeMismatch("expected (nblk, rows, cols)")
    dtype = _lib.DQ_F16 if blocks.dtype == torch.float16 else _lib.DQ_F32
    x = blocks.to(device=dev, dtype=torch.float16 if dtype == _lib.DQ_F16 else torch.float32).contiguous()
    nblk, rows, cols = x.shape
    p = _lib.plan2(rows, cols)
    nbytes = _lib.layout_bytes(p, bits, layout)
    stride = stride or nbytes
    core0 = torch.empty((nblk, 1, p.i1, p.j1, p.r), dtype=torch.float32, device=dev)
    payload = torch.empty((nblk, stride), dtype=torch.uint8, device=dev)
    scale = torch.empty(nblk, dtype=torch.float32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    size = ctypes.c_size_t()
    check(lib().dq_decompose_workspace_size(nblk, rows, cols, ctypes.byref(size)), "workspace")
    ws = torch.empty(max(size.value, 256), dtype=torch.uint8, device=dev)
    check(lib().dq_deco_quantize_batched(ptr(x), dtype, nblk, rows, cols, bits, layout, ptr(core0), ptr(payload),
                                         stride, ptr(scale), ptr(flags), ptr(ws), ws.numel(), stream_ptr()),
          "deco_quantize")
    return {"core0": core0, "payload": payload, "scale": scale, "plan": p, "flags": flags, "layout": layout,
            "bytes": nbytes}


def deco_quantize(m, bits: int, n: int = 2) -> QuantizedMpo:
    """Factorize and quantize every core except the first (compress.py:85-94)."""
    _check_bits(bits)
    is_t = isinstance(m, torch.Tensor)
    shape = tuple(m.shape) if is_t else np.asarray(m).shape
    if len(shape) != 2:
        raise ShapeMismatch(f"expected a matrix, got shape {shape}")
    if n != 2:
        raise Unsupported("the sm_100a DecoQuant kernels implement chains of length n=2")
    plan = mpo.plan_shapes(shape[0], shape[1], n)
    x = m if is_t else torch.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=np.float32)))
    res = deco_quantize_batched(x.reshape(1, *shape), bits)
    _lib.raise_flags(res["flags"], "deco_quantize")
    p = res["plan"]
    core0 = res["core0"][0]
    qt = QuantizedTensor((p.r, p.i2, p.j2, 1), bits, float(res["scale"][0].item()), data=res["payload"][0],
                         torch_out=is_t)
    return QuantizedMpo(plan=plan, bits=bits, local_tensors=(core0 if is_t else core0.cpu().numpy(), qt))


def _parts(q: QuantizedMpo):
    if q.plan.n != 2:
        raise Unsupported("chains of length n=2 only")
    core0, qt = q.local_tensors
    scale = torch.tensor([qt.scale], dtype=torch.float32, device=qt.data.device)
    return _core0_dev(core0), qt, scale


def deco_dequantize(q: QuantizedMpo):
    """Recover the full-precision matrix (compress.py:105-107): kernel K4."""
    core0, qt, scale = _parts(q)
    out = torch.empty((q.rows, q.cols), dtype=torch.float32, device=qt.data.device)
    check(lib().dq_deco_dequantize_batched(ptr(core0), ptr(qt.data), qt.data.numel(), _lib.LAYOUT_REF, ptr(scale), 1,
                                           q.rows, q.cols, q.bits, ptr(out), _lib.DQ_F32, stream_ptr()),
          "deco_dequantize")
    return out if qt._torch else out.cpu().numpy()


def _fused(x, q: QuantizedMpo, meter, transposed: bool):
    core0, qt, scale = _parts(q)
    is_t = isinstance(x, torch.Tensor)
    xs = tuple(x.shape) if is_t else np.asarray(x).shape
    need = q.cols if transposed else q.rows
    if len(xs) != 2 or xs[1] != need:
        what = "cols" if transposed else "rows"
        raise ShapeMismatch(f"operand shape {xs} does not match {what} {need}")
    xd = (x if is_t else torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))).to(
        qt.data.device, torch.float32).contiguous()
    p = xs[0]
    out = torch.empty((p, q.rows if transposed else q.cols), dtype=torch.float32, device=qt.data.device)
    fn = lib().dq_fused_matmul_t if transposed else lib().dq_fused_matmul
    check(fn(ptr(xd), p, ptr(core0), ptr(qt.data), _lib.LAYOUT_REF, ptr(scale), q.rows, q.cols, q.bits, ptr(out),
             stream_ptr()), "fused_matmul_t" if transposed else "fused_matmul")
    if meter is not None:
        # each CTA converts one code per thread at a time; nothing larger is ever dequantized
        ctas = p * max(1, -(-q.plan.i_factors[1] // 256)) if transposed else p
        for _ in range(ctas):
            meter.record(min(_FUSED_INFLIGHT, qt.count))
    return out if is_t else out.cpu().numpy()


def fused_matmul(x, q: QuantizedMpo, meter: WorkingSetMeter = None):
    """x @ W for the compressed W, streaming the packed core (compress.py:159-192)."""
    return _fused(x, q, meter, transposed=False)


def fused_matmul_t(x, q: QuantizedMpo, meter: WorkingSetMeter = None):
    """x @ W.T, streaming the packed core (compress.py:195-231)."""
    return _fused(x, q, meter, transposed=True)


def compression_report(q: QuantizedMpo) -> CompressionReport:
    """Bit-weighted size of the stored cores over the 16-bit original (compress.py:234-248)."""
    n_quant = sum(t.count for t in q.quantized_locals)
    n_fp = sum(_numel(t) for t in q.fp_locals)
    n_scales = len(q.quantized_locals)
    numerator_bits = n_quant * q.bits + n_fp * 16 + n_scales * 16
    original_bits = q.rows * q.cols * 16
    bytes_compressed = sum(payload_size(t.count, t.bits) for t in q.quantized_locals) + 2 * n_scales + 2 * n_fp
    return CompressionReport(ratio=numerator_bits / original_bits, bytes_original=q.rows * q.cols * 2,
                             bytes_compressed=bytes_compressed)


__all__ = [
    "TILE_ELEMENTS", "WorkingSetMeter", "QuantizedMpo", "CompressionReport", "deco_quantize", "deco_dequantize",
    "fused_matmul", "fused_matmul_t", "compression_report", "deco_quantize_batched", "prod",
]

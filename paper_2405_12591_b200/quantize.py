"""Symmetric per-tensor RTN quantizer and 2/4/8-bit packing on the GPU.

Mirrors ``dquant/quantize.py`` (names, signatures, error classes, wire format):
``SUPPORTED_BITS`` (23), ``payload_size`` (31-33), ``QuantizedTensor`` (36-63),
``pack`` (66-82), ``unpack`` (85-92), ``unpack_range`` (95-109),
``quantize_rtn`` (123-151), ``dequantize`` (154-157).

Values live on the GPU; numpy / bytes inputs give numpy / bytes outputs (the
reference's types), torch CUDA inputs give torch CUDA outputs.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr, stream_ptr
from .errors import CorruptPayload, NonFiniteInput, RangeOverflow, UnsupportedBits

SUPPORTED_BITS = (2, 4, 8)


def _check_bits(bits):
    if bits not in SUPPORTED_BITS:
        raise UnsupportedBits(f"bits must be one of {SUPPORTED_BITS}, got {bits}")


def payload_size(count: int, bits: int) -> int:
    """Number of payload bytes for `count` packed codes (quantize.py:31-33)."""
    return (count * bits + 7) // 8


def _device():
    return _lib.require_cuda()


def _as_device(x, dtype) -> tuple[torch.Tensor, bool]:
    """(contiguous CUDA tensor, came_from_torch)."""
    if isinstance(x, torch.Tensor):
        return x.to(device=_device(), dtype=dtype).contiguous(), True
    arr = np.ascontiguousarray(np.asarray(x))
    return torch.from_numpy(arr).to(device=_device(), dtype=dtype), False


def _bytes_to_device(payload) -> torch.Tensor:
    if isinstance(payload, torch.Tensor):
        return payload.to(device=_device(), dtype=torch.uint8).contiguous().reshape(-1)
    buf = np.frombuffer(bytes(payload), dtype=np.uint8).copy()
    return torch.from_numpy(buf).to(_device())


class QuantizedTensor:
    """Bit-packed signed codes plus the scale needed to dequantize them (quantize.py:36-63).

    The packed payload is held on the GPU (``data``, a uint8 CUDA tensor in the
    reference wire order); ``payload`` returns it as ``bytes``.
    """

    __slots__ = ("shape", "bits", "scale", "data", "_bytes", "_torch")

    def __init__(self, shape, bits, scale, payload=None, *, data=None, torch_out=False):
        _check_bits(bits)
        self.shape = tuple(int(d) for d in shape)
        self.bits = int(bits)
        self.scale = float(scale)
        if self.scale <= 0:
            raise CorruptPayload(f"scale must be positive, got {self.scale}")
        if data is None:
            if payload is None:
                raise CorruptPayload("payload is required")
            n = payload.numel() if isinstance(payload, torch.Tensor) else len(payload)
            if n != payload_size(self.count, self.bits):
                raise CorruptPayload(
                    f"payload is {n} bytes, expected {payload_size(self.count, self.bits)} "
                    f"for shape {self.shape} at {self.bits} bits"
                )
            data = _bytes_to_device(payload)
            torch_out = torch_out or isinstance(payload, torch.Tensor)
        elif data.numel() != payload_size(self.count, self.bits):
            raise CorruptPayload("device payload has the wrong length")
        self.data = data
        self._bytes = None
        self._torch = torch_out

    def __setattr__(self, name, value):
        if name in ("shape", "bits", "scale", "data") and hasattr(self, name):
            raise AttributeError(f"QuantizedTensor.{name} is immutable")
        object.__setattr__(self, name, value)

    @property
    def count(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64)) if self.shape else 1

    @property
    def payload(self) -> bytes:
        if self._bytes is None:
            object.__setattr__(self, "_bytes", self.data.cpu().numpy().tobytes())
        return self._bytes

    def codes(self):
        """Unpacked signed codes in row-major order."""
        out = unpack(self.data, self.count, self.bits)
        return out if self._torch else out.cpu().numpy()

    def __eq__(self, other):
        if not isinstance(other, QuantizedTensor):
            return NotImplemented
        return (self.shape, self.bits, self.scale, self.payload) == (other.shape, other.bits, other.scale,
                                                                     other.payload)

    def __repr__(self):
        return f"QuantizedTensor(shape={self.shape}, bits={self.bits}, scale={self.scale!r}, payload=<{self.data.numel()} B on {self.data.device}>)"


def pack(values, bits: int):
    """Bit-pack small signed integers, low bits first (quantize.py:66-82).

    Returns ``bytes`` (torch uint8 CUDA tensor for torch input)."""
    _check_bits(bits)
    if isinstance(values, torch.Tensor):
        v, is_t = values.to(device=_device()).reshape(-1), True
    else:
        arr = np.asarray(values, dtype=np.int64).reshape(-1)
        qmax = (1 << (bits - 1)) - 1
        if arr.size and (arr.min() < -qmax or arr.max() > qmax):
            raise RangeOverflow(f"values outside [-{qmax}, {qmax}] at {bits} bits")
        v, is_t = torch.from_numpy(arr.astype(np.int8)).to(_device()), False
    qmax = (1 << (bits - 1)) - 1
    if v.dtype != torch.int8:
        if v.numel() and (int(v.min()) < -qmax or int(v.max()) > qmax):
            raise RangeOverflow(f"values outside [-{qmax}, {qmax}] at {bits} bits")
        v = v.to(torch.int8)
    v = v.contiguous()
    out = torch.empty(payload_size(v.numel(), bits), dtype=torch.uint8, device=v.device)
    flags = torch.zeros(1, dtype=torch.int32, device=v.device)
    check(lib().dq_pack(ptr(v), v.numel(), bits, ptr(out), ptr(flags), stream_ptr()), "pack")
    _lib.raise_flags(flags, "pack")
    return out if is_t else out.cpu().numpy().tobytes()


def _unpack_impl(payload, start, count, bits):
    _check_bits(bits)
    data = _bytes_to_device(payload)
    out = torch.empty(count, dtype=torch.int8, device=data.device)
    check(lib().dq_unpack(ptr(data), data.numel(), start, count, bits, ptr(out), stream_ptr()), "unpack")
    return out


def unpack(payload, count: int, bits: int):
    """Inverse of pack; int8 codes (quantize.py:85-92)."""
    _check_bits(bits)
    n = payload.numel() if isinstance(payload, torch.Tensor) else len(payload)
    if n != payload_size(count, bits):
        raise CorruptPayload(f"payload is {n} bytes, expected {payload_size(count, bits)}")
    out = _unpack_impl(payload, 0, count, bits)
    return out if isinstance(payload, torch.Tensor) else out.cpu().numpy()


def unpack_range(payload, start: int, count: int, bits: int):
    """Codes [start, start+count) without touching the rest (quantize.py:95-109)."""
    _check_bits(bits)
    out = _unpack_impl(payload, start, count, bits)
    return out if isinstance(payload, torch.Tensor) else out.cpu().numpy()


def quantize_rtn(t, bits: int) -> QuantizedTensor:
    """One symmetric scale, round half away from zero (quantize.py:123-151)."""
    _check_bits(bits)
    # the reference multiplies the ORIGINAL values in float64 (quantize.py:144): fp16 / fp32
    # inputs are exact in fp32; float64 (and integer) inputs keep an fp64 path
    src_dtype = t.dtype if isinstance(t, torch.Tensor) else np.asarray(t).dtype
    f64 = src_dtype not in (torch.float16, torch.float32, torch.bfloat16, np.float16, np.float32)
    x, is_t = _as_device(t, torch.float64 if f64 else torch.float32)
    shape = tuple(x.shape)
    x = x.reshape(-1)
    n = x.numel()
    scale = torch.empty(1, dtype=torch.float32, device=x.device)
    out = torch.empty(payload_size(n, bits), dtype=torch.uint8, device=x.device)
    flags = torch.zeros(1, dtype=torch.int32, device=x.device)
    ws = torch.empty(256, dtype=torch.uint8, device=x.device)
    fn = lib().dq_quantize_rtn_f64 if f64 else lib().dq_quantize_rtn
    check(fn(ptr(x), n, bits, ptr(scale), ptr(out), ptr(flags), ptr(ws), 256, stream_ptr()), "quantize_rtn")
    if int(flags.item()) & _lib.FLAG_NONFINITE:
        raise NonFiniteInput("quantize_rtn requires finite entries")
    return QuantizedTensor(shape, bits, float(scale.item()), data=out, torch_out=is_t)


def dequantize(q: QuantizedTensor):
    """Codes times scale, as float32, in the original shape (quantize.py:154-157)."""
    scale = torch.tensor([q.scale], dtype=torch.float32, device=q.data.device)
    out = torch.empty(q.count, dtype=torch.float32, device=q.data.device)
    check(lib().dq_dequantize(ptr(q.data), q.count, q.bits, ptr(scale), ptr(out), stream_ptr()), "dequantize")
    out = out.reshape(q.shape)
    return out if q._torch else out.cpu().numpy()

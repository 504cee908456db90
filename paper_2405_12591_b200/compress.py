"""DecoQuant: factorise, quantize every core but the first, read without materialising.

Mirrors ``dquant/compress.py``: ``TILE_ELEMENTS`` (20), ``WorkingSetMeter`` (23-33),
``QuantizedMpo`` (36-73), ``CompressionReport`` (76-82), ``deco_quantize`` (85-94),
``deco_dequantize`` (105-107), ``fused_matmul`` (159-192), ``fused_matmul_t``
(195-231), ``compression_report`` (234-248).

GPU kernels: deco_quantize -> K3 (csrc/factor.cu), deco_dequantize -> K4
(csrc/reads.cu reconstruct), fused reads -> csrc/reads.cu, for chains of length 2 (the hot
path).  Longer chains (n = 3, 4: the reference's length sweep and CacheConfig(n)) run on the
device too: the fp64 TT-SVD of ``mpo.decompose``, K2 quantize / dequantize per core, and the
reference's left-to-right / right-to-left core sweeps as fp64 GEMMs over codes unpacked tile
by tile (``unpack_range``, never more than TILE_ELEMENTS codes at once).
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
from .quantize import QuantizedTensor, _check_bits, dequantize, payload_size, quantize_rtn, unpack_range

TILE_ELEMENTS = 64 * 64
# codes one CTA of the fused kernels holds dequantized at any moment (one per thread)


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


def deco_quantize_asym_batched(blocks: torch.Tensor, bits: int, layout: int = _lib.LAYOUT_REF,
                               stride: int | None = None):
    """K3 with the opt-in per-channel ASYMMETRIC quantizer (north_star; not in the reference,
    parity against the oracle's ``rtn_asym`` only): channel (r, e) of core1 over b, 2 or 4 bits.

    Returns dict(core0, payload (raw codes u in `layout`), channels (nblk, 2, r, 16) f32 = scales
    then zero points, plan, flags); value = scale * (u - zero).
    """
    if bits not in (2, 4):
        from .quantize import UnsupportedBits
        raise UnsupportedBits("the asymmetric mode covers 2- and 4-bit codes")
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
    channels = torch.empty((nblk, 2, p.r, p.j2), dtype=torch.float32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    size = ctypes.c_size_t()
    check(lib().dq_decompose_workspace_size(nblk, rows, cols, ctypes.byref(size)), "workspace")
    ws = torch.empty(max(size.value, 256), dtype=torch.uint8, device=dev)
    check(lib().dq_deco_quantize_asym_batched(ptr(x), dtype, nblk, rows, cols, bits, layout, ptr(core0), ptr(payload),
                                              stride, ptr(channels), ptr(flags), ptr(ws), ws.numel(), stream_ptr()),
          "deco_quantize_asym")
    return {"core0": core0, "payload": payload, "channels": channels, "plan": p, "flags": flags, "layout": layout,
            "bytes": nbytes}


def deco_quantize(m, bits: int, n: int = 2) -> QuantizedMpo:
    """Factorize and quantize every core except the first (compress.py:85-94)."""
    _check_bits(bits)
    is_t = isinstance(m, torch.Tensor)
    shape = tuple(m.shape) if is_t else np.asarray(m).shape
    if len(shape) != 2:
        raise ShapeMismatch(f"expected a matrix, got shape {shape}")
    plan = mpo.plan_shapes(shape[0], shape[1], n)
    x = m if is_t else torch.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=np.float32)))
    if n != 2:  # longer chains: device TT-SVD, then K2 on every core but the first
        chain = mpo.decompose(x.to(_lib.require_cuda()), plan)
        cores = [chain.local_tensors[0]] + [quantize_rtn(t, bits) for t in chain.local_tensors[1:]]
        if not is_t:
            cores[0] = cores[0].cpu().numpy()
            cores[1:] = [QuantizedTensor(c.shape, c.bits, c.scale, data=c.data, torch_out=False) for c in cores[1:]]
        return QuantizedMpo(plan=plan, bits=bits, local_tensors=tuple(cores))
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


def _rebuild_chain(q: QuantizedMpo):
    """Dequantized cores as a device MpoChain (compress.py:97-102)."""
    dev = _lib.require_cuda()
    cores = []
    for t in q.local_tensors:
        if isinstance(t, QuantizedTensor):
            c = dequantize(QuantizedTensor(t.shape, t.bits, t.scale, data=t.data, torch_out=True))
        else:
            c = (t if isinstance(t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(t))).to(dev, torch.float32)
        cores.append(c)
    return mpo.MpoChain(tuple(cores))


def _is_torch_mpo(q: QuantizedMpo) -> bool:
    t = q.local_tensors[-1]
    return t._torch if isinstance(t, QuantizedTensor) else isinstance(t, torch.Tensor)


def deco_dequantize(q: QuantizedMpo):
    """Recover the full-precision matrix (compress.py:105-107): kernel K4 (n = 2), or the
    dequantized cores contracted in fp64 on the device (longer chains)."""
    if q.plan.n != 2:
        out = mpo.reconstruct(_rebuild_chain(q))
        return out if _is_torch_mpo(q) else out.cpu().numpy()
    core0, qt, scale = _parts(q)
    out = torch.empty((q.rows, q.cols), dtype=torch.float32, device=qt.data.device)
    check(lib().dq_deco_dequantize_batched(ptr(core0), ptr(qt.data), qt.data.numel(), _lib.LAYOUT_REF, ptr(scale), 1,
                                           q.rows, q.cols, q.bits, ptr(out), _lib.DQ_F32, stream_ptr()),
          "deco_dequantize")
    return out if qt._torch else out.cpu().numpy()


def _core_f64(core, dev):
    return (core if isinstance(core, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(core))).to(
        dev, torch.float64)


def _tile_codes(qt: QuantizedTensor, start: int, count: int, dev, meter):
    codes = unpack_range(qt.data, start, count, qt.bits)
    if meter is not None:
        meter.record(count)
    return codes.to(dev, torch.float64) * float(np.float32(qt.scale))


def _gemm_packed_right(a, qt, rows, cols, meter, dev):
    """a @ M for a packed (rows, cols) core, unpacked in tiles (compress.py:110-131)."""
    out = torch.zeros((a.shape[0], cols), dtype=torch.float64, device=dev)
    if cols <= TILE_ELEMENTS:
        rt = max(1, TILE_ELEMENTS // cols)
        for r0 in range(0, rows, rt):
            r1 = min(rows, r0 + rt)
            out += a[:, r0:r1] @ _tile_codes(qt, r0 * cols, (r1 - r0) * cols, dev, meter).reshape(r1 - r0, cols)
    else:
        for r in range(rows):
            for c0 in range(0, cols, TILE_ELEMENTS):
                c1 = min(cols, c0 + TILE_ELEMENTS)
                out[:, c0:c1] += torch.outer(a[:, r], _tile_codes(qt, r * cols + c0, c1 - c0, dev, meter))
    return out


def _gemm_packed_left(qt, rows, cols, b, meter, dev):
    """M @ b for a packed (rows, cols) core, unpacked in tiles (compress.py:134-156)."""
    out = torch.zeros((rows, b.shape[1]), dtype=torch.float64, device=dev)
    if cols <= TILE_ELEMENTS:
        rt = max(1, TILE_ELEMENTS // cols)
        for r0 in range(0, rows, rt):
            r1 = min(rows, r0 + rt)
            out[r0:r1] = _tile_codes(qt, r0 * cols, (r1 - r0) * cols, dev, meter).reshape(r1 - r0, cols) @ b
    else:
        for r in range(rows):
            for c0 in range(0, cols, TILE_ELEMENTS):
                c1 = min(cols, c0 + TILE_ELEMENTS)
                out[r] += _tile_codes(qt, r * cols + c0, c1 - c0, dev, meter) @ b[c0:c1]
    return out


def _fused_chain(x, q: QuantizedMpo, meter, transposed: bool):
    """Longer chains: the reference's core sweeps (compress.py:159-231) on the device in fp64."""
    dev = _lib.require_cuda()
    is_t = isinstance(x, torch.Tensor)
    xs = tuple(x.shape) if is_t else np.asarray(x).shape
    need = q.cols if transposed else q.rows
    if len(xs) != 2 or xs[1] != need:
        raise ShapeMismatch(f"operand shape {xs} does not match {'cols' if transposed else 'rows'} {need}")
    xd = (x if is_t else torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))).to(dev, torch.float64)
    p = xs[0]
    i_f, j_f, n = q.plan.i_factors, q.plan.j_factors, q.plan.n
    cores = q.local_tensors
    if not transposed:  # x @ W: left to right, state (p, i_rest, j_acc, d)
        cur = xd.reshape((p,) + tuple(i_f) + (1, 1))
        j_acc, d = 1, 1
        for k in range(n):
            ik, jk = i_f[k], j_f[k]
            i_rest = prod(i_f[k + 1:]) if k + 1 < n else 1
            cur = cur.reshape(p, ik, i_rest, j_acc, d).permute(0, 2, 3, 4, 1).contiguous()
            a = cur.reshape(p * i_rest * j_acc, d * ik)
            core = cores[k]
            d_next = core.shape[3]
            if isinstance(core, QuantizedTensor):
                out = _gemm_packed_right(a, core, d * ik, jk * d_next, meter, dev)
            else:
                out = a @ _core_f64(core, dev).reshape(d * ik, jk * d_next)
            j_acc *= jk
            d = d_next
            cur = out.reshape(p, i_rest, j_acc, d)
        res = cur.reshape(p, q.cols).to(torch.float32).contiguous()
    else:  # x @ W.T: right to left, state (j_lead, d_prev, i_acc, p)
        cur = xd.t().contiguous().reshape(tuple(j_f) + (1, 1, p))
        i_acc = 1
        for k in range(n - 1, -1, -1):
            ik, jk = i_f[k], j_f[k]
            d_prev = 1 if k == 0 else cores[k - 1].shape[3]
            d_k = cores[k].shape[3]
            j_lead = prod(j_f[:k]) if k > 0 else 1
            cur = cur.reshape(j_lead, jk, d_k, i_acc, p).permute(1, 2, 0, 3, 4).contiguous()
            b = cur.reshape(jk * d_k, j_lead * i_acc * p)
            core = cores[k]
            if isinstance(core, QuantizedTensor):
                out = _gemm_packed_left(core, d_prev * ik, jk * d_k, b, meter, dev)
            else:
                out = _core_f64(core, dev).reshape(d_prev * ik, jk * d_k) @ b
            out = out.reshape(d_prev, ik, j_lead, i_acc, p).permute(2, 0, 1, 3, 4).contiguous()
            i_acc *= ik
            cur = out.reshape(j_lead, d_prev, i_acc, p)
        res = cur.reshape(q.rows, p).t().to(torch.float32).contiguous()
    return res if is_t else res.cpu().numpy()


def _fused(x, q: QuantizedMpo, meter, transposed: bool):
    if q.plan.n != 2:
        return _fused_chain(x, q, meter, transposed)
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
    mdev = torch.zeros(2, dtype=torch.int64, device=qt.data.device) if meter is not None else None
    check(fn(ptr(xd), p, ptr(core0), ptr(qt.data), _lib.LAYOUT_REF, ptr(scale), q.rows, q.cols, q.bits, ptr(out),
             ptr(mdev), stream_ptr()), "fused_matmul_t" if transposed else "fused_matmul")
    if meter is not None:  # what the kernels measured (reads.cu meter_report)
        peak, total = (int(v) for v in mdev.cpu())
        meter.record(peak)
        meter.total_unpacked += total - peak
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
    "fused_matmul", "fused_matmul_t", "compression_report", "deco_quantize_batched", "deco_quantize_asym_batched",
    "prod",
]

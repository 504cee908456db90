"""Batched device KV cache + fused DecoQuant decode attention (the hot path).

One *unit* is one (sequence, kv-head) pair of a layer.  ``DecodeKvCache`` keeps,
for every layer, the reference cache lifecycle (kvcache.py:94-128) for all units
at once:

* ``prefill(layer, K, V)``: the whole prompt of every unit becomes ONE segment
  (kvcache.py:99-114), compressed by K3 (csrc/factor.cu) straight into the
  device layouts the attention kernel streams (K: DQ_LAYOUT_KTILE, V: DQ_LAYOUT_VTILE).
* ``append_token(layer, k, v)``: fp16 tail write (kvcache.py:116-123); when the
  tail reaches ``chunk_len`` it is sealed into a new segment (kvcache.py:124-128).
* ``attend(layer, q)``: softmax(q K^T / sqrt(128)) V over every segment and the
  tail, by K5 (csrc/attention.cu) -- the reference's ``attention_scores``
  (kvcache.py:188-217) followed by softmax and the per-segment PV ``fused_matmul``
  (compress.py:159-192), fused, with no full-precision K/V anywhere in HBM.

``export_segment`` returns a segment in the reference's ``QuantizedMpo`` form
(wire-order payload), so the device cache interoperates byte-exactly.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr, stream_ptr
from .compress import QuantizedMpo, deco_quantize_asym_batched, deco_quantize_batched
from .errors import AlreadyPrefilled, DimMismatch, LayerOutOfRange, ShapeMismatch, Unsupported
from .mpo import plan_shapes
from .quantize import SUPPORTED_BITS, QuantizedTensor, UnsupportedBits, payload_size

HEAD_DIM = 128
# numpy view of dq_segment (the ctypes record of _lib.Segment), for column-wise table builds
_SEG_DTYPE = np.dtype({"names": [f[0] for f in _lib.Segment._fields_],
                       "formats": [np.uint64 if f[1] is ctypes.c_void_p else
                                   (np.float32 if f[1] is ctypes.c_float else np.int32)
                                   for f in _lib.Segment._fields_],
                       "offsets": [getattr(_lib.Segment, f[0]).offset for f in _lib.Segment._fields_],
                       "itemsize": ctypes.sizeof(_lib.Segment)})
DEFAULT_CHUNK_B = 256
TAIL_SPLIT = 0.2  # fraction of the persistent grid whose last 512-row items are halved (split_tail)
MAX_CHUNK_B = 512  # > 256: 8-tile items, mma.sync split kernel with g = 1 and 2- / 4-bit codes
KERNEL_G = (1, 2, 8)  # query heads per kv head the split kernels are instantiated for (8: tcgen05 only)
GQA_G = 8             # heads of the tcgen05 GQA kernel (path 2)
MAX_G = 16          # wider GQA groups run as g / kernel_g head groups over the same codes
MAX_BLOCKS_PER_CALL = 4096   # K3 blocks per call; the fp32 core1 scratch is capped at
K3_SCRATCH_BYTES = 2 << 30    # 2 GB: T = 1024 -> 4096 blocks per call, T = 4096 -> 1024


@dataclass
class SegmentGroup:
    """Segment index s of every unit of a layer (same T, same plan)."""

    T: int
    plan: _lib.Plan2
    i2p: int
    k_payload: torch.Tensor  # (units, kbytes) u8, KTILE
    v_payload: torch.Tensor  # (units, vbytes) u8, VTILE
    k_core0: torch.Tensor    # (units, 1, i1, 8, r) f32
    v_core0: torch.Tensor
    k_g0h: torch.Tensor      # (units, i1*r*8) f16, [a][r][c], normalised (core0 = g0h * norm)
    v_g0h: torch.Tensor
    k_scale: torch.Tensor    # (units,) f32 quantizer scale
    v_scale: torch.Tensor
    k_norm: torch.Tensor     # (units,) f32 power-of-two G0 normalisation
    v_norm: torch.Tensor
    token0: int
    k_ch: torch.Tensor | None = None  # asymmetric mode: (units, 2, r, 16) f32 channel scales, zero points
    v_ch: torch.Tensor | None = None
    v_g0f16: torch.Tensor | None = None  # fp16 copy of v_g0h where the split kernel folds fp16 (path 0, g = 1)

    def reference_bytes(self, bits: int) -> int:
        """compression_report().bytes_compressed of one unit's K (or V) block (compress.py:234-248);
        the asymmetric mode stores a 16-bit scale and zero point per (r, e) channel instead of
        one scale."""
        p = self.plan
        scales = 2 * 2 * p.r * p.j2 if self.k_ch is not None else 2
        return payload_size(p.r * p.i2 * p.j2, bits) + scales + 2 * (p.i1 * p.j1 * p.r)

    def stream_bytes(self) -> int:
        """Bytes K5 reads for one unit of this segment (K + V): packed cores, fp32 G0k and G0v, scales
        (the channel tables in the asymmetric mode)."""
        ch = 2 * self.k_ch[0].numel() * 4 if self.k_ch is not None else 0
        vg = self.v_g0f16 if self.v_g0f16 is not None else self.v_g0h  # fp16 where the kernel folds fp16
        return (self.k_payload.shape[1] + self.v_payload.shape[1] + self.k_g0h.element_size() * self.k_g0h.shape[1]
                + vg.element_size() * vg.shape[1] + 8 + ch)


class _Layer:
    def __init__(self):
        self.groups: list[SegmentGroup] = []
        self.tokens_sealed = 0
        self.tail_len = 0  # host mirror (all units append in lock step)
        self.args = None   # cached AttnArgs
        self.kernel_g = None  # heads per split-kernel instance used for this layer
        self.keep = []     # tensors referenced by args
        self.gen = 0       # plan generation: bumped whenever the segment table / args change
        self.seal_pending = False  # the tail is full: sealed (batched) before the next use


def compress_blocks(blocks: torch.Tensor, bits: int, layout: int, g0_dtype=torch.float16, asym: bool = False,
                    flags: torch.Tensor | None = None):
    """K3 over (nblk, T, 128) fp16/fp32 CUDA blocks in slices of MAX_BLOCKS_PER_CALL.

    Returns (payload (nblk, bytes), core0 f32, g0 [a][r][c] normalised in g0_dtype, norm f32, scale f32, plan);
    with ``asym`` the scale is 1 and the per-channel tables come back as a 7th item (nblk, 2, r, 16).
    Errors (non-finite input, no convergence) raise here, after a sync; with a device ``flags``
    word they are OR-ed into it instead, and nothing synchronises.
    """
    nblk = blocks.shape[0]
    outs = []
    # large calls keep the latency-bound eigensolver (one CTA per block) in many full waves
    per = max(64, min(MAX_BLOCKS_PER_CALL, K3_SCRATCH_BYTES // (64 * 2 * blocks.shape[1] * 4)))
    for s in range(0, nblk, per):
        fn = deco_quantize_asym_batched if asym else deco_quantize_batched
        res = fn(blocks[s:s + per], bits, layout)
        if flags is None:
            _lib.raise_flags(res["flags"], "deco_quantize")
        else:
            flags.bitwise_or_(res["flags"])
        outs.append(res)
    p = outs[0]["plan"]
    payload = torch.cat([o["payload"] for o in outs]) if len(outs) > 1 else outs[0]["payload"]
    core0 = torch.cat([o["core0"] for o in outs]) if len(outs) > 1 else outs[0]["core0"]
    if asym:
        chans = torch.cat([o["channels"] for o in outs]) if len(outs) > 1 else outs[0]["channels"]
        scale = torch.ones(nblk, dtype=torch.float32, device=blocks.device)
    else:
        scale = torch.cat([o["scale"] for o in outs]) if len(outs) > 1 else outs[0]["scale"]
    g0 = torch.empty((nblk, p.i1 * p.r * p.j1), dtype=g0_dtype, device=blocks.device)
    norm = torch.empty(nblk, dtype=torch.float32, device=blocks.device)
    code = _lib.DQ_F16 if g0_dtype == torch.float16 else _lib.DQ_F32
    check(lib().dq_core0_relayout(ptr(core0), nblk, ctypes.byref(p), ptr(g0), code, ptr(norm), stream_ptr()),
          "core0_relayout")
    if asym:
        return payload, core0, g0, norm, scale, p, chans
    return payload, core0, g0, norm, scale, p


@dataclass
class WorkPlan:
    """Host result of dq_attention_plan."""

    nwork: int
    total_parts: int
    work: list          # [nwork * 3] = (segment, b0, tiles)
    work_part: list     # [nwork]
    unit_part0: list    # [units]
    unit_nparts: list   # [units]


def plan_work(seg_arr, nseg: int, units: int, chunk_b: int) -> WorkPlan:
    """Split-kernel work list for a host segment table (dq_attention_plan)."""
    nwork, total = ctypes.c_int32(), ctypes.c_int32()
    p0 = (ctypes.c_int32 * max(units, 1))()
    npt = (ctypes.c_int32 * max(units, 1))()
    check(lib().dq_attention_plan(seg_arr, nseg, units, chunk_b, 0, None, ctypes.byref(nwork), None, p0, npt,
                                  ctypes.byref(total)), "attention_plan")
    n = nwork.value
    work = (ctypes.c_int32 * max(3 * n, 3))()
    wpart = (ctypes.c_int32 * max(n, 1))()
    check(lib().dq_attention_plan(seg_arr, nseg, units, chunk_b, n, work, ctypes.byref(nwork), wpart, p0, npt,
                                  ctypes.byref(total)), "attention_plan")
    return WorkPlan(n, total.value, list(work)[:3 * n], list(wpart)[:n], list(p0)[:units], list(npt)[:units])


def split_tail(wp: WorkPlan, seg_units, nsplit: int) -> WorkPlan:
    """``wp`` with its last ``nsplit`` items split into two halves each, queued after the
    others: the scheduler's last round then runs half-length items.  Partial slots are
    renumbered per unit in work-list order (dq_attention_plan's rule)."""
    big, small = [], []
    for i in range(wp.nwork):
        s, b0, t = wp.work[3 * i: 3 * i + 3]
        if i < wp.nwork - nsplit or t < 2:
            big.append((s, b0, t))
        else:
            h = t // 2
            small += [(s, b0, h), (s, b0 + h * 64, t - h)]
    items = big + small
    units = len(wp.unit_part0)
    npt = [0] * units
    for s, _, _ in items:
        npt[seg_units[s]] += 1
    p0, acc = [], 0
    for u in range(units):
        p0.append(acc)
        acc += npt[u]
    cur = list(p0)
    wpart = []
    for s, _, _ in items:
        wpart.append(cur[seg_units[s]])
        cur[seg_units[s]] += 1
    return WorkPlan(len(items), acc, [x for it in items for x in it], wpart, p0, npt)


class DecodeKvCache:
    """Device DecoQuant KV cache for ``layers`` x ``units`` with fused decode attention.

    ``g`` query heads share each kv head (GQA group).  ``bits`` in {2, 4, 8}.
    """

    def __init__(self, layers: int, units: int, g: int = 1, bits: int = 4, chunk_len: int = 1024,
                 dim: int = HEAD_DIM, chunk_b: int | None = None, sm_scale: float | None = None,
                 ctas: int | None = None, kernel_g: int | None = None, tc: bool | None = None, asym: bool = False):
        if dim != HEAD_DIM:
            raise Unsupported("the fused decode kernel is specialised for head_dim 128 (j = (8, 16))")
        if not 1 <= g <= MAX_G:
            raise Unsupported(f"GQA groups of 1..{MAX_G} query heads per kv head are supported (got {g})")
        if chunk_b is not None and (chunk_b % 64 or not 64 <= chunk_b <= MAX_CHUNK_B):
            raise Unsupported(f"work items must be 64..{MAX_CHUNK_B} rows, a multiple of 64")
        if bits not in SUPPORTED_BITS:
            raise UnsupportedBits(f"bits must be in {SUPPORTED_BITS}")
        if layers < 1 or units < 1 or chunk_len < 1:
            raise ShapeMismatch("layers, units and chunk_len must be >= 1")
        self.device = _lib.require_cuda()
        self.layers, self.units, self.g, self.bits = layers, units, g, bits
        # the split kernel runs kernel_g heads at a time; g > kernel_g becomes head_groups
        # virtual units per kv head that share its segments (their re-reads of the codes are L2
        # hits: the work list puts a tile range's head groups next to each other).
        # kernel_g = 8 is the tcgen05 GQA kernel (path 2: 4-bit codes, full plans i1 = 8,
        # r = 64); a layer whose segments do not qualify falls back to mma.sync heads of 2.
        # asym: the opt-in per-channel asymmetric quantizer (north_star; the reference's own scheme,
        # per-tensor symmetric, is the default and the parity mode).  2- / 4-bit, mma.sync kernel.
        self.asym = bool(asym)
        if self.asym and (bits not in (2, 4) or tc or (kernel_g or 1) > 2):
            raise Unsupported("the asymmetric mode covers 2- / 4-bit codes on the mma.sync split kernel (g <= 2)")
        if kernel_g is None:
            kernel_g = (GQA_G if (g % GQA_G == 0 and bits == 4 and tc is not False and not self.asym)
                        else (2 if g % 2 == 0 else 1))
        self.kernel_g = kernel_g
        if self.kernel_g not in KERNEL_G or g % self.kernel_g:
            raise Unsupported(f"kernel_g must be in {KERNEL_G} and divide g")
        if self.kernel_g == GQA_G and (bits != 4 or tc is False):
            raise Unsupported("kernel_g = 8 is the tcgen05 GQA kernel: 4-bit codes, tc not False")
        self.head_groups = g // self.kernel_g
        # split kernel for kernel_g = 1: tcgen05 (path 1) for 4-bit codes and the full plan
        # (i1 = 8, r = 64 -- any segment of >= 512 tokens with 8 | T), mma.sync (path 0)
        # otherwise.  True = tcgen05 (required), None / False = mma.sync (path 1 is correct but
        # not yet faster).  kernel_g = 8 always runs tcgen05 (path 2).
        self.tc = tc
        self.split_ctas = None
        self.chunk_len, self.dim, self.chunk_b = chunk_len, dim, chunk_b
        # split-kernel grid: None = persistent (resident CTAs of this device), 0 = one CTA
        # per work item, k > 0 = k persistent CTAs
        self.ctas = ctas
        self.sm_scale = float(sm_scale) if sm_scale is not None else float(1.0 / math.sqrt(dim))
        self._layers = [_Layer() for _ in range(layers)]
        shape = (layers, units, chunk_len, dim)
        self.tail_k = torch.zeros(shape, dtype=torch.float16, device=self.device)
        self.tail_v = torch.zeros(shape, dtype=torch.float16, device=self.device)
        self.tail_len = torch.zeros((layers, units), dtype=torch.int32, device=self.device)
        self.bytes_moved_read = 0
        self._pending = []  # deferred seal error words: (pinned host copy, event, layer)

    # ---- lifecycle -----------------------------------------------------------
    def _layer(self, layer: int) -> _Layer:
        if not 0 <= layer < self.layers:
            raise LayerOutOfRange(f"layer {layer} outside 0..{self.layers - 1}")
        return self._layers[layer]

    def tokens(self, layer: int) -> int:
        lay = self._layer(layer)
        return lay.tokens_sealed + lay.tail_len

    def _add_group(self, layer: int, keys: torch.Tensor, values: torch.Tensor, deferred: bool = False):
        """Compress (units, T, 128) K / V into a new segment group of ``layer`` (a list of layers
        with keys / values (len(layers) * units, T, 128): one batched K3 call for all of them).
        ``deferred`` (seals inside decoding): no host sync -- the device error word is copied back
        asynchronously and raised by the first later call that finds it on the host."""
        layers = layer if isinstance(layer, list) else [layer]
        for ly in layers:
            self._layer(ly)
        T = keys.shape[1]
        flags = torch.zeros(1, dtype=torch.int32, device=self.device) if deferred else None
        # fp32 G0 on the score side: scores of outlier-heavy keys are large, and the fp16
        # rounding of G0k (2^-11) would show up as absolute logit error
        kres = compress_blocks(keys, self.bits, _lib.LAYOUT_KTILE, torch.float32, self.asym, flags)
        vres = compress_blocks(values, self.bits, _lib.LAYOUT_VTILE, torch.float32, self.asym, flags)
        if deferred:
            host = torch.empty(1, dtype=torch.int32, pin_memory=True)
            host.copy_(flags, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self._pending.append((host, ev, layers))
        p = kres[5]
        i2p = -(-p.i2 // _lib.I2_PAD) * _lib.I2_PAD
        U = self.units
        for i, ly in enumerate(layers):
            lay = self._layers[ly]
            sl = slice(i * U, (i + 1) * U)
            kp, kc0, kg, kn, ks = (x[sl] for x in kres[:5])
            vp, vc0, vg, vn, vs = (x[sl] for x in vres[:5])
            kch, vch = (kres[6][sl], vres[6][sl]) if self.asym else (None, None)
            lay.groups.append(SegmentGroup(T, p, i2p, kp, vp, kc0, vc0, kg, vg, ks, vs, kn, vn, lay.tokens_sealed,
                                           kch, vch))
            lay.tokens_sealed += T
            lay.args = None
            lay.gen += 1

    def _flush_seals(self):
        """Seal every full tail (kvcache.py:124-128) in ONE batched K3 call.  A tail that reaches
        chunk_len stays in place until its layer is next read or written; in lock-step decoding
        every layer fills at the same step, so all of them compress together (32 x 1024 blocks at
        C2 instead of 32 calls of 1024: the eigensolver's one CTA per block then runs in full
        waves).  Results are identical to sealing at the append (the reference's point)."""
        full = [ly for ly, lay in enumerate(self._layers) if lay.seal_pending]
        if not full:
            return
        runs = []  # contiguous layer runs: their tails are one (n * units, chunk, 128) view
        for ly in full:
            if runs and runs[-1][-1] == ly - 1:
                runs[-1].append(ly)
            else:
                runs.append([ly])
        for run in runs:
            a, b = run[0], run[-1] + 1
            self._add_group(run, self.tail_k[a:b].reshape(-1, self.chunk_len, self.dim),
                            self.tail_v[a:b].reshape(-1, self.chunk_len, self.dim), deferred=True)
            self.tail_len[a:b].zero_()
            for ly in run:
                self._layers[ly].tail_len = 0
                self._layers[ly].seal_pending = False

    def prefill(self, layer: int, keys: torch.Tensor, values: torch.Tensor):
        """keys/values: (units, T, 128) CUDA fp16 or fp32.  One segment per unit (kvcache.py:99-114)."""
        lay = self._layer(layer)
        if lay.tokens_sealed or lay.tail_len:
            raise AlreadyPrefilled("layer already holds tokens")
        if keys.shape != values.shape or keys.ndim != 3 or keys.shape[0] != self.units:
            raise DimMismatch(f"keys and values must both be ({self.units}, T, {self.dim})")
        if keys.shape[2] != self.dim:
            raise DimMismatch(f"row width {keys.shape[2]} differs from dim {self.dim}")
        if keys.shape[1] == 0:
            return
        self._add_group(layer, keys.to(self.device), values.to(self.device))

    def append_token(self, layer: int, k_rows: torch.Tensor, v_rows: torch.Tensor):
        """k_rows/v_rows: (units, 128).  Seals the tail at chunk_len (kvcache.py:116-128)."""
        if self._layer(layer).seal_pending:
            self._flush_seals()
        if self._pending:
            self._check_seals()
        k, v = self._rows(k_rows, v_rows)
        check(lib().dq_tail_append(ptr(k), ptr(v), self.units, ptr(self.tail_k[layer]), ptr(self.tail_v[layer]),
                                   ptr(self.tail_len[layer]), self.chunk_len, stream_ptr()), "tail_append")
        self._after_append(layer)

    def extend_tail(self, layer: int, k_rows: torch.Tensor, v_rows: torch.Tensor):
        """Append n tokens per unit at once (k_rows / v_rows: (units, n, 128)): the same state as n
        append_token calls that do not reach chunk_len (the seal, kvcache.py:124-128, stays with
        the single-token path)."""
        lay = self._layer(layer)
        if lay.seal_pending:
            self._flush_seals()
        n = k_rows.shape[1] if k_rows.ndim == 3 else -1
        if k_rows.shape != (self.units, n, self.dim) or v_rows.shape != k_rows.shape:
            raise DimMismatch(f"rows must be ({self.units}, n, {self.dim})")
        if lay.tail_len + n >= self.chunk_len:
            raise ShapeMismatch("extend_tail would reach chunk_len: append the sealing token with append_token")
        t0 = lay.tail_len
        self.tail_k[layer, :, t0:t0 + n].copy_(k_rows)
        self.tail_v[layer, :, t0:t0 + n].copy_(v_rows)
        self.tail_len[layer].add_(n)
        lay.tail_len += n

    def _rows(self, k_rows: torch.Tensor, v_rows: torch.Tensor):
        if k_rows.shape != (self.units, self.dim) or v_rows.shape != (self.units, self.dim):
            raise DimMismatch(f"rows must be ({self.units}, {self.dim})")
        return (k_rows.to(self.device, torch.float16).contiguous(), v_rows.to(self.device, torch.float16).contiguous())

    def _check_seals(self, wait: bool = False):
        """Raise the error of a deferred seal whose device flags have reached the host."""
        pending, self._pending = self._pending, []
        for i, (host, ev, layer) in enumerate(pending):
            if wait:
                ev.synchronize()
            if ev.query():
                if int(host.item()):
                    self._pending += pending[i + 1:]  # raise once; the later seals stay pending
                    _lib.raise_flags(int(host.item()), f"deco_quantize (chunk sealed in layers {layer})")
            else:
                self._pending.append((host, ev, layer))

    def check_errors(self):
        """Seal any full tail, wait for every deferred seal and raise its error, if any (the
        reference raises inside append_token; a seal inside decoding reports at the first later
        call that sees it)."""
        self._flush_seals()
        self._check_seals(wait=True)

    def _after_append(self, layer: int):
        lay = self._layers[layer]
        lay.tail_len += 1
        if lay.tail_len == self.chunk_len:
            lay.seal_pending = True  # compressed by _flush_seals before this layer is used again

    def import_segment(self, layer: int, keys: list, values: list):
        """Append one sealed segment per unit from reference-form chains (``QuantizedMpo``, n = 2,
        e.g. ``formats.read_mpo`` of a DQZ1 file the reference wrote): the wire-order payloads
        are relaid into the attention layouts on the device, core0 into the normalised G0.

        ``keys[u]`` / ``values[u]``: unit u's K / V chain; every chain must cover the same T rows
        of ``dim`` columns at this cache's bits (one segment group, kvcache.py:124-128)."""
        lay = self._layer(layer)
        if self.asym:
            raise Unsupported("reference chains carry one symmetric scale: not an asymmetric cache")
        if len(keys) != self.units or len(values) != self.units:
            raise DimMismatch(f"need one K and one V chain per unit ({self.units})")
        chains = list(keys) + list(values)
        T = chains[0].rows
        for q in chains:
            if q.plan.n != 2 or q.cols != self.dim or q.rows != T:
                raise ShapeMismatch(f"every chain must be an n = 2 chain of ({T}, {self.dim})")
            if q.bits != self.bits:
                raise UnsupportedBits(f"chain bits {q.bits} differ from the cache's {self.bits}")
        if lay.tail_len:
            raise AlreadyPrefilled("import a segment before decoding into the tail")
        p = _lib.plan2(T, self.dim)
        U, dev = self.units, self.device
        nbytes = payload_size(p.r * p.i2 * p.j2, self.bits)

        def stack(which):
            qs = chains[:U] if which == "k" else chains[U:]
            wire = torch.stack([torch.as_tensor(q.local_tensors[1].data, device=dev).reshape(-1) for q in qs])
            if wire.shape[1] != nbytes:
                raise ShapeMismatch("payload size disagrees with the plan")
            layout = _lib.LAYOUT_KTILE if which == "k" else _lib.LAYOUT_VTILE
            lb = _lib.layout_bytes(p, self.bits, layout)
            dst = torch.empty((U, lb), dtype=torch.uint8, device=dev)
            check(lib().dq_relayout(ptr(wire), _lib.LAYOUT_REF, nbytes, ptr(dst), layout, lb, U,
                                    ctypes.byref(p), self.bits, stream_ptr()), "relayout")
            core0 = torch.stack([torch.as_tensor(q.local_tensors[0], dtype=torch.float32, device=dev).reshape(-1)
                                 for q in qs]).reshape(U, 1, p.i1, p.j1, p.r).contiguous()
            g0 = torch.empty((U, p.i1 * p.r * p.j1), dtype=torch.float32, device=dev)
            norm = torch.empty(U, dtype=torch.float32, device=dev)
            check(lib().dq_core0_relayout(ptr(core0), U, ctypes.byref(p), ptr(g0), _lib.DQ_F32, ptr(norm),
                                          stream_ptr()), "core0_relayout")
            scale = torch.tensor([q.local_tensors[1].scale for q in qs], dtype=torch.float32, device=dev)
            return dst, core0, g0, norm, scale

        kp, kc0, kg, kn, ks = stack("k")
        vp, vc0, vg, vn, vs = stack("v")
        i2p = -(-p.i2 // _lib.I2_PAD) * _lib.I2_PAD
        lay.groups.append(SegmentGroup(T, p, i2p, kp, vp, kc0, vc0, kg, vg, ks, vs, kn, vn, lay.tokens_sealed))
        lay.tokens_sealed += T
        lay.args = None
        lay.gen += 1

    # ---- attention -----------------------------------------------------------
    def _build_args(self, layer: int):
        lay = self._layers[layer]
        full_plans = all(grp.plan.i1 == 8 and grp.plan.r == 64 for grp in lay.groups)
        gk = self.kernel_g
        if gk == GQA_G and not full_plans:
            if self.tc:
                raise Unsupported("the tcgen05 GQA path needs i1 = 8, r = 64 plans (8 | T, T >= 512)")
            gk = 2  # mma.sync fallback for this layer
        hg = self.g // gk
        vunits = self.units * hg
        lay.kernel_g = gk
        if gk == GQA_G:
            path = 2
        else:
            eligible = self.bits == 4 and gk == 1 and full_plans
            if self.tc and not eligible:
                raise Unsupported("the tcgen05 path needs 4-bit codes, one head (or 8) per kernel and i1 = 8, "
                                  "r = 64 plans")
            path = 1 if (eligible and self.tc) else 0


        # the segment table, built column-wise (numpy view of the dq_segment records): one record
        # per (group, unit, head group); the scales are filled in on the device below (no sync)
        nseg = len(lay.groups) * vunits
        seg_arr = (_lib.Segment * max(nseg, 1))()
        rec = np.frombuffer(seg_arr, dtype=_SEG_DTYPE, count=nseg) if nseg else None
        u_of = np.repeat(np.arange(self.units, dtype=np.int64), hg)
        for gi, grp in enumerate(lay.groups):
            p = grp.plan
            r = rec[gi * vunits:(gi + 1) * vunits]
            r["k_codes"] = grp.k_payload.data_ptr() + u_of * grp.k_payload.shape[1]
            r["v_codes"] = grp.v_payload.data_ptr() + u_of * grp.v_payload.shape[1]
            r["k_g0"] = grp.k_g0h.data_ptr() + u_of * grp.k_g0h.shape[1] * grp.k_g0h.element_size()
            r["v_g0"] = grp.v_g0h.data_ptr() + u_of * grp.v_g0h.shape[1] * grp.v_g0h.element_size()
            r["T"], r["i1"], r["i2"], r["r"], r["i2p"] = grp.T, p.i1, p.i2, p.r, grp.i2p
            r["unit"] = np.arange(vunits, dtype=np.int32)
            r["token0"] = grp.token0
            if grp.k_ch is not None:
                r["k_ch"] = grp.k_ch.data_ptr() + u_of * grp.k_ch[0].numel() * 4
                r["v_ch"] = grp.v_ch.data_ptr() + u_of * grp.v_ch[0].numel() * 4
        # work plan (host) -> device tables
        ctas = self.ctas
        if ctas is None:
            c = ctypes.c_int32()
            check(lib().dq_attention_ctas(gk, self.bits, ctypes.byref(c)), "attention_ctas")
            ctas = c.value
        self.split_ctas = ctas
        # the largest items: the per-item cost (W image, softmax, epilogue) is fixed, and
        # smaller items measured slower even where they shorten the scheduler's last round.
        # 2-bit codes carry half the bytes per row, so their items are 512 rows (C3: 0.387 ->
        # 0.453 of HBM).  At 4 bits 512-row items win only where the 256-row plan needs 1.5 to 2
        # rounds of the persistent grid, so that halving the item count fills one round
        # (scripts/chunk_sweep.py: 32 units x 32K 45.7 -> 40.9 us, 256 x 4K 45.9 -> 43.1 us);
        # with fewer items the grid idles (16 x 32K: 26.9 -> 37.7 us) and with more the
        # fixed cost saved does not repay the coarser last round (512 x 4K: 74.3 -> 79.1 us)
        path0 = gk == 1 and not (self.tc and self.bits == 4 and full_plans)
        chunk_b = self.chunk_b or (MAX_CHUNK_B if self.bits == 2 and gk == 1 else DEFAULT_CHUNK_B)
        wp = plan_work(seg_arr, nseg, vunits, chunk_b)
        if (self.chunk_b is None and self.bits == 4 and path0 and not self.asym
                and 1.5 * ctas <= wp.nwork <= 2 * ctas):
            chunk_b = MAX_CHUNK_B
            wp = plan_work(seg_arr, nseg, vunits, chunk_b)
        if (self.chunk_b is None and self.bits == 4 and path0 and not self.asym and chunk_b == DEFAULT_CHUNK_B
                and 2 * wp.nwork < ctas):
            # under half a round of 256-row items (a strong-scaling shard: C4 at 4 / 8 GPUs holds
            # 8 / 4 units per layer) the layer is one item's latency; 128-row items spread it
            # over twice the SMs (scripts/chunk_sweep.py: 8 x 32K 22.8 -> 21.6 us, 4 x 32K
            # 17.8 -> 16.9 us; 64-row items lose: 30.3 / 21.2 us)
            chunk_b = DEFAULT_CHUNK_B // 2
            wp = plan_work(seg_arr, nseg, vunits, chunk_b)
        if self.chunk_b is None and chunk_b == MAX_CHUNK_B and path0 and wp.nwork > 2 * ctas:
            # several rounds of 512-row items: the last TAIL_SPLIT x grid items run as 256-row
            # halves, evening out the scheduler's last round (C3: 230.2 -> 225.7 us; at 256-row
            # items the 128-row halves cost more than they save: C2 64.3 -> 68.5 us)
            wp = split_tail(wp, rec["unit"].tolist(), int(TAIL_SPLIT * ctas))
        g0dt = ctypes.c_int32()
        check(lib().dq_attention_g0v_dtype(gk, path, 1 if self.asym else 0, chunk_b, ctypes.byref(g0dt)),
              "g0v_dtype")
        if g0dt.value == _lib.DQ_F16:  # the split kernel folds an fp16 copy of G0v (made once per group)
            for gi, grp in enumerate(lay.groups):
                if grp.v_g0f16 is None:
                    grp.v_g0f16 = grp.v_g0h.to(torch.float16)
                vg = grp.v_g0f16
                rec[gi * vunits:(gi + 1) * vunits]["v_g0"] = vg.data_ptr() + u_of * vg.shape[1] * vg.element_size()
        if hg > 1:  # a tile range's head groups back to back in the ticket order (L2 reuse)
            order = sorted(range(wp.nwork), key=lambda i: (wp.work[3 * i] // hg, wp.work[3 * i + 1],
                                                           wp.work[3 * i] % hg))
            wp.work = [x for i in order for x in wp.work[3 * i: 3 * i + 3]]
            wp.work_part = [wp.work_part[i] for i in order]
        dev = self.device

        staged = []  # pinned host copies: the uploads do not wait for the stream

        def up(host: torch.Tensor) -> torch.Tensor:
            h = host.pin_memory()
            staged.append(h)
            return h.to(dev, non_blocking=True)

        def i32(arr, n):
            return up(torch.tensor(list(arr)[:n], dtype=torch.int32))

        seg_dev = up(torch.frombuffer(bytearray(bytes(seg_arr)), dtype=torch.uint8))
        if nseg:  # the kernel sees g0h = core0 / norm: each segment's scale carries the norm back
            rec_f = seg_dev[:nseg * ctypes.sizeof(_lib.Segment)].view(torch.float32).view(nseg, -1)
            ko, vo = _lib.Segment.k_scale.offset // 4, _lib.Segment.v_scale.offset // 4
            rec_f[:, ko] = torch.cat([(g.k_scale * g.k_norm).repeat_interleave(hg) for g in lay.groups])
            rec_f[:, vo] = torch.cat([(g.v_scale * g.v_norm).repeat_interleave(hg) for g in lay.groups])
        nwork = wp.nwork
        work_dev = i32(wp.work, 3 * nwork)
        wpart_dev = i32(wp.work_part, nwork)
        sched = torch.zeros(2, dtype=torch.int32, device=dev)
        p0_dev = i32(wp.unit_part0, vunits)
        np_dev = i32(wp.unit_nparts, vunits)
        tp = max(wp.total_parts, 1)
        part_o = torch.empty((tp, gk, self.dim), dtype=torch.float32, device=dev)
        part_ml = torch.empty((tp, gk, 2), dtype=torch.float32, device=dev)
        a = _lib.AttnArgs()
        a.segs = seg_dev.data_ptr()
        a.nseg = nseg
        a.units = vunits
        a.g = gk
        a.head_groups = hg
        a.path = path
        a.bits = self.bits
        a.asym = 1 if self.asym else 0
        a.tail_k = self.tail_k[layer].data_ptr()
        a.tail_v = self.tail_v[layer].data_ptr()
        a.tail_len = self.tail_len[layer].data_ptr()
        a.tail_cap = self.chunk_len
        a.chunk_b = chunk_b
        a.sm_scale = self.sm_scale
        a.work = work_dev.data_ptr() if nwork else None
        a.nwork = nwork
        a.sched = sched.data_ptr()
        a.nctas = ctas
        a.max_parts = tp
        a.unit_part0 = p0_dev.data_ptr()
        a.work_part = wpart_dev.data_ptr() if nwork else None
        a.unit_nparts = np_dev.data_ptr()
        a.part_o = part_o.data_ptr()
        a.part_ml = part_ml.data_ptr()
        wib = ctypes.c_int64()
        check(lib().dq_attention_wimg_bytes(gk, ctypes.byref(wib)), "wimg_bytes")
        wimg = torch.empty((max(nseg, 1), wib.value), dtype=torch.uint8, device=dev)
        a.wimg = wimg.data_ptr()
        a.wimg_stride = wib.value
        lay.args = a
        lay.gen += 1
        lay.keep = [seg_dev, work_dev, wpart_dev, sched, p0_dev, np_dev, part_o, part_ml, wimg, *staged]

    def attend(self, layer: int, q: torch.Tensor, out: torch.Tensor | None = None,
               append: tuple[torch.Tensor, torch.Tensor] | None = None,
               out_dtype: torch.dtype = torch.float16) -> torch.Tensor:
        """q: (units, g, 128) fp16 CUDA -> (units, g, 128) fp16 (or ``out_dtype=torch.bfloat16``:
        the combine kernel rounds the merged fp32 output to bf16 once, for bf16 projections).

        ``append=(k_rows, v_rows)`` (each (units, 128)) fuses ``append_token`` into the same
        launch: the rows join the tail after this attention, exactly as attend + append_token.
        """
        lay = self._layer(layer)
        if lay.seal_pending:
            self._flush_seals()
        if self._pending:
            self._check_seals()
        if q.shape != (self.units, self.g, self.dim):
            raise DimMismatch(f"q must be ({self.units}, {self.g}, {self.dim})")
        if lay.args is None:
            self._build_args(layer)
        q = q.to(self.device, torch.float16).contiguous()
        if out_dtype not in (torch.float16, torch.bfloat16):
            raise Unsupported("out_dtype must be torch.float16 or torch.bfloat16")
        if out is None:
            out = torch.empty(q.shape, dtype=out_dtype, device=q.device)
        elif out.dtype != out_dtype or out.shape != q.shape or not out.is_contiguous():
            raise DimMismatch(f"out must be a contiguous {tuple(q.shape)} {out_dtype} tensor")
        a = lay.args
        a.q = q.data_ptr()
        a.out = out.data_ptr()
        a.out_bf16 = 1 if out_dtype == torch.bfloat16 else 0
        if append is not None:
            k, v = self._rows(*append)
            a.app_k, a.app_v = k.data_ptr(), v.data_ptr()
        try:
            check(lib().dq_decode_attention(ctypes.byref(a), stream_ptr()), "decode_attention")
        finally:
            a.app_k = a.app_v = None
            a.out_bf16 = 0
        self.bytes_moved_read += self.read_bytes(layer)
        if append is not None:
            self._after_append(layer)
        return out

    def launch(self, layer: int, q: torch.Tensor, out: torch.Tensor, phases: int = 3):
        """Low-level launch (bench/profiling): phases bit 0 = split kernel, bit 1 = combine."""
        lay = self._layers[layer]
        if lay.seal_pending:
            self._flush_seals()
        if lay.args is None:
            self._build_args(layer)
        a = lay.args
        a.q, a.out, a.phases = q.data_ptr(), out.data_ptr(), phases
        check(lib().dq_decode_attention(ctypes.byref(a), stream_ptr()), "decode_attention")
        a.phases = 0

    def clone_layer(self, src: int, dst: int):
        """Copy layer ``src``'s sealed segments into empty layer ``dst`` (distinct device memory)."""
        self._flush_seals()
        s, d = self._layer(src), self._layer(dst)
        if d.groups or d.tail_len:
            raise AlreadyPrefilled("destination layer already holds tokens")
        for grp in s.groups:
            fields = {k: (v.clone() if isinstance(v, torch.Tensor) else v) for k, v in grp.__dict__.items()}
            d.groups.append(SegmentGroup(**fields))
        d.tokens_sealed = s.tokens_sealed
        d.args = None
        d.gen += 1

    # ---- accounting ----------------------------------------------------------
    def kernel_bytes(self, layer: int) -> int:
        """Algorithmic bytes of one split-kernel launch: per unit and segment, K and V
        each 128*T*bits/8 code bytes + the small core as fp16 (2*i1*8*r) + a 4-byte scale, plus q.
        (The build stores the small cores as fp32, and the split kernel reads G0v but not G0k:
        ``stream_bytes`` counts what it streams.)"""
        lay = self._layers[layer]
        per = sum(2 * (payload_size(g.plan.r * g.plan.i2 * g.plan.j2, self.bits) + 2 * g.plan.i1 * 8 * g.plan.r + 4)
                  for g in lay.groups)
        return per * self.units + self.units * self.g * self.dim * 2

    def stream_bytes(self, layer: int) -> int:
        """Bytes one split-kernel launch is given to stream: packed cores, fp32 G0k and G0v, scales, q."""
        lay = self._layers[layer]
        return sum(g.stream_bytes() for g in lay.groups) * self.units + self.units * self.g * self.dim * 2

    def read_bytes(self, layer: int) -> int:
        """Algorithmic HBM bytes one ``attend(layer)`` streams (all units)."""
        lay = self._layers[layer]
        seg = sum(g.stream_bytes() for g in lay.groups) * self.units
        tail = 2 * lay.tail_len * self.dim * 2 * self.units
        qo = 2 * self.units * self.g * self.dim * 2
        return seg + tail + qo

    def ledger(self):
        self._flush_seals()
        return self._ledger()

    def _ledger(self):
        """(bytes_fp16_equivalent, bytes_actual) with the reference's accounting (kvcache.py:130-141)."""
        fp16 = actual = 0
        for lay in self._layers:
            tokens = lay.tokens_sealed + lay.tail_len
            fp16 += 2 * tokens * self.dim * 2 * self.units
            actual += sum(2 * g.reference_bytes(self.bits) for g in lay.groups) * self.units
            actual += 2 * lay.tail_len * self.dim * 2 * self.units
        return fp16, actual

    def export_segment(self, layer: int, index: int, unit: int, which: str = "k") -> QuantizedMpo:
        """Segment ``index`` of ``unit`` as a reference-form QuantizedMpo (wire-order payload)."""
        self._flush_seals()
        grp = self._layer(layer).groups[index]
        if grp.k_ch is not None:
            raise Unsupported("asymmetric segments have no reference (symmetric per-tensor) form")
        p = grp.plan
        src = grp.k_payload if which == "k" else grp.v_payload
        layout = _lib.LAYOUT_KTILE if which == "k" else _lib.LAYOUT_VTILE
        nbytes = payload_size(p.r * p.i2 * p.j2, self.bits)
        dst = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        check(lib().dq_relayout(ptr(src[unit]), layout, src.shape[1], ptr(dst), _lib.LAYOUT_REF, nbytes, 1,
                                ctypes.byref(p), self.bits, stream_ptr()), "relayout")
        core0 = (grp.k_core0 if which == "k" else grp.v_core0)[unit].reshape(1, p.i1, p.j1, p.r)
        scale = float((grp.k_scale if which == "k" else grp.v_scale)[unit].item())
        qt = QuantizedTensor((p.r, p.i2, p.j2, 1), self.bits, scale, data=dst, torch_out=True)
        return QuantizedMpo(plan=plan_shapes(grp.T, self.dim, 2), bits=self.bits, local_tensors=(core0, qt))


__all__ = ["DecodeKvCache", "SegmentGroup", "compress_blocks", "HEAD_DIM"]

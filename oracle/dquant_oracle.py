"""CPU oracle for the DecoQuant hot path.  TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import it.  The shipped path is the sm_100a
CUDA library behind ``include/dquant_b200.h``; it never routes through here.

It restates, in numpy, the algorithm of the reference package ``dquant``
(``/root/reference/pkg/src/dquant``, cited below as ``file:line``):

* codec ............ quantize.py:23-157   (symmetric per-tensor RTN, 2/4/8-bit
                                           two's-complement packing, low bits first)
* shape planning ... mpo.py:66-96, 54-63  (peel largest divisor <= 8, bond law)
* TT-SVD, n=2 ...... mpo.py:144-178       (interleave, fp64 LAPACK SVD, sqrt(s) split)
* chains n >= 2 .... mpo.py:144-198, compress.py:85-231 (sequential TT-SVD, contraction,
                                           DecoQuant of every core but the first, core sweeps)
* reconstruction ... mpo.py:181-198, compress.py:97-107
* DecoQuant ........ compress.py:85-94    (quantize every core but the first)
* fused reads ...... compress.py:159-231  (x @ W and x @ W^T, factored order)
* accounting ....... compress.py:234-248, kvcache.py:130-141
* KV cache ......... kvcache.py:45-225    (single prefill segment, fp tail,
                                           chunk trigger, streamed scores)
* decode attention . composition (not in the reference): scores from
                     kvcache.py:188-217, fp64 softmax, per-segment x @ W
                     (compress.py:159-192) plus the dense tail.

Third-party arithmetic: the SVD is ``numpy.linalg.svd`` -> LAPACK ``dgesdd``
(OpenBLAS bundled with numpy 2.3.x; the reference pins only ``numpy>=1.24``,
``pkg/pyproject.toml:10``).  This oracle calls the same routine, so its cores
are bit-identical to the reference's on the same machine.

Parity pinning: every function here is checked against golden vectors that
``tests/golden/make_golden.py`` produced by importing the reference itself
(see ``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import prod

import numpy as np

# quantize.py:23
BITS = (2, 4, 8)
# mpo.py:22
PEEL_CAP = 8


def qmax_of(bits: int) -> int:
    """Largest code magnitude; the code -2**(bits-1) is never produced (quantize.py:133)."""
    if bits not in BITS:
        raise ValueError(f"unsupported bits {bits}")
    return (1 << (bits - 1)) - 1


# ---------------------------------------------------------------------------
# codec
# ---------------------------------------------------------------------------


def payload_bytes(count: int, bits: int) -> int:
    """quantize.py:31-33."""
    return (count * bits + 7) // 8


def pack_codes(codes, bits: int) -> np.ndarray:
    """Two's complement in ``bits`` bits, element i at bit offset bits*(i % per).

    Restates quantize.py:66-82 with a lane-shift sum instead of a loop of ORs.
    Returns a uint8 array of ``payload_bytes(len(codes), bits)`` bytes.
    """
    c = np.asarray(codes, dtype=np.int64).reshape(-1)
    q = qmax_of(bits)
    if c.size and (c.min() < -q or c.max() > q):
        raise OverflowError("code outside the symmetric range")
    per = 8 // bits
    lanes = (c & ((1 << bits) - 1)).astype(np.uint32)
    pad = (-lanes.size) % per
    if pad:
        lanes = np.concatenate([lanes, np.zeros(pad, np.uint32)])
    lanes = lanes.reshape(-1, per)
    shifts = (np.arange(per, dtype=np.uint32) * bits)[None, :]
    return (lanes << shifts).sum(axis=1).astype(np.uint8)


def unpack_codes(payload, count: int, bits: int, start: int = 0) -> np.ndarray:
    """Codes [start, start+count) of a payload, sign-extended to int8.

    quantize.py:85-120 (``unpack`` is start=0 over the whole payload;
    ``unpack_range`` reads only the covering bytes).
    """
    buf = np.frombuffer(bytes(payload), dtype=np.uint8) if not isinstance(payload, np.ndarray) else payload.astype(np.uint8)
    per = 8 // bits
    idx = np.arange(start, start + count, dtype=np.int64)
    raw = (buf[idx // per].astype(np.int32) >> ((idx % per) * bits).astype(np.int32)) & ((1 << bits) - 1)
    sign = 1 << (bits - 1)
    return ((raw ^ sign) - sign).astype(np.int8)


def rtn(t, bits: int):
    """Symmetric round-half-away-from-zero with one per-tensor scale.

    quantize.py:123-151.  Returns (scale as np.float32, int8 codes with t's shape).
    The code is computed in fp64 as copysign(floor(|t*qmax/amax| + 0.5)), the
    product evaluated before the division (quantize.py:144) so exact ties stay exact.
    """
    t = np.asarray(t)
    q = qmax_of(bits)
    if t.size and not np.isfinite(t).all():
        raise FloatingPointError("non-finite input")
    amax = float(np.abs(t).max()) if t.size else 0.0
    scale = np.float32(amax / q) if amax > 0 else np.float32(1.0)
    if amax == 0.0 or scale == 0:
        return np.float32(1.0), np.zeros(t.shape, np.int8)
    y = (t.astype(np.float64) * q) / amax
    code = np.sign(y) * np.floor(np.abs(y) + 0.5)
    return scale, np.clip(code, -q, q).astype(np.int8)


def dequant(codes, scale) -> np.ndarray:
    """quantize.py:154-157: f32 codes times the f32 scale."""
    return np.asarray(codes).astype(np.float32) * np.float32(scale)


# ---------------------------------------------------------------------------
# shape planning and the n=2 tensor-train split
# ---------------------------------------------------------------------------


def peel(x: int, cap: int = PEEL_CAP) -> int:
    """Largest divisor of x not above cap (mpo.py:66-70)."""
    return next(d for d in range(min(cap, x), 0, -1) if x % d == 0)


def plan(rows: int, cols: int, n: int = 2):
    """(i_factors, j_factors) of mpo.py:73-96."""
    if rows < 1 or cols < 1 or n < 2:
        raise ValueError("bad plan request")

    def split(size):
        out = []
        for _ in range(n - 1):
            d = peel(size)
            out.append(d)
            size //= d
        return tuple(out + [size])

    return split(rows), split(cols)


def bonds(i_f, j_f):
    """ShapePlan.bond_dims (mpo.py:54-63)."""
    ij = [a * b for a, b in zip(i_f, j_f)]
    tot = prod(ij)
    out, left = [], 1
    for k in range(len(ij) - 1):
        left *= ij[k]
        out.append(min(left, tot // left))
    return tuple(out)


@dataclass
class Plan2:
    i1: int
    i2: int
    j1: int
    j2: int

    @property
    def r(self) -> int:
        return min(self.i1 * self.j1, self.i2 * self.j2)

    @classmethod
    def of(cls, rows: int, cols: int) -> "Plan2":
        (i1, i2), (j1, j2) = plan(rows, cols, 2)
        return cls(i1, i2, j1, j2)


def interleaved(m: np.ndarray, p: Plan2) -> np.ndarray:
    """A[(a,c),(b,e)] = M[a*i2+b, c*j2+e]  (mpo.py:144-150, 162-164)."""
    return m.reshape(p.i1, p.i2, p.j1, p.j2).transpose(0, 2, 1, 3).reshape(p.i1 * p.j1, p.i2 * p.j2)


def deinterleaved(a: np.ndarray, p: Plan2) -> np.ndarray:
    """Inverse of ``interleaved`` (mpo.py:191-196)."""
    return a.reshape(p.i1, p.j1, p.i2, p.j2).transpose(0, 2, 1, 3).reshape(p.i1 * p.i2, p.j1 * p.j2)


def tt_split2(m: np.ndarray, p: Plan2 | None = None):
    """Full-rank n=2 TT-SVD with the singular values split as sqrt(s) both ways.

    mpo.py:153-178: fp64 interleave, ``np.linalg.svd(full_matrices=False)``,
    core0 = U*sqrt(s) (1,i1,j1,r), core1 = sqrt(s)[:,None]*Vt (r,i2,j2,1), both cast to f32.
    Also returns the singular values (fp64) for diagnostics.
    """
    m = np.asarray(m, dtype=np.float32)
    p = p or Plan2.of(*m.shape)
    u, s, vt = np.linalg.svd(interleaved(m.astype(np.float64), p), full_matrices=False)
    rs = np.sqrt(s)
    core0 = (u * rs).reshape(1, p.i1, p.j1, len(s)).astype(np.float32)
    core1 = (rs[:, None] * vt).reshape(len(s), p.i2, p.j2, 1).astype(np.float32)
    return core0, core1, s


def contract2(core0: np.ndarray, core1: np.ndarray, p: Plan2) -> np.ndarray:
    """mpo.py:181-198 for n=2: fp64 G0 (i1*j1, r) @ G1 (r, i2*j2), de-interleave, f32."""
    r = core0.shape[-1]
    a = core0.astype(np.float64).reshape(p.i1 * p.j1, r) @ core1.astype(np.float64).reshape(r, p.i2 * p.j2)
    return np.ascontiguousarray(deinterleaved(a, p).astype(np.float32))


# ---------------------------------------------------------------------------
# chains of any length n >= 2
# ---------------------------------------------------------------------------


def tt_split(m: np.ndarray, i_f, j_f):
    """Full-rank sequential TT-SVD (mpo.py:153-178): interleave (144-150) in fp64, then per core
    the SVD of the carry reshaped to (d_prev * i_k * j_k, rest); core = U sqrt(s), carry =
    sqrt(s) Vt; the last core is the carry.  Cores cast to f32 (mpo.py:178)."""
    n = len(i_f)
    order = [x for k in range(n) for x in (k, n + k)]
    carry = np.transpose(np.asarray(m, np.float64).reshape(tuple(i_f) + tuple(j_f)), order)
    cores, d_prev = [], 1
    for k in range(n):
        mat = carry.reshape(d_prev * i_f[k] * j_f[k], -1)
        if k == n - 1:
            cores.append(mat.reshape(d_prev, i_f[k], j_f[k], 1))
            break
        u, s, vt = np.linalg.svd(mat, full_matrices=False)
        rs = np.sqrt(s)
        cores.append((u * rs).reshape(d_prev, i_f[k], j_f[k], len(s)))
        carry = rs[:, None] * vt
        d_prev = len(s)
    return [c.astype(np.float32) for c in cores]


def contract(cores) -> np.ndarray:
    """mpo.py:181-198: fp64 left-to-right contraction, de-interleave, f32."""
    return np.ascontiguousarray(contract_f64(cores).astype(np.float32))


def deco_chain(m: np.ndarray, bits: int, n: int):
    """compress.py:85-94 for any n: TT-SVD, then RTN of every core but the first.  Returns the
    first core and (codes, scale) per quantized core, plus the dequantized chain."""
    i_f, j_f = plan(*np.asarray(m).shape, n)
    cores = tt_split(m, i_f, j_f)
    quant = [rtn(c, bits) for c in cores[1:]]  # (scale, codes)
    deq = [cores[0]] + [dequant(codes, scale).reshape(c.shape) for (scale, codes), c in zip(quant, cores[1:])]
    return cores[0], quant, deq


def chain_matmul(x: np.ndarray, deq) -> np.ndarray:
    """x @ W through the dequantized cores (compress.py:159-192; the tiling is a memory bound,
    not arithmetic, so the dense restatement computes the same fp64 products)."""
    return (np.asarray(x, np.float64) @ contract_f64(deq)).astype(np.float32)


def chain_matmul_t(x: np.ndarray, deq) -> np.ndarray:
    """x @ W.T (compress.py:195-231)."""
    return (np.asarray(x, np.float64) @ contract_f64(deq).T).astype(np.float32)


def contract_f64(cores) -> np.ndarray:
    """mpo.py:181-198 without the final f32 cast."""
    c64 = [np.asarray(c, np.float64) for c in cores]
    cur = c64[0].reshape(-1, c64[0].shape[3])
    for t in c64[1:]:
        cur = (cur @ t.reshape(t.shape[0], -1)).reshape(-1, t.shape[3])
    i_f = [c.shape[1] for c in c64]
    j_f = [c.shape[2] for c in c64]
    n = len(c64)
    full = cur.reshape([x for a, b in zip(i_f, j_f) for x in (a, b)])
    full = np.transpose(full, [2 * k for k in range(n)] + [2 * k + 1 for k in range(n)])
    return full.reshape(prod(i_f), prod(j_f))


# ---------------------------------------------------------------------------
# DecoQuant encoding (n=2) and its reads
# ---------------------------------------------------------------------------


@dataclass
class Encoded:
    """One DecoQuant block: fp32 small core, packed large core, its scale."""

    plan: Plan2
    bits: int
    core0: np.ndarray  # (1, i1, j1, r) float32
    scale: np.float32
    codes: np.ndarray  # (r, i2, j2) int8, reference payload order (unsigned codes in the asymmetric mode)
    ch_scale: np.ndarray | None = None  # asymmetric mode: (r, j2) f32 channel scales
    ch_zero: np.ndarray | None = None   # asymmetric mode: (r, j2) zero points

    @property
    def r(self) -> int:
        return self.core0.shape[-1]

    @property
    def payload(self) -> bytes:
        return pack_codes(self.codes.reshape(-1), self.bits).tobytes()

    def g1(self) -> np.ndarray:
        """Dequantized core1 (r, i2, j2) in fp64."""
        if self.ch_scale is None:
            return self.codes.astype(np.float64) * np.float64(self.scale)
        return (self.codes.astype(np.float64) - self.ch_zero[:, None, :]) * self.ch_scale.astype(np.float64)[:, None, :]

    def core1_deq(self) -> np.ndarray:
        if self.ch_scale is None:
            return dequant(self.codes, self.scale).reshape(self.r, self.plan.i2, self.plan.j2, 1)
        return self.g1().astype(np.float32).reshape(self.r, self.plan.i2, self.plan.j2, 1)


def encode(m: np.ndarray, bits: int) -> Encoded:
    """compress.py:85-94 for n=2: plan, TT-SVD, quantize core1 with rtn."""
    m = np.asarray(m, dtype=np.float32)
    if m.ndim != 2:
        raise ValueError("expected a matrix")
    p = Plan2.of(*m.shape)
    core0, core1, _ = tt_split2(m, p)
    scale, codes = rtn(core1, bits)
    return Encoded(p, bits, core0, scale, codes.reshape(core1.shape[0], p.i2, p.j2))


def rtn_asym(core1, bits: int):
    """OPT-IN per-channel asymmetric quantizer (north_star's "per-channel asymmetric int4/int2";
    NOT in the reference, whose quantizer is per-tensor symmetric -- this restates the build's own
    K3 mode, include/dquant_b200.h dq_deco_quantize_asym_batched, so its parity is unpinned).
    Channel (r, e) of core1 (r, i2, j2) over b, qmu = 2^bits - 1, fp64 arithmetic:
    s = f32((max - min) / qmu) (|max| or 1 for a constant channel), z = clip(floor(-min/s + .5)),
    u = clip(floor(v/s + .5) + z, 0, qmu).  Returns (s (r, j2) f32, z (r, j2) int32, u uint8)."""
    c = np.asarray(core1, np.float32)
    qmu = (1 << bits) - 1
    mn, mx = c.min(axis=1), c.max(axis=1)
    rng = mx.astype(np.float64) - mn.astype(np.float64)
    s = np.where(rng > 0, rng / qmu, np.where(mx != 0, np.abs(mx).astype(np.float64), 1.0)).astype(np.float32)
    s64 = s.astype(np.float64)
    z = np.clip(np.floor(-mn.astype(np.float64) / s64 + 0.5), 0, qmu)
    u = np.clip(np.floor(c.astype(np.float64) / s64[:, None, :] + 0.5) + z[:, None, :], 0, qmu)
    return s, z.astype(np.int32), u.astype(np.uint8)


def encode_asym(m: np.ndarray, bits: int) -> Encoded:
    """``encode`` with the opt-in asymmetric per-channel quantizer (``rtn_asym``) on core1."""
    m = np.asarray(m, dtype=np.float32)
    p = Plan2.of(*m.shape)
    core0, core1, _ = tt_split2(m, p)
    c1 = core1.reshape(core1.shape[0], p.i2, p.j2)
    s, z, u = rtn_asym(c1, bits)
    return Encoded(p, bits, core0, np.float32(1.0), u, s, z)


def decode(e: Encoded) -> np.ndarray:
    """compress.py:105-107: dequantize core1 (f32) then contract2."""
    return contract2(e.core0, e.core1_deq(), e.plan)


def matmul_t(x: np.ndarray, e: Encoded) -> np.ndarray:
    """x @ W^T streamed core1-first (compress.py:195-231), fp64 accumulate, f32 out.

    out[p, a*i2+b] = sum_{c,r} G0[a,c,r] * sum_e scale*code[r,b,e] * x[p, c*j2+e]
    """
    pl = e.plan
    x64 = np.asarray(x, dtype=np.float64).reshape(-1, pl.j1, pl.j2)
    g1 = e.g1()  # (r, i2, j2)
    h = np.einsum("rbe,pce->prbc", g1, x64)
    g0 = e.core0.astype(np.float64).reshape(pl.i1, pl.j1, e.r)
    out = np.einsum("acr,prbc->pab", g0, h)
    return np.ascontiguousarray(out.reshape(x64.shape[0], pl.i1 * pl.i2).astype(np.float32))


def matmul(x: np.ndarray, e: Encoded) -> np.ndarray:
    """x @ W streamed core0-first (compress.py:159-192), fp64 accumulate, f32 out.

    out[p, c*j2+e] = sum_{a,b} x[p, a*i2+b] * sum_r G0[a,c,r] * scale*code[r,b,e]
    """
    pl = e.plan
    x64 = np.asarray(x, dtype=np.float64).reshape(-1, pl.i1, pl.i2)
    g0 = e.core0.astype(np.float64).reshape(pl.i1, pl.j1, e.r)
    y = np.einsum("pab,acr->pbcr", x64, g0)
    g1 = e.g1()
    out = np.einsum("pbcr,rbe->pce", y, g1)
    return np.ascontiguousarray(out.reshape(x64.shape[0], pl.j1 * pl.j2).astype(np.float32))


def ratio_report(e: Encoded):
    """compress.py:234-248: (mu, bytes_original, bytes_compressed) for n=2."""
    n_q = e.codes.size
    n_fp = e.core0.size
    num_bits = n_q * e.bits + n_fp * 16 + 16
    rows, cols = e.plan.i1 * e.plan.i2, e.plan.j1 * e.plan.j2
    return num_bits / (rows * cols * 16), rows * cols * 2, payload_bytes(n_q, e.bits) + 2 + 2 * n_fp


# ---------------------------------------------------------------------------
# KV cache semantics and decode attention
# ---------------------------------------------------------------------------


@dataclass
class LayerOracle:
    """kvcache.py:77-141: immutable segments plus a full-precision tail."""

    dim: int
    bits: int | None
    chunk_len: int
    k_segs: list = field(default_factory=list)
    v_segs: list = field(default_factory=list)
    rows: list = field(default_factory=list)
    tail_k: list = field(default_factory=list)
    tail_v: list = field(default_factory=list)
    asym: bool = False  # the build's opt-in per-channel asymmetric mode (encode_asym)

    def _seal(self, block):
        block = np.ascontiguousarray(block, dtype=np.float32)
        if self.bits is None:
            return block
        return encode_asym(block, self.bits) if self.asym else encode(block, self.bits)

    def prefill(self, k, v):
        """kvcache.py:99-114: the whole prompt becomes ONE segment."""
        if self.rows or self.tail_k:
            raise RuntimeError("already prefilled")
        k = np.asarray(k, np.float32)
        v = np.asarray(v, np.float32)
        if k.shape[0] == 0:
            return
        self.k_segs.append(self._seal(k))
        self.v_segs.append(self._seal(v))
        self.rows.append(k.shape[0])

    def append(self, k_row, v_row):
        """kvcache.py:116-128: tail grows; at chunk_len it is sealed."""
        self.tail_k.append(np.asarray(k_row, np.float32).reshape(-1))
        self.tail_v.append(np.asarray(v_row, np.float32).reshape(-1))
        if len(self.tail_k) == self.chunk_len:
            self.k_segs.append(self._seal(np.stack(self.tail_k)))
            self.v_segs.append(self._seal(np.stack(self.tail_v)))
            self.rows.append(self.chunk_len)
            self.tail_k, self.tail_v = [], []

    @property
    def tokens(self) -> int:
        return sum(self.rows) + len(self.tail_k)

    def read(self, which: str) -> np.ndarray:
        """kvcache.py:163-186: materialise every segment, then the tail."""
        segs = self.k_segs if which == "k" else self.v_segs
        tail = self.tail_k if which == "k" else self.tail_v
        parts = [s if isinstance(s, np.ndarray) else decode(s) for s in segs]
        if tail:
            parts.append(np.stack(tail))
        return np.concatenate(parts, 0) if parts else np.zeros((0, self.dim), np.float32)

    def scores(self, q) -> np.ndarray:
        """kvcache.py:188-217 generalised to g query rows: (g, T) f32, / f32(sqrt(D))."""
        q = np.asarray(q, np.float32).reshape(-1, self.dim)
        parts = []
        for s in self.k_segs:
            if isinstance(s, np.ndarray):
                parts.append((q.astype(np.float64) @ s.astype(np.float64).T).astype(np.float32))
            else:
                parts.append(matmul_t(q, s))
        if self.tail_k:
            parts.append((q.astype(np.float64) @ np.stack(self.tail_k).astype(np.float64).T).astype(np.float32))
        if not parts:
            return np.zeros((q.shape[0], 0), np.float32)
        return (np.concatenate(parts, 1) / np.float32(np.sqrt(self.dim))).astype(np.float32)

    def attend(self, q) -> np.ndarray:
        """Decode attention: softmax(scores) in fp64, then P @ V per segment (compress.py:159-192) + tail."""
        s = self.scores(q).astype(np.float64)
        p = np.exp(s - s.max(axis=1, keepdims=True))
        p /= p.sum(axis=1, keepdims=True)
        out = np.zeros((p.shape[0], self.dim), np.float64)
        off = 0
        for seg, n in zip(self.v_segs, self.rows):
            ps = p[:, off : off + n]
            out += ps @ seg.astype(np.float64) if isinstance(seg, np.ndarray) else matmul(ps, seg).astype(np.float64)
            off += n
        if self.tail_v:
            out += p[:, off:] @ np.stack(self.tail_v).astype(np.float64)
        return out.astype(np.float32)

    def ledger(self):
        """kvcache.py:130-141: (fp16-equivalent bytes, actual bytes)."""
        actual = 0
        for s in self.k_segs + self.v_segs:
            actual += s.size * 2 if isinstance(s, np.ndarray) else ratio_report(s)[2]
        actual += 2 * len(self.tail_k) * self.dim * 2
        return 2 * self.tokens * self.dim * 2, actual


def attention_units(q, k_blocks, v_blocks, bits):
    """Decode attention over independent single-segment units.

    q: (U, g, D); k_blocks/v_blocks: (U, T, D).  Returns (U, g, D) f32.  Used by
    the bench's CPU baseline and by the parity tests at small sizes.
    """
    out = []
    for u in range(q.shape[0]):
        lay = LayerOracle(q.shape[-1], bits, 1 << 30)
        lay.prefill(k_blocks[u], v_blocks[u])
        out.append(lay.attend(q[u]))
    return np.stack(out)

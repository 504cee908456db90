"""LLaMA-shaped decoder with a DecoQuant KV cache: the end-to-end decode harness.

Random-init weights (std 0.02, bf16) of the named shapes; one decode step per call:

    RMSNorm -> QKV projection -> RoPE -> fused DecoQuant attention (+ KV append) -> O projection
    -> residual -> RMSNorm -> SwiGLU MLP -> residual        (x layers), RMSNorm -> LM head -> argmax

The attention of every layer is ``DecodeKvCache.attend(layer, q, append=(k, v))``: the new
token's K/V join the fp16 tail and the compressed segments are read by the fused kernels.
Dense projections are cuBLAS GEMMs through torch (library code, as the task allows); the
elementwise work between them is three fused kernels of the C ABI (csrc/model.cu: residual
add + RMSNorm, QKV split + RoPE + fp16 cast, SwiGLU), so a layer is ten launches; the step
is capturable in one CUDA graph (``capture()`` / ``replay()``).

Tensor parallelism (``tp=TpGroup``, one process per GPU): rank k of N holds kv heads
[k*KV/N, (k+1)*KV/N) of every sequence with their query heads and compressed cache (the decode
attention exchanges nothing), and 1/N of every dense weight, split by output columns
(``sharding.shard_layer_weights``).  The step is written as a generator that yields each
sliced activation and receives it gathered (``TpGroup.gather``: NCCL all-gather over NVLink,
inside the captured graph): the attention heads, the O-projection and MLP hidden slices and
the SwiGLU ffn slice per layer, and the vocabulary slice's top-1 at the end.  With one rank
every gather is the identity and the step is the single-GPU harness.  ``Lockstep`` drives N
shard models in one process (each gather a concatenation of their slices): the device test of
the sharded step against the unsharded one.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from ._lib import check, lib, ptr, stream_ptr
from .attention import DecodeKvCache
from .errors import ShapeMismatch
from .sharding import TpGroup, shard_layer_weights, tp_slices


@dataclass(frozen=True)
class ModelShape:
    layers: int
    hidden: int
    heads: int
    kv_heads: int
    ffn: int
    vocab: int = 32000
    head_dim: int = 128

    @property
    def g(self) -> int:
        return self.heads // self.kv_heads


LLAMA2_7B = ModelShape(layers=32, hidden=4096, heads=32, kv_heads=32, ffn=11008)
LLAMA2_13B = ModelShape(layers=40, hidden=5120, heads=40, kv_heads=40, ffn=13824)
LLAMA2_70B = ModelShape(layers=80, hidden=8192, heads=64, kv_heads=8, ffn=28672)


def _rms(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype) * w


def _rope(x: torch.Tensor, pos: torch.Tensor, theta: float = 10000.0) -> torch.Tensor:
    """Rotary embedding of (..., head_dim) at one position (a device scalar, so the step is
    graph-capturable), half-split convention."""
    d = x.shape[-1]
    inv = theta ** (-torch.arange(0, d, 2, device=x.device, dtype=torch.float32) / d)
    ang = pos.float() * inv
    cos, sin = torch.cos(ang), torch.sin(ang)
    x1, x2 = x[..., : d // 2].float(), x[..., d // 2:].float()
    return torch.cat([x1 * cos - x2 * sin, x1 * sin + x2 * cos], -1).to(x.dtype)


class DecoQuantLM:
    """Decoder of ``shape`` for ``batch`` sequences whose KV cache is DecoQuant-compressed."""

    def __init__(self, shape: ModelShape, batch: int, bits: int = 4, chunk_len: int = 1024, seed: int = 0,
                 device="cuda", tp: TpGroup | None = None, weights: dict | None = None):
        if shape.head_dim != 128 or shape.heads % shape.kv_heads:
            raise ShapeMismatch("head_dim must be 128 and heads a multiple of kv_heads")
        self.shape, self.batch = shape, batch
        self.tp = tp or TpGroup(world=1, rank=0)
        world, rank = self.tp.world, self.tp.rank
        self.sl = tp_slices(shape, rank, world)
        lo, hi = self.sl["kv"]
        self.kv_local = hi - lo
        self.heads_local = self.kv_local * shape.g
        self.dev = torch.device(device)
        s = shape
        if weights is None:
            # random init of this rank's shard (std 0.02, bf16); ranks draw from their own streams
            gen = torch.Generator(device=self.dev).manual_seed(seed if world == 1 else seed * 1000003 + rank)
            hl, F, hs = self.heads_local * 128, s.ffn // world, s.hidden // world

            def w(*dims):
                return (torch.randn(dims, generator=gen, device=self.dev, dtype=torch.float32) * 0.02).to(torch.bfloat16)

            weights = {"embed": w(s.vocab, s.hidden), "lm_head": w(s.hidden, s.vocab // world), "layers": []}
            for _ in range(s.layers):
                weights["layers"].append({
                    "ln1": torch.ones(s.hidden, device=self.dev, dtype=torch.bfloat16),
                    "ln2": torch.ones(s.hidden, device=self.dev, dtype=torch.bfloat16),
                    "qkv": w(s.hidden, hl + 2 * self.kv_local * 128),
                    "o": w(s.heads * 128, hs),
                    "gate_up": w(s.hidden, 2 * F),
                    "down": w(s.ffn, hs),
                })
        self.embed, self.lm_head, self.layers = weights["embed"], weights["lm_head"], weights["layers"]
        self.norm = torch.ones(s.hidden, device=self.dev, dtype=torch.bfloat16)
        self.cache = DecodeKvCache(layers=s.layers, units=batch * self.kv_local, g=s.g, bits=bits,
                                   chunk_len=chunk_len)
        self.pos = torch.zeros((), dtype=torch.int64, device=self.dev)  # decode position (device)
        self.graph = None
        self._tok = self._next = None

    @classmethod
    def shard_of(cls, full: "DecoQuantLM", tp: TpGroup, bits: int = 4, chunk_len: int = 1024) -> "DecoQuantLM":
        """Rank tp.rank's shard of an unsharded model's weights (column slices, copied), with an
        empty cache of its kv heads: the parity harness of the sharded step."""
        s, r, n = full.shape, tp.rank, tp.world
        v0, v1 = tp_slices(s, r, n)["vocab"]
        weights = {"embed": full.embed, "lm_head": full.lm_head[:, v0:v1].contiguous(),
                   "layers": [shard_layer_weights(L, s, r, n) for L in full.layers]}
        return cls(s, full.batch, bits=bits, chunk_len=chunk_len, device=full.dev, tp=tp, weights=weights)

    def prefill_random(self, tokens: int, seed: int = 1):
        """Fill every layer's cache with `tokens` positions of synthetic K/V (N(0,1) fp16),
        compressed by the K3 write path (one segment per (sequence, kv head)).  The draw is the
        whole model's (batch x kv heads units); a tensor-parallel rank keeps its kv heads."""
        gen = torch.Generator(device=self.dev).manual_seed(seed)
        units = self.batch * self.shape.kv_heads
        for layer in range(self.shape.layers):
            k = torch.randn((units, tokens, 128), generator=gen, device=self.dev).to(torch.float16)
            v = torch.randn((units, tokens, 128), generator=gen, device=self.dev).to(torch.float16)
            self.prefill_units(layer, k, v)
        self.pos.fill_(tokens)

    def prefill_units(self, layer: int, k: torch.Tensor, v: torch.Tensor):
        """Prefill one layer from the whole model's (batch * kv_heads, T, 128) K / V; this rank
        compresses its kv heads' units only."""
        if self.tp.world > 1:
            lo, hi = self.sl["kv"]
            B, T = self.batch, k.shape[1]
            k = k.view(B, self.shape.kv_heads, T, 128)[:, lo:hi].reshape(B * self.kv_local, T, 128)
            v = v.view(B, self.shape.kv_heads, T, 128)[:, lo:hi].reshape(B * self.kv_local, T, 128)
        self.cache.prefill(layer, k, v)

    # ---- fused harness kernels (csrc/model.cu); _rms / _rope above are their torch statements
    def _norm(self, x: torch.Tensor, y: torch.Tensor | None, w: torch.Tensor) -> torch.Tensor:
        """x += y in place (y None: x as is); returns RMSNorm(x) * w."""
        h = torch.empty_like(x)
        check(lib().dq_model_add_rmsnorm(x.data_ptr(), ptr(y), w.data_ptr(), x.data_ptr(), h.data_ptr(),
                                         x.shape[0], x.shape[1], 1e-5, stream_ptr()), "add_rmsnorm")
        return h

    def _qkv_rope(self, qkv: torch.Tensor):
        s, B = self.shape, self.batch
        q = torch.empty((B * self.kv_local, s.g, 128), dtype=torch.float16, device=self.dev)
        k = torch.empty((B * self.kv_local, 128), dtype=torch.float16, device=self.dev)
        v = torch.empty_like(k)
        check(lib().dq_model_qkv_rope(qkv.data_ptr(), B, self.heads_local, self.kv_local, self.pos.data_ptr(), 10000.0,
                                      q.data_ptr(), k.data_ptr(), v.data_ptr(), stream_ptr()), "qkv_rope")
        return q, k, v

    def _silu_mul(self, gu: torch.Tensor) -> torch.Tensor:
        out = torch.empty((gu.shape[0], gu.shape[1] // 2), dtype=gu.dtype, device=self.dev)
        check(lib().dq_model_silu_mul(gu.data_ptr(), gu.shape[0], gu.shape[1] // 2, out.data_ptr(), stream_ptr()),
              "silu_mul")
        return out

    def _layer(self, i: int, x: torch.Tensor, y: torch.Tensor | None):
        """Layer i on the residual x (updated in place) whose previous layer's MLP output y has not
        been added yet (it is fused into this layer's first norm).  A generator: it yields each
        sliced activation and receives it gathered over the TP group; returns this layer's MLP
        output (whole hidden width)."""
        L, B = self.layers[i], self.batch
        h = self._norm(x, y, L["ln1"])
        q, k, v = self._qkv_rope(h @ L["qkv"])
        # units = (sequence, local kv head); query heads kv * g .. kv * g + g - 1 share a kv head
        att = self.cache.attend(i, q, append=(k, v), out_dtype=torch.bfloat16)  # bf16 straight from the combine
        att = yield att.view(B, self.heads_local * 128)  # the per-layer output gather: all heads
        o = yield att @ L["o"]                            # this rank's hidden columns
        h = self._norm(x, o, L["ln2"])
        act = yield self._silu_mul(h @ L["gate_up"])      # this rank's ffn columns
        y = yield act @ L["down"]
        return y

    def _step(self, tokens: torch.Tensor):
        """One decode step as a generator over the TP gathers (see _layer); returns next tokens."""
        x = self.embed[tokens]
        y = None
        for i in range(self.shape.layers):
            y = yield from self._layer(i, x, y)
        logits = self._norm(x, y, self.norm) @ self.lm_head  # this rank's vocabulary slice
        self.pos.add_(1)
        if self.tp.world == 1:
            return logits.argmax(-1)
        v0 = self.sl["vocab"][0]
        top = logits.max(-1, keepdim=True)
        vals = yield top.values.float()                           # (B, world)
        idx = yield (top.indices + v0).to(torch.float32)          # vocab < 2^24: exact in fp32
        best = vals.argmax(-1, keepdim=True)                      # first rank with the maximum
        return idx.gather(1, best).squeeze(1).to(torch.int64)

    def step(self, tokens: torch.Tensor) -> torch.Tensor:
        """One decode step: tokens (batch,) int64 -> next tokens (batch,) (greedy)."""
        return drive(self._step(tokens), self.tp.gather)

    def capture(self, tokens: torch.Tensor | None = None) -> torch.Tensor:
        """Run one eager decode step on `tokens` (zeros by default) and record the step as a CUDA
        graph (replay() runs it; the cache's host-side token counters advance per replay).
        Returns the eager step's next tokens.  Refused when a tail chunk would seal inside."""
        self.cache._flush_seals()
        if any(lay.tail_len + 2 >= self.cache.chunk_len for lay in self.cache._layers):
            raise ShapeMismatch("a tail chunk seals within the next steps: decode them eagerly first")
        self._tok = torch.zeros(self.batch, dtype=torch.int64, device=self.dev)
        if tokens is not None:
            self._tok.copy_(tokens)
        first = self.step(self._tok).clone()  # eager step: builds every layer's segment table
        torch.cuda.synchronize()
        tails = [lay.tail_len for lay in self.cache._layers]
        self._gens = [lay.gen for lay in self.cache._layers]
        self._keep = [list(lay.keep) for lay in self.cache._layers]  # tables the graph points at
        pos = self.pos.clone()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._next = self.step(self._tok)
        for lay, t in zip(self.cache._layers, tails):  # the capture ran no device work
            lay.tail_len = t
        self.pos.copy_(pos)
        return first

    def replay(self, tokens: torch.Tensor) -> torch.Tensor:
        if any(lay.tail_len + 1 >= self.cache.chunk_len for lay in self.cache._layers):
            raise ShapeMismatch("a tail chunk seals on this token: decode it eagerly, then capture() again")
        if [lay.gen for lay in self.cache._layers] != self._gens:
            raise ShapeMismatch("a layer was re-planned (sealed chunk) since the capture: capture() again")
        self._tok.copy_(tokens)
        self.graph.replay()
        for layer in range(self.shape.layers):
            self.cache._after_append(layer)
        return self._next


def drive(gen, gather):
    """Run a step generator to completion, answering each yielded slice with gather(slice)."""
    try:
        t = next(gen)
        while True:
            t = gen.send(gather(t))
    except StopIteration as stop:
        return stop.value


class Lockstep:
    """N tensor-parallel shard models driven in one process: every gather is the concatenation
    of the shards' slices in rank order, so the sharded step runs without a process group
    (the device parity test of TP against the unsharded model; no rank waits on another)."""

    def __init__(self, shards: list[DecoQuantLM]):
        self.shards = shards

    def step(self, tokens: torch.Tensor) -> list[torch.Tensor]:
        gens = [m._step(tokens) for m in self.shards]
        outs = [None] * len(gens)
        msgs = [next(g) for g in gens]
        while True:
            full = torch.cat(msgs, -1)
            nxt = []
            for r, g in enumerate(gens):
                try:
                    nxt.append(g.send(full))
                except StopIteration as stop:
                    outs[r] = stop.value
            if all(o is not None for o in outs):
                return outs
            msgs = nxt

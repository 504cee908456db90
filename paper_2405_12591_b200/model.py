"""LLaMA-shaped decoder with a DecoQuant KV cache: the end-to-end decode harness.

Random-init weights (std 0.02, bf16) of the named shapes; one decode step per call:

    RMSNorm -> QKV projection -> RoPE -> fused DecoQuant attention (+ KV append) -> O projection
    -> residual -> RMSNorm -> SwiGLU MLP -> residual        (x layers), RMSNorm -> LM head -> argmax

The attention of every layer is ``DecodeKvCache.attend(layer, q, append=(k, v))``: the new
token's K/V join the fp16 tail and the compressed segments are read by the fused kernels.
Dense projections are cuBLAS GEMMs through torch (library code, as the task allows); the
elementwise work between them is three fused kernels of the C ABI (csrc/model.cu: residual
add + RMSNorm, QKV split + RoPE + fp16 cast, SwiGLU), so a layer is ten launches; the step
is capturable in one CUDA graph (``capture()`` / ``replay()``).  Tensor parallelism across
GPUs shards the KV heads (``sharding.py``); this harness runs the single-GPU shard.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from ._lib import check, lib, ptr, stream_ptr
from .attention import DecodeKvCache
from .errors import ShapeMismatch


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
                 device="cuda"):
        if shape.head_dim != 128 or shape.heads % shape.kv_heads:
            raise ShapeMismatch("head_dim must be 128 and heads a multiple of kv_heads")
        self.shape, self.batch = shape, batch
        self.dev = torch.device(device)
        gen = torch.Generator(device=self.dev).manual_seed(seed)
        s, hd = shape, shape.head_dim

        def w(*dims):
            return (torch.randn(dims, generator=gen, device=self.dev, dtype=torch.float32) * 0.02).to(torch.bfloat16)

        self.embed = w(s.vocab, s.hidden)
        self.lm_head = w(s.hidden, s.vocab)
        self.norm = torch.ones(s.hidden, device=self.dev, dtype=torch.bfloat16)
        self.layers = []
        for _ in range(s.layers):
            self.layers.append({
                "ln1": torch.ones(s.hidden, device=self.dev, dtype=torch.bfloat16),
                "ln2": torch.ones(s.hidden, device=self.dev, dtype=torch.bfloat16),
                "qkv": w(s.hidden, (s.heads + 2 * s.kv_heads) * hd),
                "o": w(s.heads * hd, s.hidden),
                "gate_up": w(s.hidden, 2 * s.ffn),
                "down": w(s.ffn, s.hidden),
            })
        self.cache = DecodeKvCache(layers=s.layers, units=batch * s.kv_heads, g=s.g, bits=bits,
                                   chunk_len=chunk_len)
        self.pos = torch.zeros((), dtype=torch.int64, device=self.dev)  # decode position (device)
        self.graph = None
        self._tok = self._next = None

    def prefill_random(self, tokens: int, seed: int = 1):
        """Fill every layer's cache with `tokens` positions of synthetic K/V (N(0,1) fp16),
        compressed by the K3 write path (one segment per (sequence, kv head))."""
        gen = torch.Generator(device=self.dev).manual_seed(seed)
        units = self.batch * self.shape.kv_heads
        for layer in range(self.shape.layers):
            k = torch.randn((units, tokens, 128), generator=gen, device=self.dev).to(torch.float16)
            v = torch.randn((units, tokens, 128), generator=gen, device=self.dev).to(torch.float16)
            self.cache.prefill(layer, k, v)
        self.pos.fill_(tokens)

    # ---- fused harness kernels (csrc/model.cu); _rms / _rope above are their torch statements
    def _norm(self, x: torch.Tensor, y: torch.Tensor | None, w: torch.Tensor) -> torch.Tensor:
        """x += y in place (y None: x as is); returns RMSNorm(x) * w."""
        h = torch.empty_like(x)
        check(lib().dq_model_add_rmsnorm(x.data_ptr(), ptr(y), w.data_ptr(), x.data_ptr(), h.data_ptr(),
                                         x.shape[0], x.shape[1], 1e-5, stream_ptr()), "add_rmsnorm")
        return h

    def _qkv_rope(self, qkv: torch.Tensor):
        s, B = self.shape, self.batch
        q = torch.empty((B * s.kv_heads, s.g, 128), dtype=torch.float16, device=self.dev)
        k = torch.empty((B * s.kv_heads, 128), dtype=torch.float16, device=self.dev)
        v = torch.empty_like(k)
        check(lib().dq_model_qkv_rope(qkv.data_ptr(), B, s.heads, s.kv_heads, self.pos.data_ptr(), 10000.0,
                                      q.data_ptr(), k.data_ptr(), v.data_ptr(), stream_ptr()), "qkv_rope")
        return q, k, v

    def _silu_mul(self, gu: torch.Tensor) -> torch.Tensor:
        out = torch.empty((gu.shape[0], gu.shape[1] // 2), dtype=gu.dtype, device=self.dev)
        check(lib().dq_model_silu_mul(gu.data_ptr(), gu.shape[0], gu.shape[1] // 2, out.data_ptr(), stream_ptr()),
              "silu_mul")
        return out

    def _layer(self, i: int, x: torch.Tensor, y: torch.Tensor | None) -> torch.Tensor:
        """Layer i on the residual x (updated in place) whose previous layer's MLP output y has not
        been added yet (it is fused into this layer's first norm); returns this layer's MLP output."""
        s, L, B = self.shape, self.layers[i], self.batch
        h = self._norm(x, y, L["ln1"])
        q, k, v = self._qkv_rope(h @ L["qkv"])
        # units = (sequence, kv head); query heads kv * g .. kv * g + g - 1 share a kv head
        att = self.cache.attend(i, q, append=(k, v), out_dtype=torch.bfloat16)  # bf16 straight from the combine
        h = self._norm(x, att.view(B, s.heads * 128) @ L["o"], L["ln2"])
        return self._silu_mul(h @ L["gate_up"]) @ L["down"]

    def step(self, tokens: torch.Tensor) -> torch.Tensor:
        """One decode step: tokens (batch,) int64 -> next tokens (batch,) (greedy)."""
        x = self.embed[tokens]
        y = None
        for i in range(self.shape.layers):
            y = self._layer(i, x, y)
        logits = self._norm(x, y, self.norm) @ self.lm_head
        self.pos.add_(1)
        return logits.argmax(-1)

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

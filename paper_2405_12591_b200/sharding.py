"""KV-head sharding across the GPUs of one node (north_star item 3).

Every (sequence, kv head, layer) block is independent (compress.py:85-94; each
segment is decomposed on its own, SPEC "Per-segment decomposition"), so rank k
of N owns kv heads [k*H/N, (k+1)*H/N) for all sequences and layers, with the
matching g query heads each.  The decode attention path exchanges nothing; the
only collective is the optional per-layer gather of attention outputs for a
tensor-parallel end-to-end stack (``gather_heads``).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def kv_head_range(kv_heads: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) kv heads owned by ``rank``; requires kv_heads % world == 0."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if kv_heads % world:
        raise ValueError(f"{kv_heads} kv heads do not shard evenly over {world} ranks")
    per = kv_heads // world
    return rank * per, (rank + 1) * per


def local_units(batch: int, kv_heads: int, rank: int, world: int) -> list[tuple[int, int]]:
    """(sequence, kv head) pairs owned by ``rank``, in the unit order DecodeKvCache uses."""
    lo, hi = kv_head_range(kv_heads, rank, world)
    return [(b, h) for b in range(batch) for h in range(lo, hi)]


def shard_heads(x: torch.Tensor, rank: int, world: int, dim: int = 1) -> torch.Tensor:
    """Slice the kv-head axis ``dim`` of a (batch, heads, ...) tensor to this rank's range."""
    lo, hi = kv_head_range(x.shape[dim], rank, world)
    return x.narrow(dim, lo, hi - lo)


def gather_heads(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather (batch, local_heads, ...) shards into (batch, heads, ...) in rank order.

    NCCL over NVLink on GPUs (``all_gather_into_tensor``), gloo in CPU tests.
    """
    world = dist.get_world_size(group)
    if world == 1:
        return local
    moved = local.movedim(1, 0).contiguous()  # (local_heads, batch, ...)
    out = torch.empty((world * moved.shape[0],) + tuple(moved.shape[1:]), dtype=moved.dtype, device=moved.device)
    if moved.is_cuda:
        dist.all_gather_into_tensor(out, moved, group=group)
    else:
        parts = [torch.empty_like(moved) for _ in range(world)]
        dist.all_gather(parts, moved, group=group)
        out = torch.cat(parts, 0)
    return out.movedim(0, 1).contiguous()


# ---- tensor parallelism for the end-to-end decode harness (model.py) -------
#
# Gather-only TP: every weight matrix is split by OUTPUT columns, so each output element is
# computed whole on one rank (no partial sums, no all-reduce) and the only collective is an
# all-gather of the sliced activations, four per layer:
#   attention heads (B, heads*128), O-projection hidden slice, SwiGLU ffn slice, MLP hidden slice.
# The first is north_star's "per-layer output gather"; the other three keep the dense weights
# sharded (1/N of the bytes per GPU) instead of replicating them.


class TpGroup:
    """This rank's place in a tensor-parallel group and its gather along the last dim.

    ``gather(local)`` concatenates the ranks' (rows, n) slices into (rows, world * n) in rank
    order: NCCL ``all_gather_into_tensor`` over NVLink on GPUs (capturable in a CUDA graph),
    gloo on CPU tensors.  ``group=None`` and world 1 make it the identity (one GPU)."""

    def __init__(self, group=None, world: int | None = None, rank: int | None = None):
        self.group = group
        if world is None:
            world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if world > 1 else 0
        self.world, self.rank = world, rank

    def gather(self, local: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return local
        local = local.contiguous()
        rows = local.shape[0]
        if local.is_cuda:
            buf = torch.empty((self.world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
            dist.all_gather_into_tensor(buf, local, group=self.group)
        else:
            parts = [torch.empty_like(local) for _ in range(self.world)]
            dist.all_gather(parts, local, group=self.group)
            buf = torch.stack(parts, 0)
        return buf.permute(1, 0, 2).reshape(rows, -1)


def tp_slices(shape, rank: int, world: int) -> dict:
    """Column ranges of this rank's weight shards for a ModelShape (all divisibility checked)."""
    for name, n in (("kv_heads", shape.kv_heads), ("hidden", shape.hidden), ("ffn", shape.ffn),
                    ("vocab", shape.vocab)):
        if n % world:
            raise ValueError(f"{name} = {n} does not shard evenly over {world} ranks")
    lo, hi = kv_head_range(shape.kv_heads, rank, world)
    g, hd = shape.heads // shape.kv_heads, shape.head_dim

    def part(n):
        return rank * n // world, (rank + 1) * n // world

    return {"kv": (lo, hi), "q_cols": (lo * g * hd, hi * g * hd), "k_cols": (lo * hd, hi * hd),
            "hidden": part(shape.hidden), "ffn": part(shape.ffn), "vocab": part(shape.vocab)}


def shard_layer_weights(layer: dict, shape, rank: int, world: int) -> dict:
    """This rank's copy of one decoder layer's weights (model.py layout: qkv = [q | k | v]
    columns, gate_up = [gate | up]); norms stay whole."""
    s = tp_slices(shape, rank, world)
    H, KV, F = shape.heads * shape.head_dim, shape.kv_heads * shape.head_dim, shape.ffn
    (q0, q1), (k0, k1), (h0, h1), (f0, f1) = s["q_cols"], s["k_cols"], s["hidden"], s["ffn"]
    qkv = layer["qkv"]
    return {
        "ln1": layer["ln1"], "ln2": layer["ln2"],
        "qkv": torch.cat([qkv[:, q0:q1], qkv[:, H + k0:H + k1], qkv[:, H + KV + k0:H + KV + k1]], 1).contiguous(),
        "o": layer["o"][:, h0:h1].contiguous(),
        "gate_up": torch.cat([layer["gate_up"][:, f0:f1], layer["gate_up"][:, F + f0:F + f1]], 1).contiguous(),
        "down": layer["down"][:, h0:h1].contiguous(),
    }

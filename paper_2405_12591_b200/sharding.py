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

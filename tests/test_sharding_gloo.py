"""KV-head sharding over 2 ranks (gloo, CPU): the multi-GPU path of SURVEY.md 8(e).

Each rank owns kv heads [k*H/N, (k+1)*H/N) of every sequence (sharding.kv_head_range),
runs decode attention on its units only (here the CPU oracle stands in for the device
kernel, which has no GPU in this container), and the per-layer output gather
(sharding.gather_heads, NCCL all_gather_into_tensor on GPUs) restores the full
(batch, heads, g, 128) output.  The gathered result must equal the unsharded one
bit for bit: the attention path exchanges nothing, so sharding cannot change numerics.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dquant_oracle as O

BATCH, HEADS, G, T, BITS = 2, 4, 2, 64, 4


def _inputs():
    rng = np.random.default_rng(3)
    k = rng.standard_normal((BATCH, HEADS, T, 128)).astype(np.float16).astype(np.float32)
    v = rng.standard_normal((BATCH, HEADS, T, 128)).astype(np.float16).astype(np.float32)
    q = rng.standard_normal((BATCH, HEADS, G, 128)).astype(np.float16).astype(np.float32)
    return q, k, v


def _attend(q, k, v):
    """(b, h, g, D) outputs of the units (b, h) given."""
    b, h = q.shape[:2]
    out = O.attention_units(q.reshape(b * h, G, 128), k.reshape(b * h, T, 128), v.reshape(b * h, T, 128), BITS)
    return out.reshape(b, h, G, 128)


def _worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_12591_b200.sharding import gather_heads, kv_head_range, local_units, shard_heads

        q, k, v = _inputs()
        lo, hi = kv_head_range(HEADS, rank, world)
        assert local_units(BATCH, HEADS, rank, world) == [(b, h) for b in range(BATCH) for h in range(lo, hi)]
        ql = shard_heads(torch.from_numpy(q), rank, world).numpy()
        kl = shard_heads(torch.from_numpy(k), rank, world).numpy()
        vl = shard_heads(torch.from_numpy(v), rank, world).numpy()
        local = torch.from_numpy(_attend(ql, kl, vl))
        full = gather_heads(local)
        if rank == 0:
            result.put(full.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_kv_head_ranges():
    from paper_2405_12591_b200.sharding import kv_head_range

    assert [kv_head_range(32, r, 8) for r in range(8)] == [(4 * r, 4 * r + 4) for r in range(8)]
    assert kv_head_range(8, 7, 8) == (7, 8)
    with pytest.raises(ValueError):
        kv_head_range(6, 0, 4)
    with pytest.raises(ValueError):
        kv_head_range(8, 2, 2)


def test_sharded_decode_matches_unsharded_world2():
    ctx = mp.get_context("spawn")
    result = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, result)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = result.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    q, k, v = _inputs()
    ref = _attend(q, k, v)
    assert gathered.shape == ref.shape
    assert np.array_equal(gathered, ref)

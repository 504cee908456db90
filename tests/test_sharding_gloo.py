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


# ---- tensor-parallel decoder layer (model.py's gather-only TP) on 2 gloo ranks -------------

class _Shape:  # the ModelShape fields the sharding helpers read
    layers, hidden, heads, kv_heads, ffn, vocab, head_dim = 1, 64, 8, 4, 96, 40, 128

    @property
    def g(self):
        return self.heads // self.kv_heads


def _tp_weights():
    s, gen = _Shape(), torch.Generator().manual_seed(11)
    H, KV = s.heads * 128, s.kv_heads * 128
    return {"ln1": torch.ones(s.hidden), "ln2": torch.ones(s.hidden),
            "qkv": torch.randn(s.hidden, H + 2 * KV, generator=gen), "o": torch.randn(H, s.hidden, generator=gen),
            "gate_up": torch.randn(s.hidden, 2 * s.ffn, generator=gen),
            "down": torch.randn(s.ffn, s.hidden, generator=gen)}, torch.randn(3, s.hidden, generator=gen)


def _tp_layer(L, x, heads, kv, gather):
    """model._layer's dataflow in fp32 torch with a stand-in attention (q * v of the head's kv
    head, per head: it shards exactly like the real one) and the same four gathers."""
    s = _Shape()
    B, g = x.shape[0], s.g
    qkv = x @ L["qkv"]
    q = qkv[:, : heads * 128].view(B, kv, g, 128)
    v = qkv[:, heads * 128 + kv * 128:].view(B, kv, 1, 128)
    att = gather((q * v).reshape(B, heads * 128))
    x = x + gather(att @ L["o"])
    gu = x @ L["gate_up"]
    F = gu.shape[1] // 2
    act = gather(torch.nn.functional.silu(gu[:, :F]) * gu[:, F:])
    return x + gather(act @ L["down"])


def _tp_worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_12591_b200.sharding import TpGroup, shard_layer_weights

        tp = TpGroup()
        assert (tp.rank, tp.world) == (rank, world)
        # gather order: rank r's (rows, n) slice lands in columns [r n, (r + 1) n)
        got = tp.gather(torch.full((2, 3), float(rank)))
        assert torch.equal(got, torch.tensor([[0.0] * 3 + [1.0] * 3] * 2))
        L, x = _tp_weights()
        s = _Shape()
        Ls = shard_layer_weights(L, s, rank, world)
        out = _tp_layer(Ls, x, s.heads // world, s.kv_heads // world, tp.gather)
        if rank == 0:
            result.put(out.numpy())
    finally:
        dist.destroy_process_group()


def test_tensor_parallel_layer_matches_unsharded_world2():
    """The weight shards (output-column slices) and the rank-ordered gathers compose to the
    unsharded layer: every output element is computed whole on one rank."""
    ctx = mp.get_context("spawn")
    result = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_worker, args=(r, 2, port, result)) for r in range(2)]
    for p in procs:
        p.start()
    got = result.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = _Shape()
    L, x = _tp_weights()
    ref = _tp_layer(L, x, s.heads, s.kv_heads, lambda t: t).numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-3)


def test_tp_slices_reject_uneven():
    from paper_2405_12591_b200.sharding import tp_slices

    s = _Shape()
    assert tp_slices(s, 1, 2)["q_cols"] == (512, 1024) and tp_slices(s, 1, 2)["ffn"] == (48, 96)
    with pytest.raises(ValueError):
        tp_slices(s, 0, 3)

"""KV-head sharding on the device: each rank's DecodeKvCache holds only its kv
heads; the gathered outputs equal the unsharded cache's bit for bit.

The ranks run one after another on cuda:0 (their kernels never wait on each other: the
attention path has no collective), each with the shard that sharding.shard_heads gives it.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,g", [(2, 1), (4, 1), (8, 8)])
def test_sharded_caches_match_unsharded(world, g):
    from paper_2405_12591_b200.attention import DecodeKvCache
    from paper_2405_12591_b200.sharding import local_units, shard_heads

    batch, heads, T, steps = 2, 8, 1024, 3
    rng = np.random.default_rng(world + g)
    k = torch.from_numpy(rng.standard_normal((batch, heads, T + steps, 128)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((batch, heads, T + steps, 128)).astype(np.float16)).cuda()
    q = torch.from_numpy(rng.standard_normal((batch, heads, g, 128)).astype(np.float16)).cuda()

    def run(kk, vv, qq):
        b, h = kk.shape[:2]
        c = DecodeKvCache(layers=1, units=b * h, g=g, bits=4, chunk_len=256)
        c.prefill(0, kk[:, :, :T].reshape(b * h, T, 128), vv[:, :, :T].reshape(b * h, T, 128))
        for t in range(T, T + steps):
            out = c.attend(0, qq.reshape(b * h, g, 128),
                           append=(kk[:, :, t].reshape(b * h, 128), vv[:, :, t].reshape(b * h, 128)))
        return out.reshape(b, h, g, 128)

    full = run(k, v, q)
    parts = []
    for rank in range(world):
        assert len(local_units(batch, heads, rank, world)) == batch * heads // world
        parts.append(run(shard_heads(k, rank, world).contiguous(), shard_heads(v, rank, world).contiguous(),
                         shard_heads(q, rank, world).contiguous()))
    gathered = torch.cat(parts, 1)  # what gather_heads' all_gather_into_tensor assembles
    assert torch.equal(gathered, full)

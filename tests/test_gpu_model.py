"""The LLaMA-shaped decode harness: one step's attention equals dense attention over the
decompressed cache (oracle) plus the appended token; the step is deterministic."""

import numpy as np
import pytest
import torch

from oracle import dquant_oracle as O

pytestmark = pytest.mark.gpu


def test_tiny_model_step_attention_matches_oracle():
    from paper_2405_12591_b200 import model as M

    shape = M.ModelShape(layers=2, hidden=512, heads=4, kv_heads=2, ffn=1024, vocab=1000)
    lm = M.DecoQuantLM(shape, batch=3, bits=4, chunk_len=64)
    lm.prefill_random(520)
    captured = {}
    real_attend = lm.cache.attend

    def spy(layer, q, out=None, append=None, out_dtype=torch.float16):
        if layer == 0:
            captured["q"] = q.float().cpu().numpy()
            captured["k"], captured["v"] = (t.float().cpu().numpy() for t in append)
            # the same attention in fp16 (no append: the prefix the model's call sees)
            captured["out"] = real_attend(layer, q).float().cpu().numpy()
        o = real_attend(layer, q, out, append, out_dtype=out_dtype)
        if layer == 0:
            captured["out_model"] = o.float().cpu().numpy()
            captured["out_dtype"] = o.dtype
        return o

    lm.cache.attend = spy
    tok = lm.step(torch.tensor([1, 2, 3], device="cuda"))
    assert tok.shape == (3,) and int(tok.max()) < shape.vocab
    # layer 0: the kernel's output vs the oracle over the same compressed prefix (the new
    # token joins the tail after this step's attention, kvcache.py semantics)
    gen = torch.Generator(device="cuda").manual_seed(1)
    units = 3 * shape.kv_heads
    k0 = torch.randn((units, 520, 128), generator=gen, device="cuda").to(torch.float16).float().cpu().numpy()
    v0 = torch.randn((units, 520, 128), generator=gen, device="cuda").to(torch.float16).float().cpu().numpy()
    ref = O.attention_units(captured["q"], k0, v0, 4)
    rel = np.linalg.norm(captured["out"] - ref) / np.linalg.norm(ref)
    assert rel < 1e-3, rel
    # the model reads the attention as bf16 straight from the combine kernel: one rounding of
    # the same merged value, so within one bf16 ulp of the fp16 output
    assert captured["out_dtype"] == torch.bfloat16
    x, y = captured["out"], captured["out_model"]
    assert np.all(np.abs(x - y) <= 2.0 ** -7 * np.maximum(np.abs(x), 2.0 ** -20))
    assert lm.cache.tokens(0) == 521 and lm.cache.tokens(1) == 521


def test_model_step_deterministic():
    from paper_2405_12591_b200 import model as M

    shape = M.ModelShape(layers=2, hidden=256, heads=2, kv_heads=2, ffn=512, vocab=500)
    outs = []
    for _ in range(2):
        lm = M.DecoQuantLM(shape, batch=2, seed=5)
        lm.prefill_random(600, seed=6)
        tok = torch.tensor([7, 9], device="cuda")
        seq = []
        for _ in range(4):
            tok = lm.step(tok)
            seq.append(tok.cpu().tolist())
        outs.append(seq)
    assert outs[0] == outs[1]


def test_captured_step_matches_eager():
    """capture() + replay() gives the same tokens as eager steps (capture itself runs one
    eager step on zero tokens; the eager twin does the same)."""
    from paper_2405_12591_b200 import model as M

    shape = M.ModelShape(layers=2, hidden=256, heads=2, kv_heads=1, ffn=512, vocab=500)
    twins = []
    for _ in range(2):
        lm = M.DecoQuantLM(shape, batch=2, seed=5, chunk_len=64)
        lm.prefill_random(600, seed=6)
        twins.append(lm)
    eager, graphed = twins
    zero = torch.zeros(2, dtype=torch.int64, device="cuda")
    first = eager.step(zero)
    assert torch.equal(first, graphed.capture(zero))
    tok_e, tok_g = first.clone(), first.clone()
    for _ in range(4):
        tok_e = eager.step(tok_e)
        tok_g = graphed.replay(tok_g).clone()
        assert torch.equal(tok_e, tok_g)
    assert eager.cache.tokens(0) == graphed.cache.tokens(0) == 605
    assert torch.equal(eager.cache.tail_len, graphed.cache.tail_len)


def _bf16_ulps(a: torch.Tensor, b: torch.Tensor) -> int:
    """Largest distance in bf16 units in the last place (ordered-integer view)."""
    ia, ib = (t.contiguous().view(torch.int16).to(torch.int32) for t in (a, b))
    ia = torch.where(ia < 0, -32768 - ia, ia)
    ib = torch.where(ib < 0, -32768 - ib, ib)
    return int((ia - ib).abs().max())


@pytest.mark.parametrize("hidden,with_y", [(4096, True), (5120, False), (8192, True), (256, True)])
def test_add_rmsnorm_kernel_matches_torch(hidden, with_y):
    """dq_model_add_rmsnorm vs model._rms(x + y): the residual sum is bit-exact, the normalised
    row within one bf16 ulp (only the fp32 sum-of-squares order differs)."""
    from paper_2405_12591_b200 import model as M

    g = torch.Generator(device="cuda").manual_seed(hidden)
    x = torch.randn((16, hidden), generator=g, device="cuda").to(torch.bfloat16)
    y = torch.randn((16, hidden), generator=g, device="cuda").to(torch.bfloat16) if with_y else None
    w = (1 + 0.1 * torch.randn(hidden, generator=g, device="cuda")).to(torch.bfloat16)
    ref_x = x + y if with_y else x.clone()
    ref_h = M._rms(ref_x, w)
    lm = M.DecoQuantLM.__new__(M.DecoQuantLM)
    h = M.DecoQuantLM._norm(lm, x, y, w)
    assert torch.equal(x, ref_x)
    assert _bf16_ulps(h, ref_h) <= 1


@pytest.mark.parametrize("heads,kv_heads,pos", [(32, 32, 4096), (64, 8, 16384), (4, 2, 0)])
def test_qkv_rope_kernel_matches_torch(heads, kv_heads, pos):
    """dq_model_qkv_rope vs model._rope on the split QKV row: v bit-exact, q/k within one bf16
    ulp (cos/sin/pow of the device libm vs torch's kernels)."""
    from paper_2405_12591_b200 import model as M

    B = 5
    shape = M.ModelShape(layers=1, hidden=heads * 128, heads=heads, kv_heads=kv_heads, ffn=256)
    g = torch.Generator(device="cuda").manual_seed(heads)
    qkv = torch.randn((B, (heads + 2 * kv_heads) * 128), generator=g, device="cuda").to(torch.bfloat16)
    p = torch.tensor(pos, dtype=torch.int64, device="cuda")
    lm = M.DecoQuantLM.__new__(M.DecoQuantLM)
    lm.shape, lm.batch, lm.dev, lm.pos = shape, B, torch.device("cuda"), p
    lm.kv_local, lm.heads_local = kv_heads, heads
    q, k, v = lm._qkv_rope(qkv)
    rq, rk, rv = qkv.split([heads * 128, kv_heads * 128, kv_heads * 128], dim=-1)
    rq = M._rope(rq.reshape(B, heads, 128), p).reshape(B * kv_heads, heads // kv_heads, 128)
    rk = M._rope(rk.reshape(B, kv_heads, 128), p).reshape(B * kv_heads, 128)
    assert torch.equal(v, rv.reshape(B * kv_heads, 128).to(torch.float16))
    assert _bf16_ulps(q.to(torch.bfloat16), rq) <= 1
    assert _bf16_ulps(k.to(torch.bfloat16), rk) <= 1
    assert q.dtype == k.dtype == torch.float16


def test_silu_mul_kernel_matches_torch():
    from paper_2405_12591_b200 import model as M

    g = torch.Generator(device="cuda").manual_seed(3)
    gu = (4 * torch.randn((16, 2 * 11008), generator=g, device="cuda")).to(torch.bfloat16)
    lm = M.DecoQuantLM.__new__(M.DecoQuantLM)
    lm.dev = torch.device("cuda")
    out = lm._silu_mul(gu)
    gate, up = gu.chunk(2, dim=-1)
    assert _bf16_ulps(out, torch.nn.functional.silu(gate) * up) <= 1


def test_harness_kernels_reject_bad_shapes():
    from paper_2405_12591_b200._lib import lib
    from paper_2405_12591_b200.errors import ShapeMismatch
    from paper_2405_12591_b200._lib import check

    x = torch.zeros((2, 12), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ShapeMismatch):
        check(lib().dq_model_add_rmsnorm(x.data_ptr(), None, x.data_ptr(), x.data_ptr(), x.data_ptr(), 2, 12,
                                         1e-5, None))
    with pytest.raises(ShapeMismatch):
        check(lib().dq_model_qkv_rope(x.data_ptr(), 1, 3, 2, x.data_ptr(), 1e4, x.data_ptr(), x.data_ptr(),
                                      x.data_ptr(), None))


@pytest.mark.parametrize("world", [2, 4])
def test_tensor_parallel_step_matches_unsharded(world):
    """The gather-only TP step (N shard models driven in lock-step: every gather concatenates
    their slices in rank order) against the unsharded model on the same weights and K/V: the
    attention outputs per head within fp16 tolerance, the next tokens equal, and the shards'
    caches holding their kv heads only."""
    from paper_2405_12591_b200 import model as M
    from paper_2405_12591_b200.sharding import TpGroup

    shape = M.ModelShape(layers=2, hidden=512, heads=8, kv_heads=4, ffn=1024, vocab=1000)
    full = M.DecoQuantLM(shape, batch=3, seed=5, chunk_len=64)
    shards = [M.DecoQuantLM.shard_of(full, TpGroup(world=world, rank=r), chunk_len=64) for r in range(world)]
    for m in [full, *shards]:
        m.prefill_random(300, seed=6)
    assert all(m.cache.units == 3 * shape.kv_heads // world for m in shards)
    seen = {}

    def spy(model, key):
        real = model.cache.attend

        def f(layer, q, out=None, append=None, out_dtype=torch.float16):
            o = real(layer, q, out, append, out_dtype=out_dtype)
            seen.setdefault(key, []).append(o.float().view(3, -1, 128).clone())
            return o
        model.cache.attend = f

    spy(full, "full")
    for r, m in enumerate(shards):
        spy(m, r)
    lock = M.Lockstep(shards)
    tok = torch.tensor([1, 2, 3], device="cuda")
    for _ in range(3):
        ref = full.step(tok)
        outs = lock.step(tok)
        assert all(torch.equal(o, outs[0]) for o in outs)
        assert torch.equal(outs[0], ref)
        tok = ref
    for call, ref in enumerate(seen["full"]):
        got = torch.cat([seen[r][call] for r in range(world)], 1)
        rel = float((got - ref).norm() / ref.norm())
        assert rel < 1e-2, (call, rel)
    assert full.cache.tokens(0) == shards[0].cache.tokens(0) == 303

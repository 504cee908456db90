"""K5 fused decode attention and the generic fused reads against the CPU oracle.

Tolerance (north_star): relative Frobenius error <= 1e-3 of the attention output
against the oracle's fp64 composition (scores kvcache.py:188-217 -> softmax ->
per-segment x@W compress.py:159-192 + tail).  Inputs are fp16-rounded so both
sides see identical K/V/q values.
"""

import numpy as np
import pytest
import torch

from oracle import dquant_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-3


@pytest.fixture(scope="module")
def dq():
    import paper_2405_12591_b200 as dq

    return dq


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30))


@pytest.mark.parametrize("name", ["c1h0", "out512", "b2_256", "b8_256", "odd1009", "r1023", "tiny8", "s37x41",
                                  "s64x48", "d64_512"])
def test_generic_fused_reads_golden(golden, dq, name):
    """fused_matmul / fused_matmul_t on the reference's own encoding vs its outputs."""
    g, meta = golden
    info = meta["blocks"][name]
    bits = info["bits"]
    core1 = g[f"{name}_core1"]
    qt = dq.quantize_rtn(core1, bits)
    plan = dq.plan_shapes(*info["shape"], 2)
    q = dq.QuantizedMpo(plan=plan, bits=bits, local_tensors=(g[f"{name}_core0"], qt))
    assert qt.payload == g[f"{name}_payload"].tobytes()
    assert rel(g[f"{name}_mmt"], dq.fused_matmul_t(g[f"{name}_xt"], q)) < 1e-5
    assert rel(g[f"{name}_mm"], dq.fused_matmul(g[f"{name}_x"], q)) < 1e-5
    # the working set is what the kernels report (reads.cu meter_report), not a formula: at most
    # one tile (test_compress.py:112-121), and every code of the core dequantized once per row of x
    meter = dq.WorkingSetMeter()
    dq.fused_matmul(g[f"{name}_x"], q, meter)
    assert 0 < meter.peak_elements <= 64 * 64
    assert meter.total_unpacked == g[f"{name}_x"].shape[0] * qt.count
    meter_t = dq.WorkingSetMeter()
    dq.fused_matmul_t(g[f"{name}_xt"], q, meter_t)
    assert 0 < meter_t.peak_elements <= 64 * 64
    assert meter_t.total_unpacked == g[f"{name}_xt"].shape[0] * qt.count


def _oracle_attend(k, v, q, bits, segs_T, tail):
    """k, v: (T_total, 128) fp32; segments of lengths segs_T then `tail` dense rows."""
    lay = O.LayerOracle(128, bits, 1 << 30)
    off = 0
    for i, T in enumerate(segs_T):
        blk_k, blk_v = k[off:off + T], v[off:off + T]
        if i == 0:
            lay.prefill(blk_k, blk_v)
        else:
            lay.k_segs.append(O.encode(blk_k, bits))
            lay.v_segs.append(O.encode(blk_v, bits))
            lay.rows.append(T)
        off += T
    for t in range(tail):
        lay.tail_k.append(k[off + t])
        lay.tail_v.append(v[off + t])
    return lay.attend(q)


@pytest.mark.parametrize("bits,g,T,units", [
    (4, 1, 4096, 4), (4, 1, 1024, 3), (4, 2, 2048, 2), (2, 2, 1024, 2), (2, 1, 2048, 2), (8, 1, 1024, 2), (8, 2, 640, 2),
    (4, 1, 1009, 2), (4, 1, 1023, 2), (4, 1, 8192, 1), (4, 1, 24, 2), (4, 1, 100, 2), (2, 1, 1009, 1),
    (8, 1, 1023, 1),
])
@pytest.mark.parametrize("ctas", [None, 0, 3])  # persistent grid / one CTA per item / 3 CTAs
@pytest.mark.parametrize("tc", [False, True])    # mma.sync / tcgen05 split kernel (where eligible)
def test_decode_attention_prefill_only(dq, bits, g, T, units, ctas, tc):
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(T + 7 * g + bits)
    k = rng.standard_normal((units, T, 128)).astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, g, 128)).astype(np.float16)
    eligible = bits == 4 and g == 1 and T >= 512 and T % 8 == 0
    if tc and not eligible:
        pytest.skip("tcgen05 path: 4-bit codes, g = 1, full plans only")
    cache = DecodeKvCache(layers=1, units=units, g=g, bits=bits, ctas=ctas, tc=tc)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    assert cache._layers[0].args.path == (1 if tc else 0)
    for u in range(units):
        ref = _oracle_attend(k[u].astype(np.float32), v[u].astype(np.float32), q[u].astype(np.float32), bits,
                             [T], 0)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


@pytest.mark.parametrize("bits,T,units,scale", [(4, 4096, 3, 1.0), (2, 8192, 2, 1.0), (4, 1009, 2, 1.0),
                                                (4, 2240, 2, 20.0), (2, 600, 2, 20.0), (4, 100, 2, 1.0)])
def test_decode_attention_512_row_items(dq, bits, T, units, scale):
    """8-tile work items (chunk_b = 512, mma.sync split kernel, g = 1): ragged last items, outlier keys."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(T + bits + int(scale))
    k = rng.standard_normal((units, T, 128)).astype(np.float32)
    k[:, :, [3, 77]] *= scale
    k = k.astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, 1, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=1, bits=bits, chunk_b=512)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    assert cache._layers[0].args.chunk_b == 512 and cache._layers[0].args.path == 0
    for u in range(units):
        ref = _oracle_attend(k[u].astype(np.float32), v[u].astype(np.float32), q[u].astype(np.float32), bits, [T], 0)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


def test_decode_attention_split_tail(dq):
    """Several rounds of 512-row items (int2): the last TAIL_SPLIT x grid items run as 256-row
    halves (attention.split_tail); ragged T, results against the oracle."""
    from paper_2405_12591_b200.attention import TAIL_SPLIT, DecodeKvCache

    rng = np.random.default_rng(7)
    units, T, ctas = 12, 8000, 10
    k = rng.standard_normal((units, T, 128)).astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, 1, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=1, bits=2, ctas=ctas)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    a = cache._layers[0].args
    assert a.chunk_b == 512 and a.nwork == 2 * units + int(TAIL_SPLIT * ctas)
    for u in range(units):
        ref = _oracle_attend(k[u].astype(np.float32), v[u].astype(np.float32), q[u].astype(np.float32), 2, [T], 0)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


@pytest.mark.parametrize("scale,bits", [(20.0, 4), (50.0, 4), (20.0, 2), (20.0, 8)])
@pytest.mark.parametrize("ctas", [None, 0])  # persistent grid / one CTA per item
@pytest.mark.parametrize("tc", [False, True])
def test_decode_attention_outlier_channels(dq, scale, bits, ctas, tc):
    """Outlier key channels (LLM-like) make the softmax peaky: tolerance must still hold."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(int(scale) + bits)
    units, T = 2, 4096
    k = rng.standard_normal((units, T, 128)).astype(np.float32)
    k[:, :, [3, 77]] *= scale
    k = k.astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, 1, 128)).astype(np.float16)
    if tc and bits != 4:
        pytest.skip("tcgen05 path: 4-bit codes")
    cache = DecodeKvCache(layers=1, units=units, g=1, bits=bits, ctas=ctas, tc=tc)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    for u in range(units):
        ref = _oracle_attend(k[u].astype(np.float32), v[u].astype(np.float32), q[u].astype(np.float32), bits,
                             [T], 0)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


@pytest.mark.parametrize("g,tc", [(2, False), (1, True)])
def test_decode_attention_segments_and_tail(dq, g, tc):
    """prefill 1500 + 2 sealed chunks of 512 + tail 77, int4, outlier columns; g = 1 also on
    the tcgen05 split kernel (prefill 1504 keeps every segment on the full i1 = 8 plan)."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    units, chunk = 3, 512
    rng = np.random.default_rng(5)
    P, steps = (1504 if tc else 1500), 2 * chunk + 77
    total = P + steps
    k = rng.standard_normal((units, total, 128)).astype(np.float32)
    k[:, :, [3, 77]] *= 15.0  # outlier channels
    k = k.astype(np.float16)
    v = rng.standard_normal((units, total, 128)).astype(np.float16)
    q = rng.standard_normal((units, g, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=2, units=units, g=g, bits=4, chunk_len=chunk, tc=tc)
    kd, vd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
    cache.prefill(1, kd[:, :P], vd[:, :P])
    for t in range(P, total):
        cache.append_token(1, kd[:, t], vd[:, t])
    assert cache.tokens(1) == total
    assert len(cache._layers[1].groups) == 3 and cache._layers[1].tail_len == 77
    out = cache.attend(1, torch.from_numpy(q).cuda()).float().cpu().numpy()
    for u in range(units):
        ref = _oracle_attend(k[u].astype(np.float32), v[u].astype(np.float32), q[u].astype(np.float32), 4,
                             [P, chunk, chunk], 77)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))
    # ledger: reference accounting (kvcache.py:130-141)
    fp16, actual = cache.ledger()
    assert fp16 == 2 * total * 128 * 2 * units
    assert actual / fp16 < 0.32


def test_tail_only_and_empty(dq):
    from paper_2405_12591_b200.attention import DecodeKvCache

    cache = DecodeKvCache(layers=1, units=2, g=1, bits=4, chunk_len=64)
    q = torch.randn(2, 1, 128, device="cuda", dtype=torch.float16)
    assert torch.count_nonzero(cache.attend(0, q)) == 0
    rng = np.random.default_rng(2)
    k = rng.standard_normal((2, 10, 128)).astype(np.float16)
    v = rng.standard_normal((2, 10, 128)).astype(np.float16)
    for t in range(10):
        cache.append_token(0, torch.from_numpy(k[:, t]).cuda(), torch.from_numpy(v[:, t]).cuda())
    out = cache.attend(0, q).float().cpu().numpy()
    qn = q.float().cpu().numpy()
    for u in range(2):
        s = qn[u].astype(np.float64) @ k[u].astype(np.float64).T / np.sqrt(128)
        p = np.exp(s - s.max())
        p /= p.sum()
        assert rel(p @ v[u].astype(np.float64), out[u]) < TOL


@pytest.mark.parametrize("g,kernel_g", [(4, None), (8, None), (4, 1), (3, None)])
def test_gqa_head_groups(dq, g, kernel_g):
    """g > 2 query heads per kv head: head groups of kernel_g heads share the segments and the
    tail; segments + fp16 tail + fused append, against the oracle."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    units, P, steps = 3, 1100, 21
    rng = np.random.default_rng(40 + g)
    k = rng.standard_normal((units, P + steps, 128)).astype(np.float32)
    k[:, :, [5, 90]] *= 12.0
    k = k.astype(np.float16)
    v = rng.standard_normal((units, P + steps, 128)).astype(np.float16)
    q = rng.standard_normal((units, g, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=g, bits=4, chunk_len=256, kernel_g=kernel_g)
    kd, vd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
    cache.prefill(0, kd[:, :P], vd[:, :P])
    qd = torch.from_numpy(q).cuda()
    for t in range(P, P + steps - 1):
        cache.attend(0, qd, append=(kd[:, t], vd[:, t]))
    out = cache.attend(0, qd).float().cpu().numpy()
    for u in range(units):
        ref = _oracle_attend(k[u, :P + steps - 1].astype(np.float32), v[u, :P + steps - 1].astype(np.float32),
                             q[u].astype(np.float32), 4, [P], steps - 1)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


@pytest.mark.parametrize("g,T,units,scale", [
    (8, 4096, 3, 1.0), (8, 1024, 2, 1.0), (8, 2240, 2, 1.0), (8, 600, 2, 1.0), (8, 4096, 2, 20.0),
    (8, 8192, 1, 50.0), (16, 2048, 2, 12.0),
])
def test_gqa_tcgen05(dq, g, T, units, scale):
    """The tcgen05 GQA split kernel (path 2: 8 heads x 2 limbs x 8 columns per N = 128 UMMA),
    items of 1..4 tiles (T = 2240: 35 tiles; T = 600: a partial last tile), outlier key
    channels, g = 16 as two head groups of 8."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(T + g + int(scale))
    k = rng.standard_normal((units, T, 128)).astype(np.float32)
    k[:, :, [3, 77]] *= scale
    k = k.astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, g, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=g, bits=4)
    assert cache.kernel_g == 8
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    assert cache._layers[0].args.path == 2
    for u in range(units):
        ref = _oracle_attend(k[u].astype(np.float32), v[u].astype(np.float32), q[u].astype(np.float32), 4, [T], 0)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


def test_gqa_tcgen05_segments_tail_append(dq):
    """Path 2 over prefill + sealed chunks + fp16 tail with the fused append, step by step."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    units, g, chunk, P, steps = 2, 8, 512, 1504, 530
    rng = np.random.default_rng(77)
    k = rng.standard_normal((units, P + steps, 128)).astype(np.float32)
    k[:, :, [5, 90]] *= 10.0
    k = k.astype(np.float16)
    v = rng.standard_normal((units, P + steps, 128)).astype(np.float16)
    q = rng.standard_normal((units, g, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=g, bits=4, chunk_len=chunk)
    kd, vd, qd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(q).cuda()
    cache.prefill(0, kd[:, :P], vd[:, :P])
    for t in range(P, P + steps):
        cache.attend(0, qd, append=(kd[:, t], vd[:, t]))
    assert len(cache._layers[0].groups) == 2 and cache._layers[0].tail_len == steps - chunk
    out = cache.attend(0, qd).float().cpu().numpy()
    assert cache._layers[0].args.path == 2
    for u in range(units):
        ref = _oracle_attend(k[u].astype(np.float32), v[u].astype(np.float32), q[u].astype(np.float32), 4,
                             [P, chunk], steps - chunk)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


def test_fused_append_matches_attend_then_append(dq):
    """attend(append=(k, v)) == attend + append_token, step by step, across a tail seal."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    units, g, chunk, P, steps = 3, 2, 64, 300, 70
    rng = np.random.default_rng(11)
    k = torch.from_numpy(rng.standard_normal((units, P + steps, 128)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((units, P + steps, 128)).astype(np.float16)).cuda()
    q = torch.from_numpy(rng.standard_normal((steps, units, g, 128)).astype(np.float16)).cuda()
    a = DecodeKvCache(layers=1, units=units, g=g, bits=4, chunk_len=chunk)
    b = DecodeKvCache(layers=1, units=units, g=g, bits=4, chunk_len=chunk)
    for c in (a, b):
        c.prefill(0, k[:, :P], v[:, :P])
    for t in range(steps):
        oa = a.attend(0, q[t])
        a.append_token(0, k[:, P + t], v[:, P + t])
        ob = b.attend(0, q[t], append=(k[:, P + t], v[:, P + t]))
        assert torch.equal(oa, ob), t
        assert a.tokens(0) == b.tokens(0) == P + t + 1
    assert len(b._layers[0].groups) == 2 and b._layers[0].tail_len == steps - chunk
    assert torch.equal(a.tail_len, b.tail_len)
    assert torch.equal(a.tail_k[0, :, :steps - chunk], b.tail_k[0, :, :steps - chunk])


@pytest.mark.parametrize("g,P", [(2, 700), (8, 704)])  # mma.sync split kernel / tcgen05 GQA kernel (path 2)
def test_decode_step_graph_matches_eager(dq, g, P):
    """DecodeStepGraph (captured multi-layer step, host I/O) == eager attend(append=...) per layer."""
    from paper_2405_12591_b200.attention import DecodeKvCache
    from paper_2405_12591_b200.decode_step import DecodeStepGraph

    L, U, steps = 3, 4, 5
    rng = np.random.default_rng(21)
    kv = torch.from_numpy(rng.standard_normal((L, 2, U, P, 128)).astype(np.float16)).cuda()
    caches = [DecodeKvCache(layers=L, units=U, g=g, bits=4, chunk_len=64) for _ in range(2)]
    for c in caches:
        for layer in range(L):
            c.prefill(layer, kv[layer, 0], kv[layer, 1])
    q_h = torch.empty((L, U, g, 128), dtype=torch.float16).pin_memory()
    k_h = torch.empty((L, U, 128), dtype=torch.float16).pin_memory()
    v_h = torch.empty((L, U, 128), dtype=torch.float16).pin_memory()
    out_h = torch.empty((L, U, g, 128), dtype=torch.float16).pin_memory()
    eager, graphed = caches

    def fill(t):
        r = np.random.default_rng(100 + t)
        q_h.copy_(torch.from_numpy(r.standard_normal((L, U, g, 128)).astype(np.float16)))
        k_h.copy_(torch.from_numpy(r.standard_normal((L, U, 128)).astype(np.float16)))
        v_h.copy_(torch.from_numpy(r.standard_normal((L, U, 128)).astype(np.float16)))

    def eager_step():
        return torch.stack([eager.attend(layer, q_h[layer].cuda(), append=(k_h[layer].cuda(), v_h[layer].cuda()))
                            for layer in range(L)]).cpu()

    fill(0)
    stepper = DecodeStepGraph(graphed, q_h, k_h, v_h, out_h)  # runs step 0 eagerly, then captures
    assert graphed._layers[0].args.path == (2 if g == 8 else 0)
    ref = eager_step()
    torch.cuda.synchronize()
    assert torch.equal(out_h, ref)
    for t in range(1, steps):
        fill(t)
        stepper.replay()
        torch.cuda.synchronize()
        ref = eager_step()
        assert torch.equal(out_h, ref), t
        assert graphed.tokens(0) == eager.tokens(0) == P + t + 1
    assert torch.equal(graphed.tail_len, eager.tail_len)


def test_export_segment_wire_format(dq):
    """Device layouts -> reference wire order: same bytes as deco_quantize on the same block."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(9)
    k = rng.standard_normal((2, 1009, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=2, g=1, bits=4)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(k).cuda())
    for which in ("k", "v"):
        seg = cache.export_segment(0, 0, 1, which)
        direct = dq.deco_quantize(k[1].astype(np.float32), 4)
        assert seg.local_tensors[1].payload == direct.local_tensors[1].payload
        assert seg.local_tensors[1].scale == direct.local_tensors[1].scale
        assert rel(dq.deco_dequantize(direct), dq.deco_dequantize(seg).cpu().numpy()) < 1e-6


@pytest.mark.parametrize("g,kernel_g", [(1, None), (2, None), (8, 8)])
def test_bf16_output(dq, g, kernel_g):
    """out_dtype=bf16: the combine kernel rounds the merged fp32 output to bf16 once.  Against
    the fp16 output: within one bf16 ulp (the fp16 route rounds twice); against the oracle:
    the bf16 rounding (2^-9 relative) on top of the tolerance."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(11 + g)
    units, T = 3, 1024
    k = rng.standard_normal((units, T, 128)).astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = torch.from_numpy(rng.standard_normal((units, g, 128)).astype(np.float16)).cuda()
    cache = DecodeKvCache(layers=1, units=units, g=g, bits=4, chunk_len=64, kernel_g=kernel_g)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    for t in range(5):  # a dense tail as well
        cache.append_token(0, torch.from_numpy(k[:, t]).cuda(), torch.from_numpy(v[:, t]).cuda())
    o16 = cache.attend(0, q)
    ob = cache.attend(0, q, out_dtype=torch.bfloat16)
    assert ob.dtype == torch.bfloat16 and ob.shape == o16.shape
    x, y = o16.float(), ob.float()
    assert torch.all((x - y).abs() <= 2.0 ** -7 * x.abs().clamp_min(2.0 ** -20))
    assert cache._layers[0].args.out_bf16 == 0  # reset after the call
    kk = np.concatenate([k, k[:, :5]], 1).astype(np.float32)
    vv = np.concatenate([v, v[:, :5]], 1).astype(np.float32)
    for u in range(units):
        ref = _oracle_attend(kk[u], vv[u], q[u].float().cpu().numpy(), 4, [T], 5)
        assert rel(ref, y[u].cpu().numpy()) < TOL + 2.0 ** -8
    from paper_2405_12591_b200.errors import DimMismatch

    with pytest.raises(DimMismatch):
        cache.attend(0, q, out=torch.empty_like(q), out_dtype=torch.bfloat16)


# ---- north_star config shapes (BASELINE.json configs[3], configs[4], configs[2]) ------------

@pytest.mark.parametrize("scale", [1.0, 20.0])
def test_c4_shape_32k(dq, scale):
    """C4: int4, g = 1, T = 32768 (16-64 partials per unit, a Gram over 65,536 columns), the
    default plan (512-row items), plain and x20 outlier keys."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(32768 + int(scale))
    units, T = 2, 32768
    k = rng.standard_normal((units, T, 128)).astype(np.float32)
    k[:, :, [3, 77]] *= scale
    k = k.astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, 1, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=1, bits=4)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    a = cache._layers[0].args
    assert a.path == 0 and a.nwork >= 2 * 8
    for u in range(units):
        ref = _oracle_attend(k[u].astype(np.float32), v[u].astype(np.float32), q[u].astype(np.float32), 4, [T], 0)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


@pytest.mark.parametrize("scale", [1.0, 50.0])
def test_c5_shape_gqa_16k(dq, scale):
    """C5: g = 8 query heads per kv head, T = 16384, int4 on the tcgen05 GQA kernel (path 2),
    plain and x50 outlier keys."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(16384 + int(scale))
    units, g, T = 2, 8, 16384
    k = rng.standard_normal((units, T, 128)).astype(np.float32)
    k[:, :, [3, 77]] *= scale
    k = k.astype(np.float16)
    v = rng.standard_normal((units, T, 128)).astype(np.float16)
    q = rng.standard_normal((units, g, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=g, bits=4)
    cache.prefill(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out = cache.attend(0, torch.from_numpy(q).cuda()).float().cpu().numpy()
    assert cache._layers[0].args.path == 2
    for u in range(units):
        ref = _oracle_attend(k[u].astype(np.float32), v[u].astype(np.float32), q[u].astype(np.float32), 4, [T], 0)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


def test_c3_shape_int2_tail512(dq):
    """C3: int2, T = 8192 on the default plan (512-row items), plus a 512-token fp16 tail
    appended through the fused append."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    rng = np.random.default_rng(8192)
    units, T, tail = 2, 8192, 512
    k = rng.standard_normal((units, T + tail, 128)).astype(np.float16)
    v = rng.standard_normal((units, T + tail, 128)).astype(np.float16)
    q = rng.standard_normal((units, 1, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=1, bits=2)
    kd, vd, qd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(q).cuda()
    cache.prefill(0, kd[:, :T], vd[:, :T])
    for t in range(T, T + tail):
        cache.attend(0, qd, append=(kd[:, t], vd[:, t]))
    out = cache.attend(0, qd).float().cpu().numpy()
    assert cache._layers[0].args.chunk_b == 512 and cache._layers[0].tail_len == tail
    for u in range(units):
        ref = _oracle_attend(k[u].astype(np.float32), v[u].astype(np.float32), q[u].astype(np.float32), 2, [T], tail)
        assert rel(ref, out[u]) < TOL, (u, rel(ref, out[u]))


@pytest.mark.parametrize("g", [1, 8])
def test_decode_crosses_1024_seal(dq, g):
    """Decode through the default 1024-token seal (kvcache.py:116-128): outputs against the
    oracle's own cache lifecycle just before, at and after the step that seals the tail."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    units, P, chunk = 2, 1536, 1024
    steps = chunk + 6
    rng = np.random.default_rng(1024 + g)
    k = rng.standard_normal((units, P + steps, 128)).astype(np.float32)
    k[:, :, [9, 100]] *= 8.0
    k = k.astype(np.float16)
    v = rng.standard_normal((units, P + steps, 128)).astype(np.float16)
    q = rng.standard_normal((steps, units, g, 128)).astype(np.float16)
    cache = DecodeKvCache(layers=1, units=units, g=g, bits=4, chunk_len=chunk)
    kd, vd, qd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(q).cuda()
    cache.prefill(0, kd[:, :P], vd[:, :P])
    oracles = []
    for u in range(units):
        lay = O.LayerOracle(128, 4, chunk)
        lay.prefill(k[u, :P].astype(np.float32), v[u, :P].astype(np.float32))
        oracles.append(lay)
    check = {chunk - 2, chunk - 1, chunk, chunk + 1, steps - 1}
    for t in range(steps):
        out = cache.attend(0, qd[t], append=(kd[:, P + t], vd[:, P + t]))
        if t in check:
            o = out.float().cpu().numpy()
            for u in range(units):
                ref = oracles[u].attend(q[t, u].astype(np.float32))
                assert rel(ref, o[u]) < TOL, (t, u, rel(ref, o[u]))
        for u in range(units):
            oracles[u].append(k[u, P + t].astype(np.float32), v[u, P + t].astype(np.float32))
    lay = cache._layers[0]
    assert len(lay.groups) == 2 and lay.tail_len == steps - chunk
    assert cache.tokens(0) == oracles[0].tokens == P + steps


@pytest.mark.parametrize("g", [1, 8])
def test_tail_only_q_from_previous_kernel(dq, g):
    """A tail-only layer (no segments: no prepare / split kernels) whose q is written by the
    kernel launched right before the attention: the combine must see that q (no PDL edge to
    q's producer)."""
    from paper_2405_12591_b200.attention import DecodeKvCache

    units, steps = 4, 40
    rng = np.random.default_rng(3 + g)
    k = torch.from_numpy(rng.standard_normal((units, steps, 128)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((units, steps, 128)).astype(np.float16)).cuda()
    x = torch.from_numpy(rng.standard_normal((steps, units, g, 128)).astype(np.float32)).cuda()
    cache = DecodeKvCache(layers=1, units=units, g=g, bits=4, chunk_len=64, kernel_g=8 if g == 8 else None)
    q = torch.empty((units, g, 128), dtype=torch.float16, device="cuda")
    for t in range(steps):
        torch.mul(x[t], 0.5, out=x[t])  # a kernel in front of q's producer
        q.copy_(x[t])                   # q's producer, immediately before the attention
        out = cache.attend(0, q, append=(k[:, t], v[:, t]))
        if t == 0:
            assert torch.count_nonzero(out) == 0
            continue
        qn = q.float().cpu().numpy().astype(np.float64)
        kk, vv = k[:, :t].float().cpu().numpy(), v[:, :t].float().cpu().numpy()
        o = out.float().cpu().numpy()
        for u in range(units):
            s = qn[u] @ kk[u].T / np.sqrt(128)
            p = np.exp(s - s.max(1, keepdims=True))
            p /= p.sum(1, keepdims=True)
            assert rel(p @ vv[u], o[u]) < TOL, (t, u)


def test_step_graph_refuses_stale_plan(dq):
    """A replay after a re-plan (here a seal run eagerly) raises instead of replaying the
    captured segment tables; recapture() restores replays."""
    from paper_2405_12591_b200.attention import DecodeKvCache
    from paper_2405_12591_b200.decode_step import DecodeStepGraph
    from paper_2405_12591_b200.errors import ShapeMismatch

    L, U, g, chunk = 2, 2, 1, 8
    cache = DecodeKvCache(layers=L, units=U, g=g, bits=4, chunk_len=chunk)
    kv = torch.randn((L, 2, U, 520, 128), device="cuda").half()
    for layer in range(L):
        cache.prefill(layer, kv[layer, 0], kv[layer, 1])
    q_h = torch.randn((L, U, g, 128)).half().pin_memory()
    k_h = torch.randn((L, U, 128)).half().pin_memory()
    v_h = torch.randn((L, U, 128)).half().pin_memory()
    out_h = torch.empty((L, U, g, 128), dtype=torch.float16).pin_memory()
    st = DecodeStepGraph(cache, q_h, k_h, v_h, out_h)
    while cache._layers[0].tail_len + 1 < chunk:
        st.replay()
    with pytest.raises(ShapeMismatch):
        st.replay()  # this token seals
    for layer in range(L):  # the sealing step, eagerly
        cache.attend(layer, q_h[layer].cuda(), append=(k_h[layer].cuda(), v_h[layer].cuda()))
    assert all(lay.seal_pending for lay in cache._layers)  # full tails wait for one batched K3 call
    cache.check_errors()
    assert cache._layers[0].tail_len == 0 and len(cache._layers[1].groups) == 2
    with pytest.raises(ShapeMismatch):
        st.replay()  # stale: layer 0 was re-planned
    st.recapture()
    st.replay()
    torch.cuda.synchronize()
    assert cache.tokens(0) == 520 + chunk + 2


def test_seal_error_is_deferred_not_lost(dq):
    """A non-finite row in a chunk that seals while decoding: no host sync at the seal; the
    error (NonFiniteSvdInput, as the reference's LinAlgError) surfaces at check_errors() and at
    the first later call once the device flags are on the host."""
    from paper_2405_12591_b200.attention import DecodeKvCache
    from paper_2405_12591_b200.errors import NonFiniteInput

    units, chunk = 2, 32
    cache = DecodeKvCache(layers=1, units=units, g=1, bits=4, chunk_len=chunk)
    cache.prefill(0, torch.randn((units, 256, 128), device="cuda").half(),
                  torch.randn((units, 256, 128), device="cuda").half())
    rows = torch.randn((chunk, units, 128), device="cuda").half()
    rows[5, 1, 7] = float("nan")
    for t in range(chunk):
        cache.append_token(0, rows[t], rows[t])
    assert cache._layers[0].seal_pending  # full tail: sealed at the layer's next use
    with pytest.raises(NonFiniteInput):
        cache.check_errors()
    assert not cache._pending and len(cache._layers[0].groups) == 2
    cache2 = DecodeKvCache(layers=1, units=units, g=1, bits=4, chunk_len=chunk)
    for t in range(chunk + 1):  # the last append seals the full tail first (no sync, no raise)
        cache2.append_token(0, rows[t % chunk], rows[t % chunk])
    assert len(cache2._layers[0].groups) == 1 and cache2._layers[0].tail_len == 1
    torch.cuda.synchronize()
    with pytest.raises(NonFiniteInput):
        cache2.append_token(0, rows[0], rows[0])


@pytest.mark.parametrize("T,rows,bits,cols", [(8192, 5, 4, 128), (16384, 2, 4, 128), (1000, 7, 2, 128), (96, 3, 8, 128),
                                               (4096, 1, 4, 128), (2048, 3, 4, 256), (512, 2, 4, 64)])
def test_fused_reads_long_and_ragged(dq, T, rows, bits, cols):
    """The two-phase fused reads (reads.cu: bond-row groups for x @ W^T, b chunks for x @ W,
    fp64 partials summed in a fixed order) against the oracle's core-first sweeps on the
    oracle's own encoding, several query rows, partial tiles and chunks; the meter still sees
    one tile at most and every code once per query row."""
    rng = np.random.default_rng(T + rows)
    block = rng.standard_normal((T, cols)).astype(np.float16).astype(np.float32)
    e = O.encode(block, bits)
    qt = dq.QuantizedTensor((e.r, e.plan.i2, e.plan.j2, 1), bits, float(e.scale), e.payload)
    q = dq.QuantizedMpo(plan=dq.plan_shapes(T, cols, 2), bits=bits, local_tensors=(e.core0, qt))
    xt = rng.standard_normal((rows, cols)).astype(np.float32)
    x = rng.standard_normal((rows, T)).astype(np.float32)
    mt, m = dq.WorkingSetMeter(), dq.WorkingSetMeter()
    assert rel(O.matmul_t(xt, e), dq.fused_matmul_t(xt, q, mt)) < 1e-5
    assert rel(O.matmul(x, e), dq.fused_matmul(x, q, m)) < 1e-5
    for meter in (mt, m):
        assert 0 < meter.peak_elements <= 64 * 64
        assert meter.total_unpacked == rows * qt.count
    # deterministic: the partial sums are added in a fixed order
    assert np.array_equal(dq.fused_matmul_t(xt, q), dq.fused_matmul_t(xt, q))
    assert np.array_equal(dq.fused_matmul(x, q), dq.fused_matmul(x, q))


@pytest.mark.parametrize("L", [1, 9])
def test_step_graphs_grouped_copies_and_device(dq, L):
    """DecodeStepGraph's grouped host copies (uploads 1, 3, rest; downloads ..., 4, 2, 1) and
    DeviceStepGraph (the device-resident step as one graph) both equal eager attend per layer,
    for layer counts whose groups are ragged."""
    from paper_2405_12591_b200.attention import DecodeKvCache
    from paper_2405_12591_b200.decode_step import DecodeStepGraph, DeviceStepGraph

    U, P, steps = 3, 200, 4
    rng = np.random.default_rng(L)
    kv = torch.from_numpy(rng.standard_normal((L, 2, U, P, 128)).astype(np.float16)).cuda()
    caches = [DecodeKvCache(layers=L, units=U, g=1, bits=4, chunk_len=64) for _ in range(3)]
    for c in caches:
        for layer in range(L):
            c.prefill(layer, kv[layer, 0], kv[layer, 1])
    eager, hosted, device = caches
    q = torch.from_numpy(rng.standard_normal((L, U, 1, 128)).astype(np.float16)).cuda()
    k = torch.from_numpy(rng.standard_normal((L, U, 128)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((L, U, 128)).astype(np.float16)).cuda()
    q_h, k_h, v_h = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
    out_h = torch.empty(q_h.shape, dtype=torch.float16).pin_memory()
    out_d = torch.empty_like(q)
    hs = DecodeStepGraph(hosted, q_h, k_h, v_h, out_h)  # each runs one eager step, then captures
    ds = DeviceStepGraph(device, q, k, v, out_d)
    sizes = [b - a for a, b in hs.down_groups]
    assert sum(sizes) == L and sizes[-1] == 1 and [a for a, _ in hs.up_groups][:2] == [0, 1][:len(hs.up_groups)]
    for t in range(steps):
        ref = torch.stack([eager.attend(layer, q[layer], append=(k[layer], v[layer])) for layer in range(L)])
        if t > 0:
            hs.replay()
            ds.replay()
        torch.cuda.synchronize()
        assert torch.equal(out_h, ref.cpu()), t
        assert torch.equal(out_d, ref), t
    assert eager.tokens(0) == hosted.tokens(0) == device.tokens(0) == P + steps

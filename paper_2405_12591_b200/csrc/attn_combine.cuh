// Combine step of the fused decode attention (attention.cu): the partial merge, the dense
// fp16 tail and the fused append, run by the combine kernels behind the split kernel (PDL).
#pragma once

#include "attn_frag.cuh"

#ifndef DQ_TAIL_TV_GQ
#define DQ_TAIL_TV_GQ 1
#endif
#ifndef DQ_TAIL_MMA  // the GQA tail's scores on mma.sync (f16 in, f32 accumulate)
#define DQ_TAIL_MMA 1
#endif
#ifndef DQ_TAIL_ROWS  // K / V rows in flight per warp in the tail partial at g <= 2
#define DQ_TAIL_ROWS 8
#endif

namespace dq {
namespace attn {

// Combine of kv head unit u: merge its work-item partials (flash-decoding) with the dense
// fp16 tail, write the fp16 output, and (app_k) append the new token to the tail.  Thread
// d < 128 owns output dim d; threads d >= 128 of the calling group only join `sync`, a
// barrier over the whole group.  All head_groups virtual units of u run here: they share
// the tail, and the append must come after every head has read it.
// Dense fp16 tail attention of head h of virtual unit v (kv head unit u): the tail is one more
// flash-decoding partial (Mt, Lt, Ot) -- it does not depend on the split kernel, so the PDL
// combine computes it before waiting for the split kernel's partials.  nthr threads (a
// multiple of 128) of the calling group: scores warp-parallel over tokens (8 tokens in flight
// per warp), P.V warp-parallel over tokens (8 rows in flight) with each lane owning 4 dims, then a cross-warp
// reduction; thread d < 128 returns Ot for dim d.  tail_s holds tl floats, red 5 * nthr / 32
// floats... (red: [nw][128] O partials + [nw] sums + [nw] maxima).
template <int G, bool SCORED = false, class Sync>
__device__ __forceinline__ void tail_partial(const dq_attn_args& args, int u, int v, int h, int tid, int nthr, int tl,
                                             float* tail_s, float* red, Sync sync, float& Mt, float& Lt, float& Ot) {
  // SCORED: tail_s already holds the scores (log2 domain) and the caller has synchronised
  const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
  const float l2e = 1.4426950408889634f;
  const __half* qh = reinterpret_cast<const __half*>(args.q) + ((size_t)v * G + h) * 128;
  const uint2 qv = reinterpret_cast<const uint2*>(qh)[lane];
  const __half2* q2 = reinterpret_cast<const __half2*>(&qv);
  const float2 qa = __half22float2(q2[0]), qb = __half22float2(q2[1]);
  const __half* tk = reinterpret_cast<const __half*>(args.tail_k) + (size_t)u * args.tail_cap * 128;
  const __half* tv = reinterpret_cast<const __half*>(args.tail_v) + (size_t)u * args.tail_cap * 128;
  constexpr int kTK = G >= 8 ? 4 : DQ_TAIL_ROWS;  // rows in flight per warp (the GQA combine runs at 32 registers)
  for (int t0 = warp; !SCORED && t0 < tl; t0 += kTK * nw) {
    float dot[kTK];
#pragma unroll
    for (int i = 0; i < kTK; ++i) {
      const int t = t0 + i * nw;
      dot[i] = 0.f;
      if (t < tl) {
        const uint2 kv = reinterpret_cast<const uint2*>(tk + (size_t)t * 128)[lane];
        const __half2* k2 = reinterpret_cast<const __half2*>(&kv);
        const float2 ka = __half22float2(k2[0]), kb = __half22float2(k2[1]);
        dot[i] = qa.x * ka.x + qa.y * ka.y + qb.x * kb.x + qb.y * kb.y;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
      for (int i = 0; i < kTK; ++i) dot[i] += __shfl_xor_sync(0xffffffffu, dot[i], o);
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < kTK; ++i)
        if (t0 + i * nw < tl) tail_s[t0 + i * nw] = dot[i] * args.sm_scale * l2e;  // log2 domain
    }
  }
  if (!SCORED) sync();
  float m = -INFINITY;
  for (int t = tid; t < tl; t += nthr) m = fmaxf(m, tail_s[t]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float* red_o = red;             // [nw][128]
  float* red_l = red + nw * 128;  // [nw]
  float* red_m = red_l + nw;      // [nw]
  if (lane == 0) red_m[warp] = m;
  sync();
  m = red_m[0];
  for (int w = 1; w < nw; ++w) m = fmaxf(m, red_m[w]);
  // P once per token (not once per lane of every warp that reads it): the tail's exp2 work
  // drops 32x (the GQA combine's SFU load)
  for (int t = tid; t < tl; t += nthr) tail_s[t] = exp2f(tail_s[t] - m);
  sync();
  float o4[4] = {0.f, 0.f, 0.f, 0.f}, l = 0.f;
  // kTV rows in flight per warp (their loads before the arithmetic; the sums keep the order
  // t = warp, warp + nw, ...)
  constexpr int kTV = G >= 8 ? DQ_TAIL_TV_GQ : DQ_TAIL_ROWS;  // (GQA: 4 measured 1% slower at a 512-token tail)
  for (int t0 = warp; t0 < tl; t0 += kTV * nw) {
    uint2 vv[kTV];
    float p[kTV];
#pragma unroll
    for (int i = 0; i < kTV; ++i) {
      const int t = t0 + i * nw;
      vv[i] = make_uint2(0u, 0u);
      p[i] = 0.f;
      if (t < tl) {
        vv[i] = reinterpret_cast<const uint2*>(tv + (size_t)t * 128)[lane];
        p[i] = tail_s[t];
      }
    }
#pragma unroll
    for (int i = 0; i < kTV; ++i) {
      if (t0 + i * nw >= tl) break;
      l += p[i];
      const __half2* v2 = reinterpret_cast<const __half2*>(&vv[i]);
      const float2 va = __half22float2(v2[0]), vb = __half22float2(v2[1]);
      o4[0] = fmaf(p[i], va.x, o4[0]);
      o4[1] = fmaf(p[i], va.y, o4[1]);
      o4[2] = fmaf(p[i], vb.x, o4[2]);
      o4[3] = fmaf(p[i], vb.y, o4[3]);
    }
  }
  *reinterpret_cast<float4*>(red_o + warp * 128 + 4 * lane) = make_float4(o4[0], o4[1], o4[2], o4[3]);
  if (lane == 0) red_l[warp] = l;
  sync();
  Mt = m;
  Lt = 0.f;
  Ot = 0.f;
  for (int w = 0; w < nw; ++w) {
    Lt += red_l[w];
    if (tid < 128) Ot += red_o[w * 128 + tid];
  }
  sync();  // red and tail_s reusable
}

// Tail scores of all G heads of unit u at once (the GQA combine; at g = 1 the warp-per-token
// scores of tail_partial measured faster: 1.53 vs 1.71 ms per 16 C2 layers at a 512-token
// tail): each thread scores whole K rows (16-byte loads, 128 dims per thread: no cross-lane
// reductions) for HPT = min(G, 4) heads, G / HPT threads per token, q of the G heads from
// shared memory; each K row is read once for all heads.  tail_s[h * cap + t] = score in the
// log2 domain.
template <int G, int NT>
__device__ __forceinline__ void tail_scores_rows(const dq_attn_args& args, int u, int tl, int cap, float* tail_s,
                                                 float (*qs)[128]) {
  constexpr int HPT = G < 4 ? G : 4, TPT = G / HPT;
  const int tid = threadIdx.x;
  const float scl = args.sm_scale * 1.4426950408889634f;
  const __half* qh = reinterpret_cast<const __half*>(args.q) + (size_t)u * G * 128;
  for (int i = tid; i < G * 128; i += NT) qs[i / 128][i % 128] = __half2float(qh[i]);
  __syncthreads();
  const __half* tk = reinterpret_cast<const __half*>(args.tail_k) + (size_t)u * args.tail_cap * 128;
  const int h0 = HPT * (tid % TPT);
  for (int t = tid / TPT; t < tl; t += NT / TPT) {
    const uint4* krow = reinterpret_cast<const uint4*>(tk + (size_t)t * 128);
    float dot[HPT];
#pragma unroll
    for (int hh = 0; hh < HPT; ++hh) dot[hh] = 0.f;
#pragma unroll 4
    for (int c = 0; c < 16; ++c) {  // 8 dims per 16-byte load
      const uint4 kv = krow[c];
      const __half2* k2 = reinterpret_cast<const __half2*>(&kv);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 kf = __half22float2(k2[j]);
#pragma unroll
        for (int hh = 0; hh < HPT; ++hh) {
          const float2 qf = *reinterpret_cast<const float2*>(&qs[h0 + hh][c * 8 + 2 * j]);
          dot[hh] = fmaf(qf.x, kf.x, fmaf(qf.y, kf.y, dot[hh]));
        }
      }
    }
#pragma unroll
    for (int hh = 0; hh < HPT; ++hh) tail_s[(size_t)(h0 + hh) * cap + t] = dot[hh] * scl;
  }
  __syncthreads();
}

// Tail scores of the kGqG = 8 heads of unit u on the tensor cores (the GQA combine):
// S[h, t] = q[h, :] . K[t, :] as mma.sync m16n8k16 (f16 in, f32 accumulate; q and K are fp16,
// so the products are exact and only the summation order differs from the CUDA-core form).
// A = q (rows 0-7 = heads, rows 8-15 zero) held in registers for all 8 k-steps, B = 8 tokens'
// K rows straight from global (each lane two 32-bit loads per k-step), one warp per 8 tokens.
// tail_s[h * cap + t] = score in the log2 domain.
template <int NT>
__device__ __forceinline__ void tail_scores_mma(const dq_attn_args& args, int u, int tl, int cap, float* tail_s) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, c2 = 2 * (lane & 3);
  const float scl = args.sm_scale * 1.4426950408889634f;
  const uint32_t* q32 = reinterpret_cast<const uint32_t*>(reinterpret_cast<const __half*>(args.q) +
                                                          (size_t)u * 8 * 128 + (size_t)g * 128);
  uint32_t qa[8][2];  // per k-step: A registers 0 (row g, dims c2, c2+1) and 2 (row g, dims c2+8, c2+9)
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    qa[ks][0] = q32[(ks * 16 + c2) >> 1];
    qa[ks][1] = q32[(ks * 16 + c2 + 8) >> 1];
  }
  const __half* tk = reinterpret_cast<const __half*>(args.tail_k) + (size_t)u * args.tail_cap * 128;
  for (int t0 = warp * 8; t0 < tl; t0 += (NT / 32) * 8) {
    const int tb = min(t0 + g, tl - 1);  // this lane's B column (token); past the tail: a valid row, discarded
    const uint32_t* k32 = reinterpret_cast<const uint32_t*>(tk + (size_t)tb * 128);
    float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const uint32_t b0 = k32[(ks * 16 + c2) >> 1], b1 = k32[(ks * 16 + c2 + 8) >> 1];
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
          : "r"(qa[ks][0]), "r"(0u), "r"(qa[ks][1]), "r"(0u), "r"(b0), "r"(b1));
    }
    // d[0], d[1]: head g, tokens t0 + c2, t0 + c2 + 1 (rows 8-15, d[2..3], are the zero padding)
    if (t0 + c2 < tl) tail_s[(size_t)g * cap + t0 + c2] = d[0] * scl;
    if (t0 + c2 + 1 < tl) tail_s[(size_t)g * cap + t0 + c2 + 1] = d[1] * scl;
  }
  __syncthreads();
}

// The whole tail partial of the GQA combine (all kGqG heads of unit u, NT = kGqG * 128
// threads, group grp = head): scores with whole K rows per thread (tail_scores_rows), the
// group's maximum and P in place, then P.V with each warp on a head pair and an eighth of the
// tokens (a V row feeds two heads; V is read 4 times per CTA instead of 8), the 8 token
// subsets' partials added in a fixed order through red (>= 16 * 256 floats).  Thread d < 128
// of group grp returns (Mt, Lt, Ot[d]) of head grp.
template <int NT, class GSync>
__device__ __forceinline__ void tail_gq(const dq_attn_args& args, int u, int tl, int cap, float* tail_sg,
                                        float (*qs)[128], float* red, float* gred, GSync gsync, float& Mt, float& Lt,
                                        float& Ot) {
  constexpr int G = 8;
  const int tid = threadIdx.x, grp = tid >> 7, d = tid & 127, lane = tid & 31, warp = tid >> 5;
#if DQ_TAIL_MMA
  tail_scores_mma<NT>(args, u, tl, cap, tail_sg);
  (void)qs;
#else
  tail_scores_rows<G, NT>(args, u, tl, cap, tail_sg, qs);
#endif
  // the group's maximum, then P = exp2(s - m) in place and its sum (gred: 8 floats per group)
  float* srow = tail_sg + (size_t)grp * cap;
  float m = -INFINITY;
  for (int t = d; t < tl; t += 128) m = fmaxf(m, srow[t]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) gred[(warp & 3)] = m;
  gsync();
  m = fmaxf(fmaxf(gred[0], gred[1]), fmaxf(gred[2], gred[3]));
  float l = 0.f;
  for (int t = d; t < tl; t += 128) {
    const float p = exp2f(srow[t] - m);
    srow[t] = p;
    l += p;
  }
  for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  if (lane == 0) gred[4 + (warp & 3)] = l;
  __syncthreads();  // every head's P is in place
  l = (gred[4] + gred[5]) + (gred[6] + gred[7]);
  // P.V: warp = (head pair hp, token subset ts), lane = dims 4 lane .. 4 lane + 3
  const int hp = warp >> 3, ts = warp & 7;
  const float* p0 = tail_sg + (size_t)(2 * hp) * cap;
  const float* p1 = p0 + cap;
  const __half* tv = reinterpret_cast<const __half*>(args.tail_v) + (size_t)u * args.tail_cap * 128;
  float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  for (int t = ts; t < tl; t += 8) {
    const uint2 vv = reinterpret_cast<const uint2*>(tv + (size_t)t * 128)[lane];
    const __half2* v2 = reinterpret_cast<const __half2*>(&vv);
    const float2 va = __half22float2(v2[0]), vb = __half22float2(v2[1]);
    const float a = p0[t], b = p1[t];
    o[0][0] = fmaf(a, va.x, o[0][0]);
    o[0][1] = fmaf(a, va.y, o[0][1]);
    o[0][2] = fmaf(a, vb.x, o[0][2]);
    o[0][3] = fmaf(a, vb.y, o[0][3]);
    o[1][0] = fmaf(b, va.x, o[1][0]);
    o[1][1] = fmaf(b, va.y, o[1][1]);
    o[1][2] = fmaf(b, vb.x, o[1][2]);
    o[1][3] = fmaf(b, vb.y, o[1][3]);
  }
  // partials of token subsets ts and ts + 4 into slot (ts & 3), then the 4 slots in order
  float* slot = red + ((ts & 3) * 4 + hp) * 256;  // [slot][head pair][2 heads x 128 dims]
  if (ts < 4) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      *reinterpret_cast<float4*>(slot + k * 128 + 4 * lane) = make_float4(o[k][0], o[k][1], o[k][2], o[k][3]);
  }
  __syncthreads();
  if (ts >= 4) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      float4* dst = reinterpret_cast<float4*>(slot + k * 128 + 4 * lane);
      const float4 x = *dst;
      *dst = make_float4(x.x + o[k][0], x.y + o[k][1], x.z + o[k][2], x.w + o[k][3]);
    }
  }
  __syncthreads();
  const float* hsum = red + (grp >> 1) * 256 + (grp & 1) * 128 + d;
  Ot = (hsum[0] + hsum[4 * 256]) + (hsum[8 * 256] + hsum[12 * 256]);
  Mt = m;
  Lt = l;
  __syncthreads();  // red and tail_sg reusable
}

// Merge of head h of virtual unit v: its work-item partials plus the tail partial (Mt, Lt, Ot;
// Mt = -inf without a tail), fp16 (or bf16: out_bf16) output row.  Thread d < 128 owns dim d.
template <int G>
__device__ __forceinline__ void merge_head(const dq_attn_args& args, int v, int h, int d, float Mt, float Lt, float Ot) {
  if (d >= 128) return;
  const int p0 = args.unit_part0[v], np = args.unit_nparts[v];
  // partials in passes of 8 with every load issued before the arithmetic (the sums keep the
  // partials' order)
  constexpr int kB = 8;
  float M = Mt;
  for (int i0 = 0; i0 < np; i0 += kB) {
    float m[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) m[k] = i0 + k < np ? args.part_ml[((size_t)(p0 + i0 + k) * G + h) * 2] : -INFINITY;
#pragma unroll
    for (int k = 0; k < kB; ++k) M = fmaxf(M, m[k]);
  }
  float L = 0.f, O = 0.f;
  if (Mt != -INFINITY) {
    const float f = exp2f(Mt - M);
    L = f * Lt;
    O = f * Ot;
  }
  for (int i0 = 0; i0 < np; i0 += kB) {
    float m[kB], l[kB], o[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const size_t s = (size_t)(p0 + min(i0 + k, np - 1)) * G + h;
      m[k] = i0 + k < np ? args.part_ml[s * 2] : -INFINITY;
      l[k] = args.part_ml[s * 2 + 1];
      o[k] = args.part_o[s * 128 + d];
    }
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      if (m[k] == -INFINITY) continue;
      const float f = exp2f(m[k] - M);
      L += f * l[k];
      O += f * o[k];
    }
  }
  const float o = L > 0.f ? O / L : 0.f;
  const size_t i = ((size_t)v * G + h) * 128 + d;
  if (args.out_bf16) reinterpret_cast<__nv_bfloat16*>(args.out)[i] = __float2bfloat16_rn(o);  // one rounding
  else reinterpret_cast<__half*>(args.out)[i] = __float2half_rn(o);
}

// One head: tail partial then merge (callers that have already waited for the split kernel)
template <int G, class Sync>
__device__ __forceinline__ void combine_head(const dq_attn_args& args, int u, int v, int h, int d, int nthr, int tl,
                                             float* tail_s, float* red, Sync sync) {
  float Mt = -INFINITY, Lt = 0.f, Ot = 0.f;
  if (tl > 0) tail_partial<G>(args, u, v, h, d, nthr, tl, tail_s, red, sync, Mt, Lt, Ot);
  merge_head<G>(args, v, h, d, Mt, Lt, Ot);
}

// fused dq_tail_append: the new token joins unit u's tail after this step's attention (the
// caller's barrier guarantees every head has read tail_len[u] and the tail)
__device__ __forceinline__ void combine_append(const dq_attn_args& args, int u, int d, int tl) {
  if (d < 128 && tl < args.tail_cap) {
    const size_t dst = ((size_t)u * args.tail_cap + tl) * 128 + d;
    reinterpret_cast<__half*>(args.tail_k)[dst] = reinterpret_cast<const __half*>(args.app_k)[(size_t)u * 128 + d];
    reinterpret_cast<__half*>(args.tail_v)[dst] = reinterpret_cast<const __half*>(args.app_v)[(size_t)u * 128 + d];
  }
  if (d == 0) args.tail_len[u] = tl + 1;
}

// Combine of kv head unit u: merge its work-item partials (flash-decoding) with the dense
// fp16 tail, write the fp16 output, and (app_k) append the new token to the tail.  All
// head_groups virtual units of u run here, head after head: they share the tail, and the
// append must come after every head has read it.
template <int G, class Sync>
__device__ __forceinline__ void combine_unit(const dq_attn_args& args, int u, int d, int nthr, float* tail_s, float* red,
                                             Sync sync) {
  const int hg = args.head_groups > 1 ? args.head_groups : 1;
  const int tl = args.tail_len ? args.tail_len[u] : 0;
  for (int hh = 0; hh < G * hg; ++hh)
    combine_head<G>(args, u, u * hg + hh / G, hh % G, d, nthr, tl, tail_s, red, sync);
  if (args.app_k) {
    sync();  // every thread has read tail_len[u]
    combine_append(args, u, d, tl);
  }
}

}  // namespace attn
}  // namespace dq

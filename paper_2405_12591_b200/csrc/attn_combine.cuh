// Combine step of the fused decode attention (attention.cu): the standalone combine
// kernel, or the split kernel's last work item of a unit (fused combine).
#pragma once

#include "attn_frag.cuh"

namespace dq {
namespace attn {

// Combine of kv head unit u: merge its work-item partials (flash-decoding) with the dense
// fp16 tail, write the fp16 output, and (app_k) append the new token to the tail.  Thread
// d < 128 owns output dim d; threads d >= 128 of the calling group only join `sync`, a
// barrier over the whole group.  All head_groups virtual units of u run here: they share
// the tail, and the append must come after every head has read it.
// One head h of virtual unit v (of kv head unit u): merge the v's work-item partials with the
// dense fp16 tail and write the fp16 output row.  Thread d < 128 owns output dim d; `sync` is
// a barrier over the calling group (128 threads, or more threads that only join it).
template <int G, class Sync>
__device__ __forceinline__ void combine_head(const dq_attn_args& args, int u, int v, int h, int d, int tl,
                                             float* tail_s, float* red, Sync sync) {
  const int lane = d & 31, warp = d >> 5;
  const bool act = d < 128;
  const float l2e = 1.4426950408889634f;
  const int p0 = args.unit_part0[v], np = args.unit_nparts[v];
  // dense tail scores (log2 domain)
  float tm = -INFINITY;
  if (tl > 0) {
    const __half* qh = reinterpret_cast<const __half*>(args.q) + ((size_t)v * G + h) * 128;
    const uint2 qv = reinterpret_cast<const uint2*>(qh)[lane];
    const __half2* q2 = reinterpret_cast<const __half2*>(&qv);
    const float2 qa = __half22float2(q2[0]), qb = __half22float2(q2[1]);
    const __half* tk = reinterpret_cast<const __half*>(args.tail_k) + (size_t)u * args.tail_cap * 128;
    for (int t = warp; act && t < tl; t += 4) {
      const uint2 kv = reinterpret_cast<const uint2*>(tk + (size_t)t * 128)[lane];
      const __half2* k2 = reinterpret_cast<const __half2*>(&kv);
      const float2 ka = __half22float2(k2[0]), kb = __half22float2(k2[1]);
      float dot = qa.x * ka.x + qa.y * ka.y + qb.x * kb.x + qb.y * kb.y;
      for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (lane == 0) tail_s[t] = dot * args.sm_scale * l2e;
    }
    sync();
    for (int t = d; act && t < tl; t += 128) tm = fmaxf(tm, tail_s[t]);
    for (int o = 16; o; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
    if (act && lane == 0) red[warp] = tm;
    sync();
    tm = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    sync();
  }
  float M = tm;
  for (int i = 0; i < np; ++i) M = fmaxf(M, args.part_ml[((size_t)(p0 + i) * G + h) * 2]);
  float L = 0.f, O = 0.f;
  for (int i = 0; i < np; ++i) {
    const size_t s = (size_t)(p0 + i) * G + h;
    const float m = args.part_ml[s * 2];
    if (m == -INFINITY) continue;
    const float f = exp2f(m - M);
    L += f * args.part_ml[s * 2 + 1];
    O += f * args.part_o[s * 128 + (d & (128 - 1))];
  }
  if (tl > 0) {
    const __half* tv = reinterpret_cast<const __half*>(args.tail_v) + (size_t)u * args.tail_cap * 128;
    float lt = 0.f, ot = 0.f;
    for (int t = 0; act && t < tl; ++t) {
      const float p = exp2f(tail_s[t] - M);
      lt += p;
      ot = fmaf(p, __half2float(tv[(size_t)t * 128 + d]), ot);
    }
    L += lt;
    O += ot;
    sync();
  }
  __half* out = reinterpret_cast<__half*>(args.out) + ((size_t)v * G + h) * 128;
  if (act) out[d] = __float2half_rn(L > 0.f ? O / L : 0.f);
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
__device__ __forceinline__ void combine_unit(const dq_attn_args& args, int u, int d, float* tail_s, float* red,
                                             Sync sync) {
  const int hg = args.head_groups > 1 ? args.head_groups : 1;
  const int tl = args.tail_len ? args.tail_len[u] : 0;
  for (int hh = 0; hh < G * hg; ++hh) combine_head<G>(args, u, u * hg + hh / G, hh % G, d, tl, tail_s, red, sync);
  if (args.app_k) {
    sync();  // every thread has read tail_len[u]
    combine_append(args, u, d, tl);
  }
}

}  // namespace attn
}  // namespace dq

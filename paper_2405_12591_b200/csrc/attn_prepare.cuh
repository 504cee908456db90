// Prepare kernel of the fused decode attention: per segment, W = q . G0k turned into the
// two-limb int8 B operand of the score MMAs, written as the exact shared-memory image
// the split kernel loads with one TMA bulk copy (W depends on the segment, not on the
// work item, so it is computed once per segment instead of once per item).
#pragma once

#include "attn_frag.cuh"

namespace dq {
namespace attn {

constexpr int kMaxRW = 64;   // bond dimension bound of the W image
constexpr int kGroupR = 8;   // W is quantized per column and per bond-row group: rr < 8 | rr >= 8

// fixed-point precision of the two-limb (hi*256 + lo) 8-bit MMA operands; int8 codes
// use fewer bits so the s32 accumulators cannot overflow
template <int BITS>
constexpr int kWBits = BITS == 8 ? 13 : 15;  // |W * 2^sW| < 2^kWBits

// per-column metadata that follows the W chunks in the image
// the low bytes of 4 ints as one word (value j in byte j): 3 byte permutes
__device__ __forceinline__ uint32_t pack_low_bytes4(const int (&v)[4]) {
  return __byte_perm(__byte_perm((uint32_t)v[0], (uint32_t)v[1], 0x0040),
                     __byte_perm((uint32_t)v[2], (uint32_t)v[3], 0x0040), 0x5410);
}

template <int G>
struct WMeta {
  int beta[G][8][2];   // excess correction: kExcess * sum_k Wint[a][k] per bond-row group
  float cs[G][8][2];   // 2^(e - kWBits): Wint -> W
};

template <int G>
constexpr int kWChunkBytes = G * 2 * kMaxRW * 8 * 16;  // W limb chunks (bond rows >= r unused)
template <int G>
constexpr int kWImageBytes = kWChunkBytes<G> + (int)sizeof(WMeta<G>);

// 16-byte chunk of limb `limb` of W[h][a][rr][16 e] (e in ord16 order): bank-swizzled for
// the mma.sync fragments (path 0), or plain for tcgen05 (path 1: rows a of one bond row
// form a K-major core matrix, 8 rows x 16 bytes, the next bond row 128 bytes further)
__device__ __forceinline__ int w_chunk(int h, int limb, int r, int rr, int a, int path = 0) {
  if (path == 2)  // GQA path (8 heads, r = 64): slices of 8 bond rows [rr / 8][h*2 + limb][rr % 8][a], 16 KB each
    return (((rr >> 3) * 16 + h * 2 + limb) * 8 + (rr & 7)) * 8 + a;
  return ((h * 2 + limb) * r + rr) * 8 + (path ? a : (a ^ (2 * (rr & 3))));
}

// kPrepSplit CTAs per segment (blockIdx.y: a block of columns a; the W scales are per
// column, so the blocks are independent), one thread per (h, a, rr) of W (threads beyond i1 / r idle): a
// single wave of short-lived CTAs (the kernel is pure latency: ~16 KB in, ~16 KB out)
#ifndef DQ_PREP_SPLIT
#define DQ_PREP_SPLIT 4
#endif
constexpr int kPrepSplit = DQ_PREP_SPLIT;  // CTAs per segment, each 8 / kPrepSplit columns a
template <int G>
constexpr int kPrepThreadsOf = G * (8 / kPrepSplit) * kMaxRW;

// ASYM: the segments carry per-(rr, e) channel tables (asymmetric mode): their scales fold
// into W and their zero points into beta (instantiated separately so the symmetric kernel
// keeps its register budget)
template <int BITS, int G, bool ASYM = false>
__global__ void __launch_bounds__(kPrepThreadsOf<G>, (ASYM ? 1024 : 2048) / kPrepThreadsOf<G>)
    attn_prepare_kernel(dq_attn_args args) {
  constexpr int X = kExcess<BITS>;
  __shared__ __align__(16) float q[G][128];
  __shared__ unsigned wmax[G][8][2];
  __shared__ WMeta<G> meta;
  // the dependent split kernel may start its prologue (barriers, code copies) right away;
  // q may come from the previous kernel in the stream (launched with programmatic
  // serialization, this grid can be scheduled before that kernel finished): the segment
  // table and G0k (written at prefill) are loaded before waiting for it, q after
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int s = blockIdx.x;
  const int tid = threadIdx.x;
  constexpr int kA = 8 / kPrepSplit;
  const int h = G == 1 ? 0 : tid / (kA * kMaxRW), a = kA * blockIdx.y + (tid / kMaxRW) % kA, rr = tid % kMaxRW;
  const dq_segment& seg = args.segs[s];
  const int r = seg.r, i1 = seg.i1;
  const bool live = a < i1 && rr < r;
  // issue the global loads first: this thread's G0k row and (spread over threads) q
  const float4* g0k = reinterpret_cast<const float4*>(seg.k_g0);  // fp32 [a][rr][c], normalised
  float4 g_lo = make_float4(0.f, 0.f, 0.f, 0.f), g_hi = g_lo;
  if (live) {
    g_lo = g0k[2 * (a * r + rr)];
    g_hi = g0k[2 * (a * r + rr) + 1];
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  for (int i = tid; i < G * 128; i += kPrepThreadsOf<G>) {
    const __half* qh = reinterpret_cast<const __half*>(args.q) + (size_t)seg.unit * G * 128;
    q[i / 128][i % 128] = __half2float(qh[i]);
  }
  if (tid < G * 16) {
    (&meta.beta[0][0][0])[tid] = 0;
    (&wmax[0][0][0])[tid] = 0u;
  }
  __syncthreads();
  const float gk[8] = {g_lo.x, g_lo.y, g_lo.z, g_lo.w, g_hi.x, g_hi.y, g_hi.z, g_hi.w};
  // asymmetric mode: the per-(rr, e) channel scales fold into W, the zero points into beta
  const float* kch = (ASYM && live) ? seg.k_ch : nullptr;
  float chs[ASYM ? 16 : 1], chz[ASYM ? 16 : 1];
  if (ASYM && kch) {
    const float4* s4 = reinterpret_cast<const float4*>(kch + rr * 16);
    const float4* z4 = reinterpret_cast<const float4*>(kch + r * 16 + rr * 16);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 a4 = s4[k], b4 = z4[k];
      chs[4 * k] = a4.x, chs[4 * k + 1] = a4.y, chs[4 * k + 2] = a4.z, chs[4 * k + 3] = a4.w;
      chz[4 * k] = b4.x, chz[4 * k + 1] = b4.y, chz[4 * k + 2] = b4.z, chz[4 * k + 3] = b4.w;
    }
  }
  // path 2 keeps one scale per column: its S accumulators have no room for a second group
  const int grp = (rr < kGroupR || args.path == 2) ? 0 : 1;
  const int headroom = args.path ? 1 : 0;
  // W[h][a][rr][e] in fp32 (e in ord16 order), then one fixed-point scale 2^(kWBits - e2)
  // per (h, a, bond-row group) from the exact group maximum
  float wv[16];
  float m = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) wv[i] = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {  // q[h][c*16 .. c*16+15] as four broadcast 128-bit loads
    const float4* q4 = reinterpret_cast<const float4*>(&q[h][c * 16]);
    const float4 x0 = q4[0], x1 = q4[1], x2 = q4[2], x3 = q4[3];
    const float qc[16] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w, x2.x, x2.y, x2.z, x2.w, x3.x, x3.y, x3.z, x3.w};
#pragma unroll
    for (int i = 0; i < 16; i += 2)  // two fp32 FMAs per instruction (FFMA2), each rounded as fmaf
      ffma2(wv[i], wv[i + 1], qc[ord16<BITS>(i)], qc[ord16<BITS>(i + 1)], gk[c], gk[c]);
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if constexpr (ASYM) wv[i] *= chs[ord16<BITS>(i)];
    m = fmaxf(m, fabsf(wv[i]));
  }
  {  // per-group column maxima: warp reductions (a warp = 32 bond rows of one column), then
     // one shared atomic per warp and group instead of 32 contending ones
    const unsigned mu = live ? __float_as_uint(m) : 0u;
    const unsigned m0 = __reduce_max_sync(0xffffffffu, grp == 0 ? mu : 0u);
    const unsigned m1 = __reduce_max_sync(0xffffffffu, grp == 1 ? mu : 0u);
    if ((threadIdx.x & 31) == 0) {
      if (m0) atomicMax(&wmax[h][a][0], m0);
      if (m1) atomicMax(&wmax[h][a][1], m1);
    }
  }
  __syncthreads();
  int wtot = 0;  // this thread's share of beta
  if (live) {
    // the tcgen05 paths split both limbs signed: one bit of headroom keeps the hi limb in s8
    const float wq = pow2_sub_exp(__uint_as_float(wmax[h][a][grp]), kWBits<BITS> - headroom);
    uint32_t hi[4], lo[4];
    int wsum = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int wint[4], whi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = 4 * k + j;
        wint[j] = __float2int_rn(wv[i] * wq);
        // symmetric: sum of Wint (times the excess X below); asymmetric: sum of Wint * zero point
        if constexpr (ASYM) wsum += wint[j] * (int)chz[ord16<BITS>(i)];
        else wsum += wint[j];
        // path 0: hi signed, lo unsigned; paths 1 / 2: both signed (lo in [-128, 127]) so one
        // s8 UMMA takes both limbs; wint = 256 * hi + lo either way, and lo's byte is wint's
        // low byte in both cases
        whi[j] = args.path ? (wint[j] + 128) >> 8 : wint[j] >> 8;
      }
      hi[k] = pack_low_bytes4(whi);
      lo[k] = pack_low_bytes4(wint);
    }
    unsigned char* img = static_cast<unsigned char*>(args.wimg) + (size_t)s * args.wimg_stride;
    uint4* wout = reinterpret_cast<uint4*>(img);
    wout[w_chunk(h, 0, r, rr, a, args.path)] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    wout[w_chunk(h, 1, r, rr, a, args.path)] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    wtot = ASYM ? wsum : X * wsum;
  }
  if (ASYM || X) {  // beta per group: warp sums, one shared atomic per warp and group
    const int b0 = __reduce_add_sync(0xffffffffu, grp == 0 ? wtot : 0);
    const int b1 = __reduce_add_sync(0xffffffffu, grp == 1 ? wtot : 0);
    if ((threadIdx.x & 31) == 0) {
      if (b0) atomicAdd(&meta.beta[h][a][0], b0);
      if (b1) atomicAdd(&meta.beta[h][a][1], b1);
    }
  }
  __syncthreads();
  if (tid < G * 16 && ((tid >> 1) & 7) / (8 / kPrepSplit) == (int)blockIdx.y) {  // this CTA's columns
    int* mout = reinterpret_cast<int*>(static_cast<unsigned char*>(args.wimg) + (size_t)s * args.wimg_stride +
                                       kWChunkBytes<G>);
    const float cs = pow2_exp_sub(__uint_as_float((&wmax[0][0][0])[tid]), kWBits<BITS> - (args.path ? 1 : 0));
    mout[tid] = (&meta.beta[0][0][0])[tid];                               // beta[G][8][2]
    mout[G * 16 + tid] = __float_as_int(cs);                               // cs[G][8][2]
  }
}

// Prepare kernel of the tcgen05 GQA path (path 2: 8 heads, 4-bit codes, r = 64): one CTA per
// segment (512 threads, one per (bond row rr, column a)), heads in turn.  A head's 16 W values
// per thread stay in registers across its column-maximum reduction (warp shuffles + one shared
// atomic per column and warp, one barrier per head), so W is computed once.  A warp covers 4
// bond rows x 8 columns of one 8-row slice: each of its W stores is 512 contiguous bytes.
constexpr int kPrepGqThreads = 8 * kMaxRW;

__global__ void __launch_bounds__(kPrepGqThreads, 2) attn_prepare_gqa_kernel(dq_attn_args args) {
  constexpr int G = 8, X = kExcess<4>, WB = kWBits<4> - 1;  // both limbs signed: one bit of headroom
  __shared__ __align__(16) float q[G][128];
  __shared__ unsigned wmax[G][8];
  __shared__ int bsum[G][8];
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const int rr = tid >> 3, a = tid & 7;
  const dq_segment& seg = args.segs[s];
  const int r = seg.r;
  const bool live = rr < r;
  if (tid < G * 8) {
    (&wmax[0][0])[tid] = 0u;
    (&bsum[0][0])[tid] = 0;
  }
  // the segment table and G0k (written at prefill) before waiting for the previous kernel
  float gk[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (live) {
    const float4* g0k = reinterpret_cast<const float4*>(seg.k_g0);  // fp32 [a][rr][c], normalised
    const float4 g_lo = g0k[2 * (a * r + rr)], g_hi = g0k[2 * (a * r + rr) + 1];
    gk[0] = g_lo.x, gk[1] = g_lo.y, gk[2] = g_lo.z, gk[3] = g_lo.w;
    gk[4] = g_hi.x, gk[5] = g_hi.y, gk[6] = g_hi.z, gk[7] = g_hi.w;
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // q may come from the previous kernel
  const __half* qh = reinterpret_cast<const __half*>(args.q) + (size_t)seg.unit * G * 128;
  for (int i = tid; i < G * 128; i += kPrepGqThreads) q[i / 128][i % 128] = __half2float(qh[i]);
  __syncthreads();
  unsigned char* img = static_cast<unsigned char*>(args.wimg) + (size_t)s * args.wimg_stride;
  uint4* wout = reinterpret_cast<uint4*>(img);
#pragma unroll 1
  for (int h = 0; h < G; ++h) {
    float wv[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) wv[i] = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4* q4 = reinterpret_cast<const float4*>(&q[h][c * 16]);
      const float4 x0 = q4[0], x1 = q4[1], x2 = q4[2], x3 = q4[3];
      const float qc[16] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w, x2.x, x2.y, x2.z, x2.w, x3.x, x3.y, x3.z, x3.w};
#pragma unroll
      for (int i = 0; i < 16; i += 2)  // two fp32 FMAs per instruction (FFMA2), each rounded as fmaf
        ffma2(wv[i], wv[i + 1], qc[ord16<4>(i)], qc[ord16<4>(i + 1)], gk[c], gk[c]);
    }
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) m = fmaxf(m, fabsf(wv[i]));
    unsigned mu = __float_as_uint(m);
    mu = max(mu, __shfl_xor_sync(0xffffffffu, mu, 8));
    mu = max(mu, __shfl_xor_sync(0xffffffffu, mu, 16));
    if (lane < 8) atomicMax(&wmax[h][a], mu);
    __syncthreads();
    // two signed limbs per value, wint = 256 * hi + lo, |wint| < 2^WB (lo's byte = wint's low byte)
    const float wq = pow2_sub_exp(__uint_as_float(wmax[h][a]), WB);
    uint32_t hi[4], lo[4];
    int wsum = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int wint[4], whi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        wint[j] = __float2int_rn(wv[4 * k + j] * wq);
        wsum += wint[j];
        whi[j] = (wint[j] + 128) >> 8;
      }
      hi[k] = pack_low_bytes4(whi);
      lo[k] = pack_low_bytes4(wint);
    }
    if (live) {
      wout[w_chunk(h, 0, r, rr, a, 2)] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      wout[w_chunk(h, 1, r, rr, a, 2)] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    wsum += __shfl_xor_sync(0xffffffffu, wsum, 8);
    wsum += __shfl_xor_sync(0xffffffffu, wsum, 16);
    if (lane < 8) atomicAdd(&bsum[h][a], wsum);
  }
  __syncthreads();
  if (tid < G * 16) {  // metadata: beta[G][8][2], cs[G][8][2] (group 1 unused on this path)
    const int ha = tid >> 1, grp = tid & 1;
    int* mout = reinterpret_cast<int*>(img + kWChunkBytes<G>);
    mout[tid] = grp ? 0 : X * (&bsum[0][0])[ha];
    mout[G * 16 + tid] = __float_as_int(grp ? 0.f : pow2_exp_sub(__uint_as_float((&wmax[0][0])[ha]), WB));
  }
}

}  // namespace attn
}  // namespace dq

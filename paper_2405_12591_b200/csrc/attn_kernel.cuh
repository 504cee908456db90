// The split (work-item) kernel of the fused decode attention; see attention.cu for the
// math.  One CTA = one work item = (segment, 256-row slice of b).
#pragma once

#include "attn_prepare.cuh"

namespace dq {
namespace attn {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kD = 128;
constexpr int kMaxR = 64;
constexpr int kCB = 256;              // b rows per work item
constexpr int kTiles = kCB / kI2Pad;  // 64-row tiles per work item
constexpr int kNG = kCB / 16;         // 16-row groups per work item
constexpr int kStageBytes = 16384;
constexpr int kStages = 3;

template <int BITS>
constexpr int kPBits = 15;  // P / tile max in (0.5, 1] -> round(P * 2^(kPBits - e)); Y sums per 64-row tile

template <int G>
struct AttnSmem {
  alignas(128) unsigned char ring[kStages][kStageBytes];
  uint64_t full[kStages];
  uint64_t wbar;   // W image (attn_prepare.cuh) by TMA
  uint64_t g0bar;  // G0v prefetch
  unsigned int released[kStages];
  alignas(16) WMeta<G> wmeta;  // per-column W scales and excess corrections (TMA target)
  int gamma[G][8][kTiles]; // excess correction of Y per 64-row tile: kExcess * sum_b Pint[a][b]
  float lsum[G][kWarps];   // probability mass per warp
  unsigned pmax[G][8][kTiles];  // largest probability per (h, a, tile), float bits
  // K phase: W limbs, 16-byte chunks [((h*2 + limb)*r + rr)*8 + (a ^ 2*(rr&3))];
  // V phase (aliased): P limbs [((h*2 + limb)*8 + a)*kNG + (bg ^ 4*(a&1))]
  // K phase: W limbs; V phase + epilogue (aliased, W is dead): fp32 G0v [a][rr][c] by TMA
  union {
    uint4 w[G * 2 * kMaxR * 8];
    float4 g0v[8 * kMaxR * 2];
  } wg;
  // V phase: P limbs; epilogue (aliased, P is dead): cross-warp reduction of the O partial
  union {
    uint4 p[G * 2 * 8 * kNG];
    float red[kWarps][G][kD];
  } pr;
  float rowmax[G][kWarps];
};

// stage geometry of one work item (identical in every thread)
template <int BITS>
struct Plan {
  int r, nbt, bt0;
  int RK, nK;              // K stages: RK bond rows x nbt tiles each
  int rw, kslice, RV, nV;  // V stages: (tile, slice of RV bond rows)
  int nslices;
  __device__ Plan(const dq_segment& s, int wb0) {
    constexpr int RB = 2 * BITS;
    r = s.r;
    bt0 = wb0 / kI2Pad;
    nbt = min(kTiles, (s.i2p - wb0) / kI2Pad);
    RK = (kStageBytes / (nbt * kI2Pad * RB)) & ~3;
    if (RK > r) RK = r;
    nK = (r + RK - 1) / RK;
    rw = r / kWarps;
    kslice = kWarps;
    while (kslice > 1 && kslice * rw * 16 * kI2Pad * BITS / 8 > kStageBytes) kslice >>= 1;
    RV = kslice * rw;
    nslices = kWarps / kslice;
    nV = nbt * nslices;
  }
  __device__ int stages() const { return nK + nV; }
};

// issue stage `st` of the work item into its ring slot (one thread)
template <int BITS>
__device__ __forceinline__ void issue_stage(const Plan<BITS>& pl, const dq_segment& seg, int st,
                                            unsigned char* slot_buf, uint64_t* bar) {
  constexpr int RB = 2 * BITS;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (st < pl.nK) {
    const int rk0 = st * pl.RK;
    const int nr = min(pl.RK, pl.r - rk0);
    const uint32_t chunk = (uint32_t)(nr * kI2Pad * RB);
    mbar_expect_tx(bar, chunk * pl.nbt);
    for (int j = 0; j < pl.nbt; ++j) {
      const unsigned char* src = seg.k_codes + ((size_t)(pl.bt0 + j) * pl.r + rk0) * kI2Pad * RB;
      bulk_g2s(slot_buf + j * chunk, src, chunk, bar);
    }
  } else {
    const int v = st - pl.nK;
    const int btl = v / pl.nslices, sl = v % pl.nslices;
    const uint32_t bytes = (uint32_t)(pl.RV * 16 * kI2Pad * BITS / 8);
    mbar_expect_tx(bar, bytes);
    const unsigned char* src = seg.v_codes + ((size_t)(pl.bt0 + btl) * pl.r + sl * pl.RV) * 16 * kI2Pad * BITS / 8;
    bulk_g2s(slot_buf, src, bytes, bar);
  }
}


__device__ __forceinline__ int p_chunk(int h, int limb, int a, int bg) {
  return ((h * 2 + limb) * 8 + a) * kNG + (bg ^ (4 * (a & 1)));
}

template <int BITS, int G>
__global__ void __launch_bounds__(kThreads, G == 1 ? 3 : 2) decode_attn_kernel(dq_attn_args args) {
  constexpr int RB = 2 * BITS;
  constexpr int X = kExcess<BITS>;
  constexpr bool SA = BITS == 8;  // A operand (codes) signed
  extern __shared__ __align__(128) unsigned char smem_raw[];
  AttnSmem<G>& sm = *reinterpret_cast<AttnSmem<G>*>(smem_raw);

  const int wi = blockIdx.x;
  const int seg_id = args.work[2 * wi];
  const int wb0 = args.work[2 * wi + 1];
  const dq_segment seg = args.segs[seg_id];
  const int unit = seg.unit;
  const int r = seg.r, i1 = seg.i1, i2 = seg.i2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tid4 = lane & 3;
  const Plan<BITS> pl(seg, wb0);
  const int nstages = pl.stages();

  auto stamp = [&](int k) {  // optional per-item phase timestamps (profiling only)
    if (args.trace && tid == 0) args.trace[(size_t)wi * 8 + k] = global_ns();
  };
  stamp(0);
  if (args.trace && tid == 0) args.trace[(size_t)wi * 8 + 7] = sm_id();

  // ---- prologue: barriers + the first stages in flight before anything else ----------
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      sm.released[s] = 0;
    }
    mbar_init(&sm.wbar, 1);
    mbar_init(&sm.g0bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    // the code stages do not depend on the prepare kernel: start streaming right away
    for (int s = 0; s < kStages && s < nstages; ++s) issue_stage<BITS>(pl, seg, s, sm.ring[s], &sm.full[s]);
    // programmatic dependent launch: everything above overlapped the prepare kernel;
    // its output (the segment's W image: limb chunks + per-column metadata) is read below
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const unsigned char* img = static_cast<const unsigned char*>(args.wimg) + (size_t)seg_id * args.wimg_stride;
    const uint32_t wb = (uint32_t)(G * 2 * r * 8 * 16);
    mbar_expect_tx(&sm.wbar, wb + (uint32_t)sizeof(WMeta<G>));
    bulk_g2s(sm.wg.w, img, wb, &sm.wbar);
    bulk_g2s(&sm.wmeta, img + kWChunkBytes<G>, (uint32_t)sizeof(WMeta<G>), &sm.wbar);
  }
  if (tid < G * 8 * kTiles) {
    (&sm.gamma[0][0][0])[tid] = 0;
    (&sm.pmax[0][0][0])[tid] = 0u;
  }
  __syncthreads();  // barrier inits visible
  mbar_wait(&sm.wbar, 0);

  int st = 0;  // running stage index
  auto release = [&](int s) {
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const int slot = s % kStages;
      const unsigned target = (unsigned)(s / kStages + 1) * kWarps;
      const unsigned old = atomicAdd(&sm.released[slot], 1u);
      if (old + 1 == target && s + kStages < nstages)
        issue_stage<BITS>(pl, seg, s + kStages, sm.ring[slot], &sm.full[slot]);
    }
  };

  stamp(1);
  // ---- phase 1: S = W . codes_k on the int8 tensor pipe --------------------------------
  constexpr int MT = 2;                   // 16-row m-tiles per warp (32 b rows)
  const int jt = warp >> 1;               // tile of this warp inside the item
  const int bl_base = 32 * (warp & 1);    // first row of this warp inside the tile
  int acc_hi[MT][G][4], acc_lo[MT][G][4];
  float sacc[MT][G][4];  // scores in the log2 domain, accumulated per bond-row group
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int h = 0; h < G; ++h)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc_hi[mt][h][k] = acc_lo[mt][h][k] = 0;
        sacc[mt][h][k] = 0.f;
      }
  // s = Sint / wq[h][a][grp] * scale_k * sm_scale * log2(e), exact integer Sint per group
  const float kscale = seg.k_scale * args.sm_scale * 1.4426950408889634f;
  auto flush_group = [&](int grp) {
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float cs[2];
      int bt[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        cs[j] = kscale * sm.wmeta.cs[h][2 * tid4 + j][grp];
        bt[j] = sm.wmeta.beta[h][2 * tid4 + j][grp];
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          sacc[mt][h][k] += (float)(256 * acc_hi[mt][h][k] + acc_lo[mt][h][k] - bt[k & 1]) * cs[k & 1];
          acc_hi[mt][h][k] = acc_lo[mt][h][k] = 0;
        }
    }
  };
  for (int ks = 0; ks < pl.nK; ++ks, ++st) {
    const int slot = st % kStages;
    mbar_wait(&sm.full[slot], (uint32_t)((st / kStages) & 1));
    const int rk0 = ks * pl.RK;
    const int nr = min(pl.RK, r - rk0);
    if (jt < pl.nbt) {
      const unsigned char* tile = sm.ring[slot] + jt * nr * kI2Pad * RB;
      for (int q0 = 0; q0 < nr; q0 += 4) {
        const int rl = q0 + tid4;     // bond row inside the stage
        const int rr = rk0 + rl;      // global bond row
        const int swz = ktile_swizzle(rr, BITS);
        uint4 bh[G], bl[G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
          bh[h] = sm.wg.w[w_chunk(h, 0, r, rr, gid)];
          bl[h] = sm.wg.w[w_chunk(h, 1, r, rr, gid)];
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int b0 = bl_base + mt * 16 + gid;
          uint32_t x0[4], x1[4];
          row_bytes<BITS>(lds_row<BITS>(tile + (rl * kI2Pad + (b0 ^ swz)) * RB), x0);
          row_bytes<BITS>(lds_row<BITS>(tile + (rl * kI2Pad + ((b0 + 8) ^ swz)) * RB), x1);
#pragma unroll
          for (int h = 0; h < G; ++h) {
            imma<SA, true>(acc_hi[mt][h], x0[0], x1[0], x0[1], x1[1], bh[h].x, bh[h].y);
            imma<SA, false>(acc_lo[mt][h], x0[0], x1[0], x0[1], x1[1], bl[h].x, bl[h].y);
            imma<SA, true>(acc_hi[mt][h], x0[2], x1[2], x0[3], x1[3], bh[h].z, bh[h].w);
            imma<SA, false>(acc_lo[mt][h], x0[2], x1[2], x0[3], x1[3], bl[h].z, bl[h].w);
          }
        }
        if (rk0 + q0 + 4 == kGroupR) flush_group(0);  // leading bond rows carry their own W scale
      }
    }
    release(st);
  }
  if (r > kGroupR) flush_group(1);

  stamp(2);
  // ---- phase 2: softmax of the item straight from the accumulators ------------------------
  float sv[MT][G][4];
  float mh[G];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float m = -INFINITY;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int bl = jt * kI2Pad + bl_base + mt * 16 + gid + (k >= 2 ? 8 : 0);
        const int a = 2 * tid4 + (k & 1);
        const bool ok = (a < i1) && (wb0 + bl < i2) && (jt < pl.nbt);
        sv[mt][h][k] = ok ? sacc[mt][h][k] : -INFINITY;
        m = fmaxf(m, sv[mt][h][k]);
      }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) sm.rowmax[h][warp] = m;
  }
  __syncthreads();  // every warp is past phase 1: the W buffer is dead
  if (tid == 0) {   // prefetch the fp32 G0v for the epilogue into it
    const uint32_t gb = (uint32_t)(i1 * r * 32);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(&sm.g0bar, gb);
    bulk_g2s(sm.wg.g0v, seg.v_g0, gb, &sm.g0bar);
  }
  unsigned char* pb = reinterpret_cast<unsigned char*>(sm.pr.p);
  // P = exp2(s - m) in fixed point with one scale per (h, a, 64-row tile), set by that
  // tile's largest probability: small probabilities far from the peak keep their
  // relative precision (the V side combines its accumulators per tile anyway)
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float m = sm.rowmax[h][0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) m = fmaxf(m, sm.rowmax[h][w]);
    mh[h] = m;
    float tmax[2] = {0.f, 0.f};
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float s = sv[mt][h][k];
        sv[mt][h][k] = s == -INFINITY ? 0.f : exp2f(s - m);
        tmax[k & 1] = fmaxf(tmax[k & 1], sv[mt][h][k]);
      }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      float v = tmax[j];
      v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
      v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
      v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
      if (gid == 0 && jt < pl.nbt) atomicMax(&sm.pmax[h][2 * tid4 + j][jt], __float_as_uint(v));
    }
  }
  __syncthreads();  // per-tile probability maxima complete
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float lsum = 0.f;
    int gsum[2] = {0, 0};  // per a of this thread (a = 2*tid4, 2*tid4+1), this warp's tile
    float pq[2], pinv[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      int e2;
      frexpf(fmaxf(__uint_as_float(sm.pmax[h][2 * tid4 + j][min(jt, kTiles - 1)]), 1e-30f), &e2);
      pq[j] = ldexpf(1.f, kPBits<BITS> - e2);
      pinv[j] = ldexpf(1.f, e2 - kPBits<BITS>);
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int bl = jt * kI2Pad + bl_base + mt * 16 + gid + (k >= 2 ? 8 : 0);
        const int a = 2 * tid4 + (k & 1);
        const int pint = __float2int_rn(sv[mt][h][k] * pq[k & 1]);
        lsum += (float)pint * pinv[k & 1];  // the probability mass the PV product really uses
        gsum[k & 1] += pint;
        if (jt < pl.nbt) {
          const int pos = inv_ord16<BITS>(bl & 15);
          pb[p_chunk(h, 0, a, bl >> 4) * 16 + pos] = (unsigned char)(pint >> 8);
          pb[p_chunk(h, 1, a, bl >> 4) * 16 + pos] = (unsigned char)(pint & 0xFF);
        }
      }
    // per (a, tile) sums: reduce over the 8 gid lanes sharing tid4 (same a, same tile)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      int v = gsum[j];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      if (X && gid == 0 && jt < pl.nbt) atomicAdd(&sm.gamma[h][2 * tid4 + j][jt], X * v);
    }
    for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane == 0) sm.lsum[h][warp] = lsum;
  }
  __syncthreads();  // P limbs, gamma and lsum complete

  stamp(3);
  // ---- phase 3: Y = codes_v . P^T on the int8 tensor pipe ------------------------------
  // warp w owns bond rows w*rw .. w*rw+rw-1 (an m-tile = one bond row x 16 e)
  const int rw = pl.rw;
  const int my_slice = warp / pl.kslice;
  const int rbase_in_slice = (warp % pl.kslice) * rw;
  float accv[8][G][4];
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int h = 0; h < G; ++h)
#pragma unroll
      for (int k = 0; k < 4; ++k) accv[t][h][k] = 0.f;
  for (int vs = 0; vs < pl.nV; ++vs, ++st) {
    const int slot = st % kStages;
    mbar_wait(&sm.full[slot], (uint32_t)((st / kStages) & 1));
    const int btl = vs / pl.nslices, sl = vs % pl.nslices;
    if (sl == my_slice) {
      uint4 ph[G], pl_[G];
      int gam[G][2];
      float pinv[G][2];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        ph[h] = sm.pr.p[p_chunk(h, 0, gid, btl * 4 + tid4)];
        pl_[h] = sm.pr.p[p_chunk(h, 1, gid, btl * 4 + tid4)];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          gam[h][j] = sm.gamma[h][2 * tid4 + j][btl];
          int e2;
          frexpf(fmaxf(__uint_as_float(sm.pmax[h][2 * tid4 + j][btl]), 1e-30f), &e2);
          pinv[h][j] = ldexpf(1.f, e2 - kPBits<BITS>);
        }
      }
      const unsigned char* buf = sm.ring[slot];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (t < rw) {
          const int rl = rbase_in_slice + t;
          uint32_t x0[4], x1[4];
          row_bytes<BITS>(lds_row<BITS>(buf + (rl * 16 + gid) * 8 * BITS + RB * tid4), x0);
          row_bytes<BITS>(lds_row<BITS>(buf + (rl * 16 + gid + 8) * 8 * BITS + RB * tid4), x1);
#pragma unroll
          for (int h = 0; h < G; ++h) {
            // the excess correction seeds the low-limb accumulator
            int yh[4] = {0, 0, 0, 0}, yl[4] = {-gam[h][0], -gam[h][1], -gam[h][0], -gam[h][1]};
            imma<SA, false>(yh, x0[0], x1[0], x0[1], x1[1], ph[h].x, ph[h].y);
            imma<SA, false>(yl, x0[0], x1[0], x0[1], x1[1], pl_[h].x, pl_[h].y);
            imma<SA, false>(yh, x0[2], x1[2], x0[3], x1[3], ph[h].z, ph[h].w);
            imma<SA, false>(yl, x0[2], x1[2], x0[3], x1[3], pl_[h].z, pl_[h].w);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              accv[t][h][k] += (float)(256 * yh[k] + yl[k]) * pinv[h][k & 1];
          }
        }
      }
    }
    release(st);
  }

  stamp(4);
  // ---- phase 4: O = scale_v * G0v . Y on CUDA cores, reduce, write the partial ---------
  // accv[t][h]: rows e = gid (k 0,1) / gid+8 (k 2,3); cols a = 2*tid4 + (k & 1)
  float part[G][16];  // [h][c*2 + (e == gid+8)]
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int k = 0; k < 16; ++k) part[h][k] = 0.f;
  mbar_wait(&sm.g0bar, 0);  // fp32 G0v [a][rr][c] (normalised), prefetched into the W buffer
  const float4* g0v = sm.wg.g0v;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if (t < rw) {
      const int rr = warp * rw + t;
#pragma unroll
      for (int aa = 0; aa < 2; ++aa) {
        const int a = 2 * tid4 + aa;
        if (a < i1) {
          const float4 g_lo = g0v[2 * (a * r + rr)], g_hi = g0v[2 * (a * r + rr) + 1];
          const float gc[8] = {g_lo.x, g_lo.y, g_lo.z, g_lo.w, g_hi.x, g_hi.y, g_hi.z, g_hi.w};
#pragma unroll
          for (int h = 0; h < G; ++h)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              part[h][2 * c] = fmaf(gc[c], accv[t][h][aa], part[h][2 * c]);
              part[h][2 * c + 1] = fmaf(gc[c], accv[t][h][2 + aa], part[h][2 * c + 1]);
            }
        }
      }
    }
  }
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float v = part[h][k];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      part[h][k] = v;
    }
  __syncthreads();  // every warp is past the V stages: the P buffer may now hold the reduction
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const int c = 2 * tid4 + cc;
      float v0 = 0.f, v1 = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k == c) {
          v0 = part[h][2 * k];
          v1 = part[h][2 * k + 1];
        }
      sm.pr.red[warp][h][c * 16 + gid] = v0;
      sm.pr.red[warp][h][c * 16 + gid + 8] = v1;
    }
  __syncthreads();
  const int slot_out = args.work_part[wi];
  for (int i = tid; i < G * kD; i += kThreads) {
    const int h = i / kD, d = i % kD;
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) v += sm.pr.red[w][h][d];
    args.part_o[((size_t)slot_out * G + h) * kD + d] = v * seg.v_scale;
  }
  if (tid < G) {
    float l = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) l += sm.lsum[tid][w];
    args.part_ml[((size_t)slot_out * G + tid) * 2 + 0] = mh[tid];  // log2 domain
    args.part_ml[((size_t)slot_out * G + tid) * 2 + 1] = l;
  }
  stamp(5);
}

}  // namespace attn
}  // namespace dq

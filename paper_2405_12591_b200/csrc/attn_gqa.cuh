// tcgen05 split kernel for GQA groups of 8 query heads per kv head (path 2): 4-bit codes,
// full plans (i1 = 8, r = 64).  Same work items, persistent grid, ticket scheduler, producer
// warp and partials as paths 0 / 1; the contractions run on the 5th-generation tensor cores
// with all 8 heads, both fixed-point limbs and all 8 columns a in one N = 128 operand:
//
//   S[b, (h,l,a)]      = sum_{r,e} code_k[b, (r,e)] . W_l[(r,e), (h,a)]   M = 128 b, N = 128, K = (r,e)
//   Y[(r,e), (h,l,a)]  = sum_b code_v[(r,e), b] . P_l[b, (h,a)]          M = 128 (r,e), N = 128, K = b
//
// A operands (the codes) are widened from the shared-memory ring into tensor memory by the
// consumer warps (tcgen05.st: lane = row, 4 K-bytes per column); B operands sit in shared
// memory as K-major core matrices: the W image streams through the ring in 16 KB slices of
// 8 bond rows next to the K codes of the same bond rows (so no 128 KB W buffer: the ring is
// 5 x 32 KB deep), P is written by the softmax.  One elected lane of the MMA warp issues
// every UMMA (kind::i8, s32 accumulators in TMEM) and signals through tcgen05.commit; its
// commit is also the ring slot's last release (the UMMAs read W from the slot).
//
// Per work item (<= 256 rows b = 2 M-blocks): 8 K stages (8 bond rows x all tiles + W slice)
// -> S in TMEM (2 x 128 columns) -> softmax from TMEM -> P limbs in shared memory -> 8 V
// stages (one M-block of 8 bond rows x all tiles each) -> Y per stage (128 columns, double-
// buffered in the S columns) -> the epilogue folds Y with G0v on CUDA cores while the next
// stage's UMMAs run.  TMEM: 4 A buffers [0, 256), S / Y [256, 512).  16 consumer warps (4
// warpgroups: a warp reaches TMEM lanes 32 (warp % 4) ..): K widening by (M-block, bond-row
// half), softmax by (M-block, head half), V widening by tile, the Y fold by head pair.
//
// Numerics (exact integer products, as path 0): codes excess-coded u8; W = two signed 8-bit
// limbs of a 14-bit fixed point with one scale per (h, a) column; P = exp2(s - m_h) as a
// 15-bit fixed point with one scale per (h, a) column and item (the column maximum), two
// unsigned limbs.  The excess offset is removed with beta = X sum W (K) and X sum_b P (V).
#pragma once

#include "attn_tc.cuh"

namespace dq {
namespace attn {

constexpr int kGqG = 8;                            // query heads per kernel instance
constexpr int kGqStages = 5;                       // ring: 5 x 32 KB
constexpr int kGqSlot = 32768;                     // K stage: codes [0, 16 KB) + W slice [16 KB, 32 KB)
constexpr int kGqWSlice = 16 * 8 * 8 * 16;         // W slice: 16 (h, limb) x 8 bond rows x 8 a x 16 e = 16 KB
constexpr int kGqWarps = 16;                       // math warps (softmax, Y fold, epilogue): 4 warpgroups
constexpr int kGqCons = kGqWarps * 32;
constexpr int kGqWide = 4;                         // widening warpgroup: codes ring -> TMEM A operands
constexpr int kGqProducer = kGqWarps + kGqWide;    // producer warp (20), then the MMA warp (21)
constexpr int kGqMma = kGqProducer + 1;
constexpr int kGqThreads = kGqCons + kGqWide * 32 + 64;
constexpr int kGqTmemUsers = kGqCons + kGqWide * 32 + 32;  // threads that touch TMEM (final barrier)
constexpr int kGqNumA = 4;                         // TMEM A buffers (64 columns each)
constexpr uint32_t kGqColA = 0, kGqColSY = 256;    // A: 4 x 64 columns; S / Y: 2 x 128 columns
constexpr int kGqPBits = 15;
constexpr int kGqVTileBytes = 8 * 16 * kI2Pad / 2;  // V stage per tile: 8 bond rows x 16 e x 64 b

struct GqSmem {
  alignas(128) unsigned char ring[kGqStages][kGqSlot];
  // P limbs as core matrices [(h*2 + limb)][b / 16][a][16 b]; the epilogue's cross-warp
  // reduction reuses the buffer once every V UMMA of the item has completed
  union alignas(128) {
    unsigned char pb[kGqG * 2 * (kCB / 16) * 128];
    float red[4][kGqG][kD];  // [warp quarter][head][c * 16 + e]
  } pr;
  alignas(16) float4 g0v[8 * kMaxR * 2];           // fp32 G0v [a][rr][c]
  alignas(16) WMeta<kGqG> wmeta[2];                // beta, cs per (h, a) (group 0), by item parity
  alignas(16) float pinv[kGqG * 8];                // 2^(e - 15) of the P column maxima
  alignas(16) float xoff[kGqG * 8];                // -X * gsum * pinv: the excess offset of Y per column
  alignas(16) int gsum[kGqG * 8];                  // sum_b Pint per column
  unsigned pmax[kGqG * 8];
  float rowmax[2][8][4];                           // [head half][M-block * 4 + warp quarter][head]
  SubItem sub[kSubRing];
  uint64_t full[kGqStages], empty[kGqStages];
  uint64_t g0bar, descfull[kSubRing];
  uint64_t afull[kGqNumA], afree[kGqNumA], sfull, pfull, yfull[2], yfree[2];
  uint32_t tmem;
};
static_assert(sizeof(GqSmem) <= 232448, "path-2 shared memory exceeds the 227 KB opt-in limit");

// stage geometry of path 2: K stages of 8 bond rows x all tiles (codes <= 16 KB, + the W
// slice of those bond rows); V stages of 8 bond rows (one M-block of (r, e)) x all tiles
__device__ __forceinline__ void gq_load_sub(SubItem& d, const dq_attn_args& a, int w) {
  load_sub<4>(d, a, w);
  d.RK = 8;
  d.nK = d.r / 8;
  d.RV = 8;
  d.nslices = d.r / 8;
  d.stages = d.nK + d.nslices;
}

// stage `st` of item `d` (the k-th item of this CTA) into ring slot `buf` (one thread)
__device__ __forceinline__ void gq_issue_stage(GqSmem& sm, const dq_attn_args& a, const SubItem& d, int k, int st,
                                               unsigned char* buf, uint64_t* bar) {
  const int bt0 = d.wb0 / kI2Pad;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (st < d.nK) {
    constexpr uint32_t chunk = 8 * kI2Pad * 8;  // 8 bond rows x 64 b x 8 bytes per tile
    const unsigned char* img = static_cast<const unsigned char*>(a.wimg) + (size_t)d.seg * a.wimg_stride;
    const uint32_t meta = st == 0 ? (uint32_t)sizeof(WMeta<kGqG>) : 0u;
    mbar_expect_tx(bar, chunk * d.nbt + kGqWSlice + meta);
    const unsigned char* src = d.kc + ((size_t)bt0 * d.r + 8 * st) * kI2Pad * 8;
    for (int j = 0; j < d.nbt; ++j) bulk_g2s(buf + j * chunk, src + (size_t)j * d.r * kI2Pad * 8, chunk, bar);
    bulk_g2s(buf + 16384, img + (size_t)st * kGqWSlice, kGqWSlice, bar);
    if (meta) bulk_g2s(&sm.wmeta[k & 1], img + kWChunkBytes<kGqG>, meta, bar);
    return;
  }
  const int mbv = st - d.nK;
  mbar_expect_tx(bar, (uint32_t)(kGqVTileBytes * d.nbt));
  for (int t = 0; t < d.nbt; ++t) {
    const unsigned char* src = d.vc + ((size_t)(bt0 + t) * d.r + 8 * mbv) * 16 * kI2Pad / 2;
    bulk_g2s(buf + t * kGqVTileBytes, src, (uint32_t)kGqVTileBytes, bar);
  }
}

// 2^x on the SFU (ex2.approx.ftz: -inf -> +0, relative error ~2^-22)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^(k - e) for x = m * 2^e (m in [0.5, 1)), x >= 0 clamped below to 2^-100, as float bits
// (3 integer ops; pow2_sub_exp with the exponent field kept in place)
template <int K>
__device__ __forceinline__ float pow2_sub_exp3(unsigned xbits) {
  const unsigned e = max(xbits & 0x7F800000u, 27u << 23);
  return __uint_as_float(((unsigned)(K + 253) << 23) - e);
}

// one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile(
      "{\n.reg .pred P;\n.reg .b32 r;\nelect.sync r|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}" : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ void tc_ld16(uint32_t taddr, int (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

// warp reduce-scatter of N values per lane: afterwards lane l holds, in v[0 .. N/32), the
// reduction over the 32 lanes of columns (N / 32) * l + i.  Five exchange steps of N/2,
// N/4, ... independent shuffles (no serial chain through a reduction unit).
template <int N, class T, class Op>
__device__ __forceinline__ void warp_reduce_scatter(T (&v)[N], int lane, Op op) {
#pragma unroll
  for (int o = 16, n = N; o >= 1; o >>= 1, n >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const T send = up ? v[i] : v[n / 2 + i];
      const T keep = up ? v[n / 2 + i] : v[i];
      v[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
}

__global__ void __launch_bounds__(kGqThreads, 1) decode_attn_gqa_kernel(dq_attn_args args) {
  constexpr int RB = 8;  // bytes per 16-code row at 4 bits
  constexpr int X = kExcess<4>;
  extern __shared__ __align__(1024) unsigned char smem_gq[];
  GqSmem& sm = *reinterpret_cast<GqSmem*>(smem_gq);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- prologue: barriers, TMEM ----------------------------------------------------------
  if (tid == 0) {
    for (int s = 0; s < kGqStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kGqWide + 1);  // the widening warps + the MMA warp's commit
    }
    for (int s = 0; s < kSubRing; ++s) mbar_init(&sm.descfull[s], 1);
    mbar_init(&sm.g0bar, 1);
    for (int b = 0; b < kGqNumA; ++b) {
      mbar_init(&sm.afull[b], kGqWide);
      mbar_init(&sm.afree[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.yfull[b], 1);
      mbar_init(&sm.yfree[b], kGqWarps);
    }
    mbar_init(&sm.sfull, 1);
    mbar_init(&sm.pfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < kGqG * 8) {
    sm.pmax[tid] = 0u;
    sm.gsum[tid] = 0;
  }
  if (warp == kGqMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  if (warp == kGqProducer) {
    // ---- producer: descriptors and stages of this CTA's items, in order --------------------
    if (lane == 0) {
      // the W images come from the prepare kernel, and the ticket counter is shared with the
      // previous launch on these args: wait for both grids before the first copy
      asm volatile("griddepcontrol.wait;\n" ::: "memory");
      SubItem nd;
      bool have = (int)blockIdx.x < args.nwork;
      if (have) gq_load_sub(nd, args, blockIdx.x);
      int g = 0;
      for (int k = 0;; ++k) {
        const int ds = k % kSubRing;
        if (!have) {
          sm.sub[ds].nbt = 0;
          mbar_arrive(&sm.descfull[ds]);
          break;
        }
        const SubItem d = nd;
        sm.sub[ds] = d;
        mbar_arrive(&sm.descfull[ds]);
        bool nhave = false;
        for (int ls = 0; ls < d.stages; ++ls, ++g) {
          const int slot = g % kGqStages;
          if (g >= kGqStages) mbar_wait(&sm.empty[slot], (uint32_t)((g / kGqStages - 1) & 1));
          gq_issue_stage(sm, args, d, k, ls, sm.ring[slot], &sm.full[slot]);
          if (ls == min(2, d.stages - 1)) {
            const int nxt = (int)gridDim.x + atomicAdd(args.sched, 1);
            nhave = nxt < args.nwork;
            if (nhave) gq_load_sub(nd, args, nxt);
          }
        }
        have = nhave;
      }
      __threadfence();
      if (atomicAdd(args.sched + 1, 1) == (int)gridDim.x - 1) {
        args.sched[0] = 0;
        args.sched[1] = 0;
      }
    }
    return;
  }

  if (warp == kGqMma) {
    // ---- MMA warp: the whole (converged) warp runs the schedule with warp-uniform operands,
    // one elected lane issues each UMMA / commit (operands stay in uniform registers: no
    // per-UMMA register-to-uniform moves on the issue path)
    const bool leader = elect_one();
    const uint32_t id_k = tc_idesc(128, 128, 0, 1);  // codes u8 x W limbs s8
    const uint32_t id_v = tc_idesc(128, 128, 0, 0);  // codes u8 x P limbs u8
    const uint64_t pdesc = tc_sdesc(sm.pr.pb, 128, (kCB / 16) * 128);  // P: b chunks 128 B, (h, limb) groups 2 KB
    int na = 0;              // A-buffer uses = ring stages consumed
    int uy[2] = {0, 0};      // Y-buffer uses
    for (int j = 0;; ++j) {
      mbar_wait_spin(&sm.descfull[j % kSubRing], (uint32_t)((j / kSubRing) & 1));
      const int nbt = sm.sub[j % kSubRing].nbt, nK = sm.sub[j % kSubRing].nK, nV = sm.sub[j % kSubRing].nslices;
      if (nbt == 0) break;
      // S occupies the Y columns: the previous item's epilogue must have read both buffers
      for (int b = 0; b < 2; ++b)
        if (uy[b] > 0) mbar_wait_spin(&sm.yfree[b], (uint32_t)((uy[b] - 1) & 1));
      tc_fence_after();
      for (int ks = 0; ks < nK; ++ks, ++na) {
        const int ab = na % kGqNumA;
        mbar_wait_spin(&sm.afull[ab], (uint32_t)((na / kGqNumA) & 1));
        tc_fence_after();
        // this stage's W slice: N rows (h*2 + limb)*8 + a in 16 core-matrix groups 1 KB apart,
        // bond rows 128 B apart; k-step kk (2 bond rows) = +256 B = +16 in the address field
        const uint64_t bdesc = tc_sdesc(sm.ring[na % kGqStages] + 16384, 128, 1024);
        const uint32_t a0 = tmem + kGqColA + (uint32_t)(ab * 64);
        const uint32_t acc0 = ks ? 1u : 0u;
        if (leader) {
#ifndef DQ_GQ_NULL_MMA  // measurement only: no UMMAs (the commits still signal)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            tc_mma_ts(tmem + kGqColSY, a0 + kk * 8, bdesc + kk * 16, id_k, kk ? 1u : acc0);
            if (nbt > 2) tc_mma_ts(tmem + kGqColSY + 128, a0 + 32 + kk * 8, bdesc + kk * 16, id_k, kk ? 1u : acc0);
          }
#endif
          tc_commit(&sm.afree[ab]);
          tc_commit(&sm.empty[na % kGqStages]);  // the W slice has been read
        }
        __syncwarp();
      }
      if (leader) tc_commit(&sm.sfull);
      __syncwarp();
      mbar_wait_spin(&sm.pfull, (uint32_t)(j & 1));  // P limbs in shared memory, S read
      tc_fence_after();
#ifdef DQ_GQ_MMAWAIT  // measurement only: V phase of the MMA warp: span (slot 4) and A / Y waits (slot 6, 7)
      const int64_t v0 = global_ns();
      int64_t wa = 0, wy = 0;
#endif
      for (int vs = 0; vs < nV; ++vs, ++na) {
        const int ab = na % kGqNumA, yb = vs & 1;
#ifdef DQ_GQ_MMAWAIT
        int64_t w0 = global_ns();
        mbar_wait_spin(&sm.afull[ab], (uint32_t)((na / kGqNumA) & 1));
        wa += global_ns() - w0;
        w0 = global_ns();
        if (uy[yb] > 0) mbar_wait_spin(&sm.yfree[yb], (uint32_t)((uy[yb] - 1) & 1));
        wy += global_ns() - w0;
#else
        mbar_wait_spin(&sm.afull[ab], (uint32_t)((na / kGqNumA) & 1));
        if (uy[yb] > 0) mbar_wait_spin(&sm.yfree[yb], (uint32_t)((uy[yb] - 1) & 1));
#endif
        tc_fence_after();
        const uint32_t a0 = tmem + kGqColA + (uint32_t)(ab * 64), d0 = tmem + kGqColSY + (uint32_t)(yb * 128);
        if (leader) {
#ifndef DQ_GQ_NULL_MMA
          // 32 rows b per k-step: +256 B of P = +16 in the address field
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            if (kk < 2 * nbt) tc_mma_ts(d0, a0 + kk * 8, pdesc + kk * 16, id_v, kk ? 1u : 0u);
#endif
          tc_commit(&sm.afree[ab]);
          tc_commit(&sm.empty[na % kGqStages]);
          tc_commit(&sm.yfull[yb]);
        }
        __syncwarp();
        ++uy[yb];
      }
#ifdef DQ_GQ_MMAWAIT
      if (leader && args.trace) {
        const int it = sm.sub[j % kSubRing].item;
        args.trace[(size_t)it * 8 + 4] = global_ns() - v0;
        args.trace[(size_t)it * 8 + 6] = wa;
        args.trace[(size_t)it * 8 + 7] = wy;
      }
#endif
    }
    __syncwarp();
    named_sync2(kGqTmemUsers);  // the other warps' last TMEM accesses are done
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    return;
  }

  if (warp >= kGqWarps) {
    // ---- widening warpgroup: every K and V stage, in ring order, into the TMEM A buffers ----
    // (warp & 3 = its TMEM lane quadrant); it runs ahead of the math warps by up to 4 A buffers,
    // so the next item's first K stages are widened while the math warps fold this item's Y
    const int q = warp & 3;
    const int lane_in = 32 * q + lane;
    const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
    int st = 0, na = 0;
    for (int j = 0;; ++j) {
      mbar_wait(&sm.descfull[j % kSubRing], (uint32_t)((j / kSubRing) & 1));
      const SubItem d = sm.sub[j % kSubRing];
      if (d.nbt == 0) break;
      const int nbt = d.nbt, nmb = (nbt + 1) / 2;
      for (int ks = 0; ks < d.nK + d.nslices; ++ks, ++st, ++na) {
        const int slot = st % kGqStages, ab = na % kGqNumA;
        mbar_wait(&sm.full[slot], (uint32_t)((st / kGqStages) & 1));
        if (na >= kGqNumA) mbar_wait(&sm.afree[ab], (uint32_t)((na / kGqNumA - 1) & 1));
        if (ks < d.nK) {  // K stage: 8 bond rows of rows b = 128 mb + lane_in, both M-blocks
          for (int mb = 0; mb < nmb; ++mb) {
            const int jt = 2 * mb + (q >> 1), b_in = 32 * (q & 1) + lane;
            const unsigned char* tile = sm.ring[slot] + jt * 8 * kI2Pad * RB;
            const bool live = jt < nbt;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              uint32_t v[16];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int rl = 4 * half + i;  // rr & 3 = i (stages start at multiples of 8)
                uint2 w2 = make_uint2(0u, 0u);
                if (live) w2 = *reinterpret_cast<const uint2*>(tile + (rl * kI2Pad + (b_in ^ (i * 4))) * RB);
                v[4 * i] = w2.x & 0x0F0F0F0Fu;
                v[4 * i + 1] = (w2.x >> 4) & 0x0F0F0F0Fu;
                v[4 * i + 2] = w2.y & 0x0F0F0F0Fu;
                v[4 * i + 3] = (w2.y >> 4) & 0x0F0F0F0Fu;
              }
              tc_st16(tmem + lane_addr + kGqColA + (uint32_t)(ab * 64 + mb * 32 + half * 16), v);
            }
          }
        } else {  // V stage: row (r_local, e) = lane_in of every tile
          for (int t = 0; t < nbt; ++t) {
            const unsigned char* src = sm.ring[slot] + t * kGqVTileBytes + lane_in * 32;
            const uint4 c0 = *reinterpret_cast<const uint4*>(src);
            const uint4 c1 = *reinterpret_cast<const uint4*>(src + 16);
            const uint32_t wv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            uint32_t v[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              v[2 * k] = wv[k] & 0x0F0F0F0Fu;
              v[2 * k + 1] = (wv[k] >> 4) & 0x0F0F0F0Fu;
            }
            tc_st16(tmem + lane_addr + kGqColA + (uint32_t)(ab * 64 + t * 16), v);
          }
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&sm.afull[ab]);
          mbar_arrive(&sm.empty[slot]);
        }
      }
    }
    tc_fence_before();
    named_sync2(kGqTmemUsers);
    return;
  }

  // ---- consumer warps ----------------------------------------------------------------------
#ifdef DQ_GQ_SPIN  // measurement: consumers spin on their barriers instead of suspending
  auto cwait = [](uint64_t* bar, uint32_t parity) { mbar_wait_spin(bar, parity); };
#else
  auto cwait = [](uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); };
#endif
  const int q = warp & 3;                // TMEM lane quarter of this warp
  const int wg = warp >> 2;              // warpgroup 0..3
  const int mbk = wg & 1, hh = wg >> 1;  // K / softmax: M-block (rows b) and half (bond rows / heads 4hh..4hh+3)
  const int lane_in = 32 * q + lane;     // TMEM lane
  const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
  int uyc[2] = {0, 0};
  if (tid == 0) {
    // the combine may be scheduled once this grid's prerequisites (prepare kernel, producers of
    // q) have completed: it reads q and the tail before waiting for this grid
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  }

  for (int j = 0;; ++j) {
    cwait(&sm.descfull[j % kSubRing], (uint32_t)((j / kSubRing) & 1));
    const SubItem d = sm.sub[j % kSubRing];
    if (d.nbt == 0) break;
    const int wi = d.item, nbt = d.nbt, nmb = (nbt + 1) / 2;
    auto stamp = [&](int k) {
      if (args.trace && tid == 0) args.trace[(size_t)wi * 8 + k] = global_ns();
    };
    stamp(0);
    if (tid == 0) {  // G0v of this item (the previous item's epilogue ended in a barrier)
      const uint32_t gb = (uint32_t)(d.i1 * d.r * 32);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_expect_tx(&sm.g0bar, gb);
      bulk_g2s(sm.g0v, d.vg0, gb, &sm.g0bar);
    }

    // this thread's row b for the softmax: tile jt, row b_in inside it
    const int jt = 2 * mbk + (q >> 1);
    const int b_in = 32 * (q & 1) + lane;
    stamp(1);

    // ---- softmax of the item straight from S in TMEM (this thread = row b) -----------------
    cwait(&sm.sfull, (uint32_t)(j & 1));  // all K UMMAs done (the W metadata landed with stage 0)
    tc_fence_after();
#ifdef DQ_GQ_SMTRACE  // profiling build: softmax sub-phases in the MMA warp's trace slots
    stamp(7);
#endif
    const WMeta<kGqG>& wm = sm.wmeta[j & 1];
    // this thread: row b of M-block mbk, heads 4hh .. 4hh+3 (columns 32hh .. 32hh+31)
    const bool row_ok = mbk < nmb && jt < nbt && d.wb0 + jt * kI2Pad + b_in < d.i2;
    const float kscale = d.kscale * args.sm_scale * 1.4426950408889634f;
    float s[32];  // [hl * 8 + a], log2 domain
    if (mbk < nmb) {
      int acc[4][16];
#pragma unroll
      for (int hl = 0; hl < 4; ++hl)
        tc_ld16(tmem + lane_addr + kGqColSY + (uint32_t)(mbk * 128 + (4 * hh + hl) * 16), acc[hl]);
      tc_wait_ld();
#pragma unroll
      for (int hl = 0; hl < 4; ++hl)
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          const int h = 4 * hh + hl;
          const float v = (float)(256 * acc[hl][a] + acc[hl][8 + a] - wm.beta[h][a][0]) * (kscale * wm.cs[h][a][0]);
          s[hl * 8 + a] = row_ok ? v : -INFINITY;
        }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) s[i] = -INFINITY;
    }
    tc_fence_before();
    {  // row maxima per head over (a, b): per-thread over a, then a reduce-scatter (lane & 3 = head)
      float m4[4];
#pragma unroll
      for (int hl = 0; hl < 4; ++hl) {
        float m = s[hl * 8];
#pragma unroll
        for (int a = 1; a < 8; ++a) m = fmaxf(m, s[hl * 8 + a]);
        m4[hl] = m;
      }
#pragma unroll
      for (int o = 2, n = 4; o >= 1; o >>= 1, n >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
          const float send = up ? m4[i] : m4[n / 2 + i];
          const float keep = up ? m4[n / 2 + i] : m4[i];
          m4[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, o));
        }
      }
      float m = m4[0];
#pragma unroll
      for (int o = 4; o <= 16; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane < 4) sm.rowmax[hh][mbk * 4 + q][lane] = m;  // lane = head - 4hh
    }
    named_sync(kGqCons);
#ifdef DQ_GQ_SMTRACE
    stamp(4);
#endif
    float mh[4];
#pragma unroll
    for (int hl = 0; hl < 4; ++hl) {
      float m = sm.rowmax[hh][0][hl];
#pragma unroll
      for (int w = 1; w < 8; ++w) m = fmaxf(m, sm.rowmax[hh][w][hl]);
      mh[hl] = m;
    }
    // P = exp2(s - m_h) and the per-column maxima over the item's rows
#pragma unroll
    for (int i = 0; i < 32; ++i) s[i] = ex2(s[i] - mh[i / 8]);  // masked rows: ex2(-inf) = 0
    {
      unsigned t[32];  // P >= 0: float order = unsigned order of the bits
#pragma unroll
      for (int i = 0; i < 32; ++i) t[i] = __float_as_uint(s[i]);
      warp_reduce_scatter(t, lane, [](unsigned x, unsigned y) { return max(x, y); });
      atomicMax(&sm.pmax[32 * hh + lane], t[0]);
    }
    named_sync(kGqCons);
#ifdef DQ_GQ_SMTRACE
    stamp(6);
#endif
    // 15-bit fixed point per column; limbs hi (<= 128) and lo into the B operand of the V UMMAs
    {
      int pint[32];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        pint[i] = __float2int_rn(s[i] * pow2_sub_exp3<kGqPBits>(sm.pmax[32 * hh + i]));
      if (mbk < nmb && jt < nbt) {
        const int b_item = jt * kI2Pad + b_in;
        unsigned char* pcol = sm.pr.pb + (b_item >> 4) * 128 + inv_ord16<4>(b_item & 15);
#pragma unroll
        for (int hl = 0; hl < 4; ++hl)
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            const int h = 4 * hh + hl;
            pcol[((h * 2 + 0) * (kCB / 16)) * 128 + a * 16] = (unsigned char)(pint[hl * 8 + a] >> 8);
            pcol[((h * 2 + 1) * (kCB / 16)) * 128 + a * 16] = (unsigned char)(pint[hl * 8 + a] & 0xFF);
          }
      }
      warp_reduce_scatter(pint, lane, [](int x, int y) { return x + y; });
      atomicAdd(&sm.gsum[32 * hh + lane], pint[0]);
    }
    if (tid < kGqG * 8) sm.pinv[tid] = pow2_exp_sub(__uint_as_float(sm.pmax[tid]), kGqPBits);
    named_sync(kGqCons);  // gsum complete
    if (tid < kGqG * 8) sm.xoff[tid] = -(float)(X * sm.gsum[tid]) * sm.pinv[tid];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // P read by the tensor cores
    named_sync(kGqCons);
    if (tid == 0) mbar_arrive(&sm.pfull);
    stamp(2);

    // ---- V phase: widen stage vs, fold Y of stage vs - 1 while its UMMAs run ------------------
    float o[2][8];  // [head 2wg + hl][c] for e = lane_in & 15, summed over this thread's bond rows
#pragma unroll
    for (int hl = 0; hl < 2; ++hl)
#pragma unroll
      for (int c = 0; c < 8; ++c) o[hl][c] = 0.f;
    auto fold_y = [&](int vs) {
      const int yb = vs & 1;
      cwait(&sm.yfull[yb], (uint32_t)(uyc[yb] & 1));
      ++uyc[yb];
      tc_fence_after();
      float yf[2][8];
      {
        int y[2][16];
#ifndef DQ_GQ_NULL_YLD  // measurement only: no Y reads from TMEM
#pragma unroll
        for (int hl = 0; hl < 2; ++hl)
          tc_ld16(tmem + lane_addr + kGqColSY + (uint32_t)(yb * 128 + (2 * wg + hl) * 16), y[hl]);
        tc_wait_ld();
#else
#pragma unroll
        for (int hl = 0; hl < 2; ++hl)
#pragma unroll
          for (int k = 0; k < 16; ++k) y[hl][k] = lane + k;
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.yfree[yb]);
#pragma unroll
        for (int hl = 0; hl < 2; ++hl) {
          const int h = 2 * wg + hl;
          const float4 pi0 = *reinterpret_cast<const float4*>(&sm.pinv[h * 8]);
          const float4 pi1 = *reinterpret_cast<const float4*>(&sm.pinv[h * 8 + 4]);
          const float4 xo0 = *reinterpret_cast<const float4*>(&sm.xoff[h * 8]);
          const float4 xo1 = *reinterpret_cast<const float4*>(&sm.xoff[h * 8 + 4]);
          const float pi[8] = {pi0.x, pi0.y, pi0.z, pi0.w, pi1.x, pi1.y, pi1.z, pi1.w};
          const float xo[8] = {xo0.x, xo0.y, xo0.z, xo0.w, xo1.x, xo1.y, xo1.z, xo1.w};
          // (sum_b (code + X) Pint - X sum_b Pint) * 2^(e - 15): both limbs in one exact s32
#pragma unroll
          for (int a = 0; a < 8; ++a) yf[hl][a] = fmaf((float)(256 * y[hl][a] + y[hl][8 + a]), pi[a], xo[a]);
        }
      }
#ifdef DQ_GQ_NULL_FOLD  // measurement only: no G0v contraction
      o[0][0] += yf[0][0] + yf[1][7];
      return;
#endif
      // O[h, c, e] += sum_a G0v[a, c, r] Y[h, a, (r, e)] for this thread's (r, e)
      const int rr = 8 * vs + (lane_in >> 4);
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const float4 g_lo = sm.g0v[2 * (a * kMaxR + rr)], g_hi = sm.g0v[2 * (a * kMaxR + rr) + 1];
#pragma unroll
        for (int hl = 0; hl < 2; ++hl) {
          const float y = yf[hl][a];
          ffma2(o[hl][0], o[hl][1], g_lo.x, g_lo.y, y, y);
          ffma2(o[hl][2], o[hl][3], g_lo.z, g_lo.w, y, y);
          ffma2(o[hl][4], o[hl][5], g_hi.x, g_hi.y, y, y);
          ffma2(o[hl][6], o[hl][7], g_hi.z, g_hi.w, y, y);
        }
      }
    };
    cwait(&sm.g0bar, (uint32_t)(j & 1));
    // the widening warps feed the A buffers; Y is double-buffered, so stage vs + 1's UMMAs run
    // while this stage is folded
    for (int vs = 0; vs < d.nslices; ++vs) fold_y(vs);
    stamp(3);

    // ---- reduce over bond rows: lanes l / l ^ 16, then the 4 warps of the warpgroup ----------
#pragma unroll
    for (int hl = 0; hl < 2; ++hl)
#pragma unroll
      for (int c = 0; c < 8; ++c) o[hl][c] += __shfl_xor_sync(0xffffffffu, o[hl][c], 16);
    named_sync(kGqCons);  // every V UMMA has completed (yfull): P is dead
    if (lane < 16) {
#pragma unroll
      for (int hl = 0; hl < 2; ++hl)
#pragma unroll
        for (int c = 0; c < 8; ++c) sm.pr.red[q][2 * wg + hl][c * 16 + lane] = o[hl][c];
    }
    named_sync(kGqCons);
    for (int i = tid; i < kGqG * kD; i += kGqCons) {
      const int h = i / kD, dd = i % kD;
      const float v = sm.pr.red[0][h][dd] + sm.pr.red[1][h][dd] + sm.pr.red[2][h][dd] + sm.pr.red[3][h][dd];
      args.part_o[((size_t)d.part * kGqG + h) * kD + dd] = v * d.vscale;
    }
    if (q == 0 && mbk == 0 && lane < 4) {  // warps 0 / 8: heads 4hh .. 4hh+3
      const int h = 4 * hh + lane;
      float l = 0.f;
#pragma unroll
      for (int a = 0; a < 8; ++a) l += (float)sm.gsum[h * 8 + a] * sm.pinv[h * 8 + a];
      const float mv = lane == 0 ? mh[0] : lane == 1 ? mh[1] : lane == 2 ? mh[2] : mh[3];
      args.part_ml[((size_t)d.part * kGqG + h) * 2 + 0] = mv;  // log2 domain
      args.part_ml[((size_t)d.part * kGqG + h) * 2 + 1] = l;
    }
    named_sync(kGqCons);  // red, pmax, gsum, pinv, g0v reusable
    if (tid < kGqG * 8) {
      sm.pmax[tid] = 0u;
      sm.gsum[tid] = 0;
    }
    stamp(5);
  }
  tc_fence_before();
  named_sync2(kGqTmemUsers);  // with the widening and MMA warps: TMEM may be freed
}

}  // namespace attn
}  // namespace dq

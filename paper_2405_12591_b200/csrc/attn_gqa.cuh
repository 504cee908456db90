// tcgen05 split kernel for GQA groups of 8 query heads per kv head (path 2): 4-bit codes,
// full plans (i1 = 8, r = 64).  Same work items, persistent grid, ticket scheduler, producer
// warp and partials as paths 0 / 1; the contractions run on the 5th-generation tensor cores
// with all 8 heads, both fixed-point limbs and all 8 columns a in one N = 128 operand:
//
//   S[b, (h,l,a)]      = sum_{r,e} code_k[b, (r,e)] . W_l[(r,e), (h,a)]   M = 128 b, N = 128, K = (r,e)
//   Y[(r,e), (h,l,a)]  = sum_b code_v[(r,e), b] . P_l[b, (h,a)]          M = 128 (r,e), N = 128, K = b
//
// A operands (the codes) are widened from the shared-memory ring into tensor memory by the
// widening warps (tcgen05.st: lane = row, 4 K-bytes per column); B operands sit in shared
// memory as K-major core matrices: the W image streams through the ring in 16 KB slices of
// 8 bond rows next to the K codes of the same bond rows (so no 128 KB W buffer: the ring is
// 5 x 32 KB deep), P is written by the softmax.  One elected lane of the MMA warp issues
// every UMMA (kind::i8, s32 accumulators in TMEM) and signals through tcgen05.commit; its
// commit is also the ring slot's last release (the UMMAs read W from the slot).
//
// Per work item (<= 256 rows b = 2 M-blocks): 8 K stages (8 bond rows x all tiles + W slice)
// -> S in TMEM (2 x 128 columns) -> softmax from TMEM -> P limbs in shared memory -> 8 V
// stages (one M-block of 8 bond rows x all tiles each) -> Y per stage (128 columns) -> the
// epilogue folds Y with G0v on CUDA cores.  Items overlap: the ring carries item j+1's K
// stages next to item j's V stages, so the next S accumulates in its own columns while the
// math warps run item j's softmax and fold.  TMEM: 2 A buffers [0, 128), S [128, 384), Y
// [384, 512).  16 math warps (4 warpgroups: a warp reaches TMEM lanes 32 (warp % 4) ..):
// softmax by (M-block, head half), the Y fold by head pair; a widening warpgroup turns every
// ring stage into a TMEM A operand.
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
constexpr int kGqNumA = 2;                         // TMEM A buffers (64 columns each)
constexpr uint32_t kGqColA = 0, kGqColS = 128, kGqColY = 384;  // A: 2 x 64 columns; S: 2 x 128; Y: 128
#ifndef DQ_GQ_KA
#define DQ_GQ_KA 8
#endif
constexpr int kGqKA = DQ_GQ_KA;  // K stages of item j+1 ahead of item j's first V stage
constexpr int kGqPBits = 15;
#ifndef DQ_GQ_NAP
#define DQ_GQ_NAP 0  // 1: math warps wait with __nanosleep back-off; 2: + the widening warps
#endif
#ifndef DQ_GQ_NAP_NS
#define DQ_GQ_NAP_NS 64
#endif
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
  uint64_t afull[kGqNumA], afree[kGqNumA], sfull, sfree, pfull, yfull, yfree;
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

// Stage i of block j: nkn K stages of item j+1 (0 when there is none) and nv V stages of item
// j: the first min(kGqKA, nkn) K stages, then V and K alternately, then the rest.  Returns
// whether it is a K stage; idx = its index among the item's K (or V) stages.
__device__ __forceinline__ bool gq_block_stage(int i, int nkn, int nv, int& idx) {
  const int ka = min(kGqKA, nkn);
  if (i < ka) {
    idx = i;
    return true;
  }
  const int t = i - ka, m = min(nv, nkn - ka);
  if (t < 2 * m) {
    idx = (t & 1) ? ka + (t >> 1) : (t >> 1);
    return (t & 1) != 0;
  }
  const int u = t - 2 * m;
  if (nv > m) {
    idx = m + u;
    return false;
  }
  idx = ka + m + u;
  return true;
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

// wait with back-off: a non-blocking test, then __nanosleep between tests, so a waiting warp
// leaves the issue slots of its SM sub-partition to the warps that have work (a try_wait loop
// re-issues: ncu counts this kernel's wait loops at ~19% of its executed instructions)
template <int NS>
__device__ __forceinline__ void mbar_wait_nap(uint64_t* bar, uint32_t parity) {
  while (!mbar_test(bar, parity)) __nanosleep(NS);
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
    mbar_init(&sm.sfull, 1);
    mbar_init(&sm.sfree, kGqWarps);
    mbar_init(&sm.pfull, 1);
    mbar_init(&sm.yfull, 1);
    mbar_init(&sm.yfree, kGqWarps);
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

  // Stage order (producer, widening warps and MMA warp walk the same sequence): item 0's K
  // stages, then per item j one block of item j+1's K stages interleaved with item j's V stages
  // (gq_block_stage).  S has its own columns, so item j+1's K UMMAs run while the math warps
  // compute item j's softmax and fold its Y.

  if (warp == kGqProducer) {
    // ---- producer: descriptors and stages of this CTA's items, in sequence order ----------
    if (lane == 0) {
      // the W images come from the prepare kernel, and the ticket counter is shared with the
      // previous launch on these args: wait for both grids before the first copy
      asm volatile("griddepcontrol.wait;\n" ::: "memory");
      int g = 0;
      auto put = [&](int k, const SubItem* d) {
        const int ds = k % kSubRing;
        if (d) sm.sub[ds] = *d;
        else sm.sub[ds].nbt = 0;
        mbar_arrive(&sm.descfull[ds]);
      };
      auto ticket = [&](SubItem& nd) {
        const int nxt = (int)gridDim.x + atomicAdd(args.sched, 1);
        if (nxt >= args.nwork) return false;
        gq_load_sub(nd, args, nxt);
        return true;
      };
      auto issue = [&](const SubItem& d, int k, int st) {
        const int slot = g % kGqStages;
        if (g >= kGqStages) mbar_wait(&sm.empty[slot], (uint32_t)((g / kGqStages - 1) & 1));
        gq_issue_stage(sm, args, d, k, st, sm.ring[slot], &sm.full[slot]);
        ++g;
      };
      SubItem cur, nx, nn;
      if ((int)blockIdx.x >= args.nwork) {
        put(0, nullptr);
      } else {
        gq_load_sub(cur, args, blockIdx.x);
        put(0, &cur);
        bool hn = false;
        for (int ks = 0; ks < cur.nK; ++ks) {
          issue(cur, 0, ks);
          if (ks == min(2, cur.nK - 1)) hn = ticket(nx);
        }
        for (int j = 0;; ++j) {
          put(j + 1, hn ? &nx : nullptr);
          const int nkn = hn ? nx.nK : 0, n = nkn + cur.nslices;
          bool hnn = false;
          for (int i = 0; i < n; ++i) {
            int idx;
            if (gq_block_stage(i, nkn, cur.nslices, idx)) issue(nx, j + 1, idx);
            else issue(cur, j, cur.nK + idx);
            if (hn && i == min(2, n - 1)) hnn = ticket(nn);
          }
          if (!hn) break;
          cur = nx;
          nx = nn;
          hn = hnn;
        }
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
#ifdef DQ_GQ_MMA_SLEEP  // measurement: the MMA warp suspends in its waits instead of spinning
    auto mwait = [](uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); };
#else
    auto mwait = [](uint64_t* bar, uint32_t parity) { mbar_wait_spin(bar, parity); };
#endif
    const uint32_t id_k = tc_idesc(128, 128, 0, 1);  // codes u8 x W limbs s8
    const uint32_t id_v = tc_idesc(128, 128, 0, 0);  // codes u8 x P limbs u8
    const uint64_t pdesc = tc_sdesc(sm.pr.pb, 128, (kCB / 16) * 128);  // P: b chunks 128 B, (h, limb) groups 2 KB
    int na = 0;  // A-buffer uses = ring stages consumed
    int uy = 0;  // Y uses
    // K stage ks of an item of nbt tiles into S
    auto mma_k = [&](int nbt, int ks) {
      const int ab = na % kGqNumA;
      mwait(&sm.afull[ab], (uint32_t)((na / kGqNumA) & 1));
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
          tc_mma_ts(tmem + kGqColS, a0 + kk * 8, bdesc + kk * 16, id_k, kk ? 1u : acc0);
          if (nbt > 2) tc_mma_ts(tmem + kGqColS + 128, a0 + 32 + kk * 8, bdesc + kk * 16, id_k, kk ? 1u : acc0);
        }
#endif
        tc_commit(&sm.afree[ab]);
        tc_commit(&sm.empty[na % kGqStages]);  // the W slice has been read
      }
      __syncwarp();
      ++na;
    };
    // V stage of an item of nbt tiles into Y
#ifdef DQ_GQ_MMAWAIT  // measurement only: per item, V-phase span (slot 4), A waits (6), Y waits (7)
    int64_t tv0 = 0, wa = 0, wy = 0;
#define GQ_T0(x) const int64_t x = global_ns()
#define GQ_ACC(acc, x) acc += global_ns() - x
#else
#define GQ_T0(x)
#define GQ_ACC(acc, x)
#endif
    auto mma_v = [&](int nbt) {
      const int ab = na % kGqNumA;
      GQ_T0(t0);
      mwait(&sm.afull[ab], (uint32_t)((na / kGqNumA) & 1));
      GQ_ACC(wa, t0);
      GQ_T0(t1);
      if (uy > 0) mwait(&sm.yfree, (uint32_t)((uy - 1) & 1));
      GQ_ACC(wy, t1);
      tc_fence_after();
      const uint32_t a0 = tmem + kGqColA + (uint32_t)(ab * 64), d0 = tmem + kGqColY;
      if (leader) {
#ifndef DQ_GQ_NULL_MMA
        // 32 rows b per k-step: +256 B of P = +16 in the address field
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          if (kk < 2 * nbt) tc_mma_ts(d0, a0 + kk * 8, pdesc + kk * 16, id_v, kk ? 1u : 0u);
#endif
        tc_commit(&sm.afree[ab]);
        tc_commit(&sm.empty[na % kGqStages]);
        tc_commit(&sm.yfull);
      }
      __syncwarp();
      ++na;
      ++uy;
    };
    mwait(&sm.descfull[0], 0u);
    int nbt = sm.sub[0].nbt, nv = sm.sub[0].nslices;
    if (nbt > 0) {
      const int nk = sm.sub[0].nK;
      tc_fence_after();
      for (int ks = 0; ks < nk; ++ks) mma_k(nbt, ks);
      if (leader) tc_commit(&sm.sfull);
      __syncwarp();
      for (int j = 0;; ++j) {
        const int dn = (j + 1) % kSubRing;
        mwait(&sm.descfull[dn], (uint32_t)(((j + 1) / kSubRing) & 1));
        const int nbn = sm.sub[dn].nbt, nkn = nbn ? sm.sub[dn].nK : 0, nvn = sm.sub[dn].nslices;
        for (int i = 0; i < nkn + nv; ++i) {
          int idx;
          if (gq_block_stage(i, nkn, nv, idx)) {
            // S is rewritten: the math warps must have read item j's S
            if (idx == 0) mwait(&sm.sfree, (uint32_t)(j & 1));
            mma_k(nbn, idx);
            if (idx == nkn - 1) {
              if (leader) tc_commit(&sm.sfull);
              __syncwarp();
            }
          } else {
            if (idx == 0) mwait(&sm.pfull, (uint32_t)(j & 1));  // P limbs of item j
#ifdef DQ_GQ_MMAWAIT
            if (idx == 0) tv0 = global_ns(), wa = 0, wy = 0;
#endif
            mma_v(nbt);
          }
        }
#ifdef DQ_GQ_MMAWAIT
        if (leader && args.trace) {
          const int it = sm.sub[j % kSubRing].item;
          args.trace[(size_t)it * 8 + 4] = global_ns() - tv0;
          args.trace[(size_t)it * 8 + 6] = wa;
          args.trace[(size_t)it * 8 + 7] = wy;
        }
#endif
        if (!nbn) break;
        nbt = nbn;
        nv = nvn;
      }
    }
    __syncwarp();
    named_sync2(kGqTmemUsers);  // the other warps' last TMEM accesses are done
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    return;
  }

  if (warp >= kGqWarps) {
    // ---- widening warpgroup: every K and V stage, in sequence order, into the TMEM A buffers
    // (warp & 3 = its TMEM lane quadrant)
    const int q = warp & 3;
    const int lane_in = 32 * q + lane;
    const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
#if DQ_GQ_NAP >= 2  // measurement: the widening warps back off in their waits
    auto wwait = [](uint64_t* bar, uint32_t parity) { mbar_wait_nap<DQ_GQ_NAP_NS>(bar, parity); };
#else
    auto wwait = [](uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); };
#endif
    int st = 0;  // ring stages = A-buffer uses
#ifdef DQ_GQ_WIDETRACE  // measurement only: per item, V-stage widening span (slot 4), ring waits (6), A waits (7)
    int64_t tv0 = 0, tv1 = 0, wf = 0, wa = 0;
#endif
    auto widen = [&](int nbt, bool kstage) {
      const int slot = st % kGqStages, ab = st % kGqNumA;
#ifdef DQ_GQ_WIDETRACE
      const int64_t t0 = global_ns();
      if (!kstage && tv0 == 0) tv0 = t0;
#endif
      wwait(&sm.full[slot], (uint32_t)((st / kGqStages) & 1));
#ifdef DQ_GQ_WIDETRACE
      const int64_t t1 = global_ns();
      if (!kstage) wf += t1 - t0;
#endif
      if (st >= kGqNumA) wwait(&sm.afree[ab], (uint32_t)((st / kGqNumA - 1) & 1));
#ifdef DQ_GQ_WIDETRACE
      if (!kstage) wa += global_ns() - t1;
#endif
      // all of the stage's shared-memory reads first, then the nibble splits and TMEM stores
      // (a tcgen05.st is a memory barrier to the compiler: loads are not hoisted across it)
      if (kstage) {  // K stage: 8 bond rows of rows b = 128 mb + lane_in, both M-blocks
        const int b_in = 32 * (q & 1) + lane;
        uint2 w[2][8];
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {
          const int jt = 2 * mb + (q >> 1);
          const unsigned char* tile = sm.ring[slot] + jt * 8 * kI2Pad * RB;
#pragma unroll
          for (int rl = 0; rl < 8; ++rl) {  // rr & 3 = rl & 3 (stages start at multiples of 8)
            w[mb][rl] = make_uint2(0u, 0u);
            if (jt < nbt) w[mb][rl] = *reinterpret_cast<const uint2*>(tile + (rl * kI2Pad + (b_in ^ ((rl & 3) * 4))) * RB);
          }
        }
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {
          if (mb == 1 && nbt <= 2) break;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t v[16];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint2 w2 = w[mb][4 * half + i];
              v[4 * i] = w2.x & 0x0F0F0F0Fu;
              v[4 * i + 1] = (w2.x >> 4) & 0x0F0F0F0Fu;
              v[4 * i + 2] = w2.y & 0x0F0F0F0Fu;
              v[4 * i + 3] = (w2.y >> 4) & 0x0F0F0F0Fu;
            }
            tc_st16(tmem + lane_addr + kGqColA + (uint32_t)(ab * 64 + mb * 32 + half * 16), v);
          }
        }
      } else {  // V stage: row (r_local, e) = lane_in of every tile
        // rows are 32 B apart: lanes 4k .. 4k+3 read one half of their rows and lanes
        // 4k+4 .. 4k+7 the other, so each 16-byte load covers all 32 banks per 8 lanes (4
        // wavefronts per warp instead of 8); the halves are put back in order afterwards
        const int hs = (lane >> 2) & 1;
        uint4 c[4][2];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const unsigned char* src = sm.ring[slot] + t * kGqVTileBytes + lane_in * 32;
          uint4 x = make_uint4(0u, 0u, 0u, 0u), y = x;
          if (t < nbt) {
            x = *reinterpret_cast<const uint4*>(src + 16 * hs);
            y = *reinterpret_cast<const uint4*>(src + 16 * (hs ^ 1));
          }
          c[t][0] = hs ? y : x;
          c[t][1] = hs ? x : y;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (t >= nbt) break;
          const uint32_t wv[8] = {c[t][0].x, c[t][0].y, c[t][0].z, c[t][0].w,
                                  c[t][1].x, c[t][1].y, c[t][1].z, c[t][1].w};
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
      ++st;
#ifdef DQ_GQ_WIDETRACE
      if (!kstage) tv1 = global_ns();
#endif
    };
    mbar_wait(&sm.descfull[0], 0u);
    int nbt = sm.sub[0].nbt, nv = sm.sub[0].nslices;
    if (nbt > 0) {
      const int nk = sm.sub[0].nK;
      for (int ks = 0; ks < nk; ++ks) widen(nbt, true);
      for (int j = 0;; ++j) {
        const int dn = (j + 1) % kSubRing;
        mbar_wait(&sm.descfull[dn], (uint32_t)(((j + 1) / kSubRing) & 1));
        const int nbn = sm.sub[dn].nbt, nkn = nbn ? sm.sub[dn].nK : 0, nvn = sm.sub[dn].nslices;
        for (int i = 0; i < nkn + nv; ++i) {
          int idx;
          const bool kstage = gq_block_stage(i, nkn, nv, idx);
          widen(kstage ? nbn : nbt, kstage);
        }
#ifdef DQ_GQ_WIDETRACE
        if (warp == kGqWarps && lane == 0 && args.trace) {
          const int it = sm.sub[j % kSubRing].item;
          args.trace[(size_t)it * 8 + 4] = tv1 - tv0;
          args.trace[(size_t)it * 8 + 6] = wf;
          args.trace[(size_t)it * 8 + 7] = wa;
        }
        tv0 = wf = wa = 0;
#endif
        if (!nbn) break;
        nbt = nbn;
        nv = nvn;
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
#if DQ_GQ_NAP >= 1  // the math warps back off in their waits (mbar_wait_nap)
  auto cwait = [](uint64_t* bar, uint32_t parity) { mbar_wait_nap<DQ_GQ_NAP_NS>(bar, parity); };
#else
  auto cwait = [](uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); };
#endif
#endif
  const int q = warp & 3;                // TMEM lane quarter of this warp
  const int wg = warp >> 2;              // warpgroup 0..3
  const int mbk = wg & 1, hh = wg >> 1;  // K / softmax: M-block (rows b) and half (bond rows / heads 4hh..4hh+3)
  const int lane_in = 32 * q + lane;     // TMEM lane
  const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
  int uyc = 0;
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

    // ---- softmax of the item straight from S in TMEM (this thread = row b) -----------------
    cwait(&sm.sfull, (uint32_t)(j & 1));  // all K UMMAs done (the W metadata landed with stage 0)
    tc_fence_after();
    stamp(1);
    const WMeta<kGqG>& wm = sm.wmeta[j & 1];
    // this thread: row b of M-block mbk, heads 4hh .. 4hh+3 (columns 32hh .. 32hh+31)
    const bool row_ok = mbk < nmb && jt < nbt && d.wb0 + jt * kI2Pad + b_in < d.i2;
    const float kscale = d.kscale * args.sm_scale * 1.4426950408889634f;
    float s[32];  // [hl * 8 + a], log2 domain
    if (mbk < nmb) {
      int acc[4][16];
#pragma unroll
      for (int hl = 0; hl < 4; ++hl)
        tc_ld16(tmem + lane_addr + kGqColS + (uint32_t)(mbk * 128 + (4 * hh + hl) * 16), acc[hl]);
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.sfree);  // S read: the next item's K UMMAs may overwrite it
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
#ifdef DQ_GQ_SMTRACE  // profiling build: softmax sub-phases in the spare trace slots
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
      cwait(&sm.yfull, (uint32_t)(uyc & 1));
      ++uyc;
      tc_fence_after();
      float yf[2][8];
      {
        int y[2][16];
#ifndef DQ_GQ_NULL_YLD  // measurement only: no Y reads from TMEM
#pragma unroll
        for (int hl = 0; hl < 2; ++hl)
          tc_ld16(tmem + lane_addr + kGqColY + (uint32_t)((2 * wg + hl) * 16), y[hl]);
        tc_wait_ld();
#else
#pragma unroll
        for (int hl = 0; hl < 2; ++hl)
#pragma unroll
          for (int k = 0; k < 16; ++k) y[hl][k] = lane + k;
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.yfree);
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
    // Y is single-buffered: stage vs + 1's UMMAs wait for this stage's Y read (not its fold),
    // and the next item's K UMMAs fill the tensor pipe in between
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

// tcgen05 split kernel of the fused decode attention (path 1): int4 codes, g = 1, segments
// with the full plan (i1 = 8, r = 64).  Same work items, persistent grid, ticket scheduler,
// producer warp, W images and partials as attn_kernel.cuh (path 0); the two contractions
// run on the 5th-generation tensor cores instead of mma.sync:
//
//   S[b, a]      = sum_{r,e} code_k[b, (r,e)] . W[(r,e), a]     UMMA M=128 (b), N=8 (a), K=(r,e)
//   Y[(r,e), a] += sum_b code_v[(r,e), b] . P[b, a]             UMMA M=128 ((r,e)), N=8 (a), K=b
//
// The consumer warps stream the packed codes out of the shared-memory ring, widen them to
// u8 in registers and write them into tensor memory (tcgen05.st: lane = row, 4 K-bytes
// per column): A operands never touch shared memory twice.  B operands (the two-limb
// fixed-point W image and P) sit in shared memory as K-major core matrices.  One elected
// lane of a dedicated MMA warp issues tcgen05.mma.kind::i8 with s32 accumulators in TMEM
// and signals completion with tcgen05.commit on mbarriers.  Both TMEM A buffers and both
// Y buffers are double-buffered, so the consumers widen stage s+1 while stage s's MMAs run,
// and fold stage s's Y (exact s32 -> scaled fp32) into registers afterwards.
//
// Numerics: exact integer products of the excess-coded codes with 14-bit two-limb W (per
// column and bond-row group scale, both limbs signed so one N = 16 UMMA takes them) and
// 23-bit three-limb P (one scale per item: P = exp2(s - m) <= 1 in units of 2^-23).  Y is
// accumulated over the whole item in TMEM (s32 per limb) and folded once per item; the
// excess offset is removed exactly with sum_b P, accumulated alongside by a UMMA whose A
// operand is all ones.
#pragma once

#include "attn_kernel.cuh"

namespace dq {
namespace attn {

constexpr int kTcStages = 10;                        // 10 x 16 KB ring, one CTA per SM
constexpr int kTcWide = 8;                           // widening warpgroups (warps 8 .. 15)
constexpr int kTcProducer = kWarps + kTcWide;        // producer warp (12), then the MMA warp (13)
constexpr int kTcMma = kTcProducer + 1;
constexpr int kTcWarps = kWarps + kTcWide + 2;
constexpr int kTcTmemUsers = (kWarps + kTcWide + 1) * 32;  // threads that touch TMEM (final barrier)
constexpr int kTcThreads = kTcWarps * 32;
constexpr int kTmemCols = 512;
// TMEM column map: 2 A buffers of 64 columns, S (64), Y (8 M-blocks x 32: P limbs hi / mid /
// lo / zero), a constant all-ones A operand (8 columns = K 32) and sum_b P (32)
constexpr int kNumA = 2;
constexpr uint32_t kColA = 0, kColS = 64 * kNumA, kColY = kColS + 64, kColOnes = kColY + 256, kColPsum = 480;
constexpr int kPLimbs = 4;  // P limb groups of the V B operand (N = 32): hi, mid, lo, zero

__device__ __forceinline__ uint32_t tc_idesc(int M, int N, int a_signed, int b_signed) {
  return (2u << 4) | ((uint32_t)a_signed << 7) | ((uint32_t)b_signed << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// K-major, no-swizzle shared-memory matrix descriptor (core matrices of 8 rows x 16 bytes)
__device__ __forceinline__ uint64_t tc_sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;
}

// D[tmem] (+)= A[tmem] . B[smem]
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tc_ld8(uint32_t taddr, int (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
}

__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// stage geometry of path 1: K stages of RK bond rows over all tiles of the item, with
// RK * 4 columns per 128-row M-block (<= 64 columns per A buffer); V stages of 32 bond rows
// of one tile (512 (r,e) rows = 4 M-blocks x 16 columns)
__device__ __forceinline__ void tc_geometry(SubItem& d) {
  const int nmb = (d.nbt + 1) / 2;
  int RK = (kStageBytes / (d.nbt * kI2Pad * 8)) & ~3;
  RK = min(RK, nmb == 2 ? 8 : 16);
  d.RK = RK;
  d.nK = (d.r + RK - 1) / RK;
  d.RV = 32;
  d.nslices = 2;
  d.stages = d.nK + d.nbt * d.nslices;
}

__device__ __forceinline__ void tc_load_sub(SubItem& d, const dq_attn_args& a, int w) {
  load_sub<4>(d, a, w);
  tc_geometry(d);
}

struct TcSmem {
  alignas(1024) unsigned char ring[kTcStages][kStageBytes];
  alignas(16) uint4 w[2 * kMaxR * 8];     // W limbs, chunk (limb * r + rr) * 8 + a (path-1 image)
  alignas(16) float4 g0v[8 * kMaxR * 2];  // fp32 G0v [a][rr][c]
  alignas(128) unsigned char pb[kPLimbs][kTiles * 4 * 128];  // P limbs: K-major core matrices, chunk b/16
  float red[kWarps][kD];
  alignas(16) WMeta<1> wmeta;
  SubItem sub[kSubRing];
  uint64_t full[kTcStages], empty[kTcStages];
  uint64_t wbar, g0bar, descfull[kSubRing];
  uint64_t afull[kNumA], afree[kNumA], sfull, sfree, pfull, vdone, yfree;
  float rowmax[kWarps];
  float lsum[kWarps];
  uint32_t tmem;
};

// the W image (path-1 limb chunks + metadata) of an item's segment onto wbar (one thread)
__device__ __forceinline__ void issue_wimg_tc(TcSmem& sm, const dq_attn_args& a, const SubItem& d) {
  const unsigned char* img = static_cast<const unsigned char*>(a.wimg) + (size_t)d.seg * a.wimg_stride;
  const uint32_t wb = (uint32_t)(2 * d.r * 8 * 16);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  mbar_expect_tx(&sm.wbar, wb + (uint32_t)sizeof(WMeta<1>));
  bulk_g2s(sm.w, img, wb, &sm.wbar);
  bulk_g2s(&sm.wmeta, img + kWChunkBytes<1>, (uint32_t)sizeof(WMeta<1>), &sm.wbar);
}

__global__ void __launch_bounds__(kTcThreads, 1) decode_attn_tc_kernel(dq_attn_args args) {
  constexpr int RB = 8;      // bytes per 16-code row at 4 bits
  constexpr int X = kExcess<4>;
  extern __shared__ __align__(1024) unsigned char smem_tc[];
  TcSmem& sm = *reinterpret_cast<TcSmem*>(smem_tc);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- prologue: barriers, TMEM ----------------------------------------------------------
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kTcWide);
    }
    for (int s = 0; s < kSubRing; ++s) mbar_init(&sm.descfull[s], 1);
    mbar_init(&sm.wbar, 1);
    mbar_init(&sm.g0bar, 1);
    for (int b = 0; b < kNumA; ++b) {
      mbar_init(&sm.afull[b], kTcWide);
      mbar_init(&sm.afree[b], 1);
    }
    mbar_init(&sm.sfull, 1);
    mbar_init(&sm.sfree, kWarps);
    mbar_init(&sm.pfull, 1);
    mbar_init(&sm.vdone, 1);
    mbar_init(&sm.yfree, kWarps);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == kTcMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < (int)sizeof(sm.pb[3]) / 4; i += kTcThreads) reinterpret_cast<int*>(sm.pb[3])[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  if (warp == kTcProducer) {
    // ---- producer: descriptors and code stages of this CTA's items (as path 0) -------------
    if (lane == 0) {
      SubItem nd;
      bool have = (int)blockIdx.x < args.nwork;
      if (have) tc_load_sub(nd, args, blockIdx.x);
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
          const int slot = g % kTcStages;
          if (g >= kTcStages) mbar_wait(&sm.empty[slot], (uint32_t)((g / kTcStages - 1) & 1));
          issue_stage<4>(issue_of(d), ls, sm.ring[slot], &sm.full[slot]);
          if (ls == min(2, d.stages - 1)) {
            // the ticket counter is shared with the previous launch on these args: under
            // programmatic dependent launch, wait for that grid before drawing from it
            if (k == 0) asm volatile("griddepcontrol.wait;\n" ::: "memory");
            const int nxt = (int)gridDim.x + atomicAdd(args.sched, 1);
            nhave = nxt < args.nwork;
            if (nhave) tc_load_sub(nd, args, nxt);
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

  if (warp == kTcMma) {
    // ---- MMA warp: the whole (converged) warp runs the schedule with warp-uniform operands;
    // one elected lane issues each UMMA / commit (operands stay in uniform registers)
    uint32_t lead;
    asm volatile("{\n.reg .pred P;\n.reg .b32 r;\nelect.sync r|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}" : "=r"(lead));
    const bool leader = lead != 0;
    // both limbs of a B operand in one UMMA: N = 16 rows (hi limb a = 0..7, lo limb a = 0..7)
    const uint32_t id_k = tc_idesc(128, 16, 0, 1);  // codes u8 x W limbs s8
    const uint32_t id_v = tc_idesc(128, 32, 0, 0);  // codes u8 x P limbs u8 (hi, mid, lo, 0)
    int na = 0;  // A-buffer uses
    for (int j = 0;; ++j) {
      mbar_wait_spin(&sm.descfull[j % kSubRing], (uint32_t)((j / kSubRing) & 1));
      const int nbt = sm.sub[j % kSubRing].nbt, nK = sm.sub[j % kSubRing].nK, RK = sm.sub[j % kSubRing].RK;
      const int r = sm.sub[j % kSubRing].r;
      if (nbt == 0) break;
      const int nmb = (nbt + 1) / 2;
      mbar_wait_spin(&sm.wbar, (uint32_t)(j & 1));        // W image of this item's segment
      if (j > 0) mbar_wait_spin(&sm.sfree, (uint32_t)((j - 1) & 1));  // S of the previous item read
      for (int ks = 0; ks < nK; ++ks, ++na) {
        const int ab = na % kNumA;
        mbar_wait_spin(&sm.afull[ab], (uint32_t)((na / kNumA) & 1));
        tc_fence_after();
        const int rk0 = ks * RK, nr = min(RK, r - rk0);
        // rows 0-7: hi limb chunk of bond row rr, rows 8-15: lo limb (r * 128 bytes further);
        // k-step kk (2 bond rows) = +256 B = +16 in the address field
        const uint64_t bdesc = tc_sdesc(&sm.w[rk0 * 8], 128, r * 128);
        const uint32_t acol = tmem + kColA + (uint32_t)(ab * 64);
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {  // UMMA k-step = 32 bytes = 2 bond rows
            if (kk < nr / 2) {
              const int rr = rk0 + 2 * kk;
              const uint32_t grp = rr < kGroupR ? 0u : 1u;
              const uint32_t acc = (rr != 0 && rr != kGroupR) ? 1u : 0u;  // each group's first bond rows reset S
              tc_mma_ts(tmem + kColS + grp * 32, acol + kk * 8, bdesc + kk * 16, id_k, acc);
              if (nmb == 2) tc_mma_ts(tmem + kColS + grp * 32 + 16, acol + RK * 4 + kk * 8, bdesc + kk * 16, id_k, acc);
            }
          }
          tc_commit(&sm.afree[ab]);
        }
        __syncwarp();
      }
      if (leader) tc_commit(&sm.sfull);
      __syncwarp();
      mbar_wait_spin(&sm.pfull, (uint32_t)(j & 1));  // P limbs of this item in shared memory
      if (j > 0) mbar_wait_spin(&sm.yfree, (uint32_t)((j - 1) & 1));  // Y / sum P of the previous item read
      tc_fence_after();
      const uint64_t pdesc = tc_sdesc(&sm.pb[0][0], 128, sizeof(sm.pb[0]));
      for (int t = 0; t < nbt; ++t)
        for (int sl = 0; sl < 2; ++sl, ++na) {
          const int ab = na % kNumA;
          mbar_wait_spin(&sm.afull[ab], (uint32_t)((na / kNumA) & 1));
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {  // 64 b = 2 k-steps
              // B rows: 0-7 P hi limb, 8-15 mid, 16-23 lo, 24-31 zero (the next limb buffers);
              // +256 B per k-step = +16 in the address field
              const uint64_t bdesc = pdesc + (uint64_t)((t * 4 + kk * 2) * 8);
              const uint32_t acc = (t > 0 || kk > 0) ? 1u : 0u;
#pragma unroll
              for (int mb = 0; mb < 4; ++mb)
                tc_mma_ts(tmem + kColY + (uint32_t)((sl * 4 + mb) * 32), tmem + kColA + (uint32_t)(ab * 64 + mb * 16 + kk * 8),
                          bdesc, id_v, acc);
              if (sl == 0) tc_mma_ts(tmem + kColPsum, tmem + kColOnes, bdesc, id_v, acc);  // sum_b P
            }
            tc_commit(&sm.afree[ab]);
          }
          __syncwarp();
        }
      if (leader) tc_commit(&sm.vdone);
      __syncwarp();
    }
    // wait for the other warps' last TMEM accesses, then free TMEM
    __syncwarp();
    named_sync2(kTcTmemUsers);
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    return;
  }

  if (warp >= kWarps) {
    // ---- widening warpgroup: every K and V stage, in ring order, into the TMEM A buffers ----
    // (warp & 3 = its TMEM lane quadrant).  S and Y have their own TMEM columns, so it runs
    // ahead into the next item's K stages while the consumer warps do this item's softmax and
    // fold.
    const int q = warp & 3;
    const int wwg = (warp - kWarps) >> 2;  // K: M-block wwg; V: M-blocks 2 wwg, 2 wwg + 1
    const int lane_in = 32 * q + lane;
    const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
    const int swz = (16 / 4);  // ktile swizzle unit at 4 bits: (rr & 3) * 4
    int st = 0, na = 0;
    for (int j = 0;; ++j) {
      mbar_wait(&sm.descfull[j % kSubRing], (uint32_t)((j / kSubRing) & 1));
      const SubItem d = sm.sub[j % kSubRing];
      if (d.nbt == 0) break;
      const int nbt = d.nbt, nmb = (nbt + 1) / 2, r = d.r;
      for (int ks = 0; ks < d.stages; ++ks, ++st, ++na) {
        const int slot = st % kTcStages, ab = na % kNumA;
        mbar_wait(&sm.full[slot], (uint32_t)((st / kTcStages) & 1));
        if (na >= kNumA) mbar_wait(&sm.afree[ab], (uint32_t)((na / kNumA - 1) & 1));
        if (ks < d.nK) {  // K stage: RK bond rows of rows b = 128 mb + lane_in of each M-block
          const int rk0 = ks * d.RK, nr = min(d.RK, r - rk0);
          for (int mb = wwg; mb < nmb; mb += 2) {
            const int jt = 2 * mb + (q >> 1), b_in = 32 * (q & 1) + lane;
            const unsigned char* tile = sm.ring[slot] + jt * nr * kI2Pad * RB;
            const bool live = jt < nbt;
            for (int r4 = 0; r4 < nr; r4 += 4) {
              uint32_t v[16];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int rl = r4 + i, rr = rk0 + rl;
                uint32_t o[4] = {0, 0, 0, 0};
                if (live) {
                  const uint2 w2 = *reinterpret_cast<const uint2*>(tile + (rl * kI2Pad + (b_in ^ ((rr & 3) * swz))) * RB);
                  o[0] = w2.x & 0x0F0F0F0Fu;
                  o[1] = (w2.x >> 4) & 0x0F0F0F0Fu;
                  o[2] = w2.y & 0x0F0F0F0Fu;
                  o[3] = (w2.y >> 4) & 0x0F0F0F0Fu;
                }
                v[4 * i] = o[0], v[4 * i + 1] = o[1], v[4 * i + 2] = o[2], v[4 * i + 3] = o[3];
              }
              tc_st16(tmem + lane_addr + kColA + (uint32_t)(ab * 64 + mb * d.RK * 4 + r4 * 4), v);
            }
          }
        } else {  // V stage (tile, 32-bond-row slice): rows (r_local * 16 + e) = 128 mb4 + lane_in
          const unsigned char* buf = sm.ring[slot];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int mb4 = 2 * wwg + i;
            const int rho = mb4 * 128 + lane_in;
            const uint4 c0 = *reinterpret_cast<const uint4*>(buf + rho * 32);
            const uint4 c1 = *reinterpret_cast<const uint4*>(buf + rho * 32 + 16);
            const uint32_t wv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            uint32_t v[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              v[2 * k] = wv[k] & 0x0F0F0F0Fu;
              v[2 * k + 1] = (wv[k] >> 4) & 0x0F0F0F0Fu;
            }
            tc_st16(tmem + lane_addr + kColA + (uint32_t)(ab * 64 + mb4 * 16), v);
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
    named_sync2(kTcTmemUsers);
    return;
  }

  // ---- consumer warps ----------------------------------------------------------------------
  const int q = warp & 3;              // TMEM lane quarter of this warp
  const int half = warp >> 2;          // K phase: M-block; V phase: M-blocks 2*half, 2*half+1
  const int lane_in = 32 * q + lane;   // TMEM lane (row inside an M-block)
  const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
  if (warp < 4) {  // the constant all-ones A operand (K = 32 bytes of 1) used to sum P
    uint32_t ones[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) ones[i] = 0x01010101u;
    tc_st16(tmem + lane_addr + kColOnes, ones);  // 16 columns: the 8 used + 8 spare
    tc_wait_st();
  }
  if (tid == 0) {
    mbar_wait(&sm.descfull[0], 0);
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // the combine may be scheduled
    if (sm.sub[0].nbt > 0) issue_wimg_tc(sm, args, sm.sub[0]);
  }

  for (int j = 0;; ++j) {
    mbar_wait(&sm.descfull[j % kSubRing], (uint32_t)((j / kSubRing) & 1));
    const SubItem d = sm.sub[j % kSubRing];
    if (d.nbt == 0) break;
    const int wi = d.item, nbt = d.nbt, nmb = (nbt + 1) / 2, r = d.r;
    auto stamp = [&](int k) {
      if (args.trace && tid == 0) args.trace[(size_t)wi * 8 + k] = global_ns();
    };
    stamp(0);

    if (tid == 0) {  // G0v of this item (its buffer is free: the previous epilogue ended in a barrier)
      const uint32_t gb = (uint32_t)(d.i1 * r * 32);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_expect_tx(&sm.g0bar, gb);
      bulk_g2s(sm.g0v, d.vg0, gb, &sm.g0bar);
    }

    // this thread's row b: tile jt, row b_in inside it (the widening warps fill the A buffers)
    const int jt = 2 * half + (q >> 1);
    const int b_in = 32 * (q & 1) + lane;
    stamp(1);

    // ---- S from TMEM, softmax of the item -----------------------------------------------------
    mbar_wait(&sm.wbar, (uint32_t)(j & 1));  // W metadata (beta, cs)
    mbar_wait(&sm.sfull, (uint32_t)(j & 1));
    tc_fence_after();
    float s[8];
    {
      int acc[2][2][8];
      if (half < nmb) {
#pragma unroll
        for (int g2 = 0; g2 < 2; ++g2)
#pragma unroll
          for (int limb = 0; limb < 2; ++limb)
            tc_ld8(tmem + lane_addr + kColS + (uint32_t)((g2 * 2 + half) * 16 + limb * 8), acc[g2][limb]);
        tc_wait_ld();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.sfree);
      const float kscale = d.kscale * args.sm_scale * 1.4426950408889634f;
      const bool row_ok = half < nmb && jt < nbt && d.wb0 + jt * kI2Pad + b_in < d.i2;
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        float v = 0.f;
#pragma unroll
        for (int g2 = 0; g2 < (kGroupR < kMaxR ? 2 : 1); ++g2)
          v += (float)(256 * acc[g2][0][a] + acc[g2][1][a] - sm.wmeta.beta[0][a][g2]) * (kscale * sm.wmeta.cs[0][a][g2]);
        s[a] = (row_ok && a < d.i1) ? v : -INFINITY;
      }
    }
    float m = s[0];
#pragma unroll
    for (int a = 1; a < 8; ++a) m = fmaxf(m, s[a]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) sm.rowmax[warp] = m;
    named_sync(kThreads);
    // every thread has combined its S with the W metadata, and every UMMA reading W
    // completed before sfull: W(j+1) may replace W(j)
    if (tid == 0) {
      const int jn = j + 1;
      mbar_wait(&sm.descfull[jn % kSubRing], (uint32_t)((jn / kSubRing) & 1));
      if (sm.sub[jn % kSubRing].nbt > 0) issue_wimg_tc(sm, args, sm.sub[jn % kSubRing]);
    }
    m = sm.rowmax[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) m = fmaxf(m, sm.rowmax[w]);
    float lsum = 0.f;
    {
      // P = exp2(s - m) <= 1 as a 23-bit integer, three 8-bit limbs (hi <= 128)
      const int b_item = jt * kI2Pad + b_in;
      const int pos = (b_item >> 4) * 128 + inv_ord16<4>(b_item & 15);
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int pint = s[a] == -INFINITY ? 0 : __float2int_rn(exp2f(s[a] - m) * 8388608.f);
        lsum += (float)pint;
        if (half < nmb) {
          sm.pb[0][pos + a * 16] = (unsigned char)(pint >> 16);
          sm.pb[1][pos + a * 16] = (unsigned char)((pint >> 8) & 0xFF);
          sm.pb[2][pos + a * 16] = (unsigned char)(pint & 0xFF);
        }
      }
      lsum *= 1.f / 8388608.f;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // P read by the tensor cores
    named_sync(kThreads);
    if (tid == 0) mbar_arrive(&sm.pfull);
    stamp(2);

    // Y (thread rows: slice sl, M-block 2*half + i: (r, e) = (32 sl + 8 (2 half + i) + lane_in / 16,
    // lane_in % 16)) and sum_b P, once per item
    mbar_wait(&sm.vdone, (uint32_t)(j & 1));
    tc_fence_after();
    float accv[2][2][8];
    {
      int ps[3][8];
#pragma unroll
      for (int l = 0; l < 3; ++l) tc_ld8(tmem + lane_addr + kColPsum + (uint32_t)(l * 8), ps[l]);
#pragma unroll
      for (int sl = 0; sl < 2; ++sl)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          int y[3][8];
#pragma unroll
          for (int l = 0; l < 3; ++l)
            tc_ld8(tmem + lane_addr + kColY + (uint32_t)((sl * 4 + 2 * half + i) * 32 + l * 8), y[l]);
          tc_wait_ld();
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            // sum_b (code + X) P - X sum_b P, per limb exact in s32, then 2^16 / 2^8 / 1 in fp32
            const float hi = (float)(y[0][a] - X * ps[0][a]), mid = (float)(y[1][a] - X * ps[1][a]);
            const float lo = (float)(y[2][a] - X * ps[2][a]);
            accv[sl][i][a] = fmaf(fmaf(hi, 256.f, mid), 256.f, lo) * (1.f / 8388608.f);
          }
        }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.yfree);
    stamp(3);

    // ---- epilogue: O[c, e] = scale_v * sum_{a, r} G0v[a, c, r] Y[(r, e), a] ---------------------
    mbar_wait(&sm.g0bar, (uint32_t)(j & 1));
    float part[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // [c] for e = lane_in % 16
#pragma unroll
    for (int sl = 0; sl < 2; ++sl)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int rr = 32 * sl + 8 * (2 * half + i) + lane_in / 16;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          const float4 g_lo = sm.g0v[2 * (a * r + rr)], g_hi = sm.g0v[2 * (a * r + rr) + 1];
          const float y = accv[sl][i][a];
          ffma2(part[0], part[1], g_lo.x, g_lo.y, y, y);
          ffma2(part[2], part[3], g_lo.z, g_lo.w, y, y);
          ffma2(part[4], part[5], g_hi.x, g_hi.y, y, y);
          ffma2(part[6], part[7], g_hi.z, g_hi.w, y, y);
        }
      }
    // lanes l and l + 16 hold the same e
#pragma unroll
    for (int c = 0; c < 8; ++c) part[c] += __shfl_xor_sync(0xffffffffu, part[c], 16);
    for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane < 16) {
#pragma unroll
      for (int c = 0; c < 8; ++c) sm.red[warp][c * 16 + lane] = part[c];
    }
    if (lane == 0) sm.lsum[warp] = lsum;
    named_sync(kThreads);
    if (tid < kD) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) v += sm.red[w][tid];
      args.part_o[(size_t)d.part * kD + tid] = v * d.vscale;
    }
    if (tid == 0) {
      float l = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) l += sm.lsum[w];
      args.part_ml[(size_t)d.part * 2 + 0] = m;  // log2 domain
      args.part_ml[(size_t)d.part * 2 + 1] = l;
    }
    named_sync(kThreads);  // red / lsum / g0v / pmax reusable
    stamp(5);
  }
  tc_fence_before();
  named_sync2(kTcTmemUsers);  // with the widening and MMA warps: TMEM may be freed
}

}  // namespace attn
}  // namespace dq

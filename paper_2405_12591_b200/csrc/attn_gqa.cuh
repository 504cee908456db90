// tcgen05 split kernel for GQA groups of 8 query heads per kv head (path 2): 4-bit codes,
// full plans (i1 = 8, r = 64).  Same work items, persistent grid, ticket scheduler, producer
// warp and partials as paths 0 / 1; the contractions run on the 5th-generation tensor cores
// with all 8 heads, both fixed-point limbs and all 8 columns a in one N = 128 operand:
//
//   S[b, (h,l,a)]      = sum_{r,e} code_k[b, (r,e)] . W_l[(r,e), (h,a)]   M = 128 b, N = 128, K = (r,e)
//   Y[(r,e), (h,l,a)]  = sum_b code_v[(r,e), b] . P_l[b, (h,a)]          M = 128 (r,e), N = 128, K = b
//
// A operands (the codes) are widened from the shared-memory ring into tensor memory by the
// consumer warps (tcgen05.st: lane = row, 4 K-bytes per column); B operands (W image, P)
// sit in shared memory as K-major core matrices.  One elected lane of the MMA warp issues
// every UMMA (kind::i8, s32 accumulators in TMEM) and signals through tcgen05.commit.
//
// Per work item (<= 256 rows b = 2 M-blocks): 8 K stages (8 bond rows x all tiles) -> S in
// TMEM (2 x 128 columns) -> softmax from TMEM -> P limbs in shared memory -> 8 V stages (one
// M-block of 8 bond rows x all tiles each) -> Y per stage (128 columns, double-buffered in
// the S columns) -> the epilogue folds Y with G0v on CUDA cores while the next stage's
// UMMAs run.  TMEM: A buffers [0, 128), S / Y [128, 384).
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
constexpr int kGqStages = 3;                       // ring: 3 x 16 KB (W image 128 KB + P 32 KB)
constexpr int kGqWarps = 8;                        // consumer warps: 2 warpgroups
constexpr int kGqCons = kGqWarps * 32;
constexpr int kGqThreads = kGqCons + 64;           // + producer (8) + MMA (9)
constexpr uint32_t kGqColA = 0, kGqColSY = 128;    // A: 2 x 64 columns; S / Y: 2 x 128 columns
constexpr int kGqPBits = 15;
constexpr int kGqVTileBytes = 8 * 16 * kI2Pad / 2;  // V stage per tile: 8 bond rows x 16 e x 64 b

struct GqSmem {
  alignas(1024) unsigned char ring[kGqStages][kStageBytes];
  alignas(128) uint4 w[kGqG * 2 * kMaxR * 8];      // W limbs: chunk ((h*2 + limb)*r + rr)*8 + a
  alignas(16) WMeta<kGqG> wmeta;                   // beta, cs per (h, a) (group 0)
  // P limbs as core matrices [(h*2 + limb)][b / 16][a][16 b]; the epilogue's cross-warp
  // reduction reuses the buffer once every V UMMA of the item has completed
  union alignas(128) {
    unsigned char pb[kGqG * 2 * (kCB / 16) * 128];
    float red[4][kGqG][kD];
  } pr;
  alignas(16) float4 g0v[8 * kMaxR * 2];           // fp32 G0v [a][rr][c]
  alignas(16) float pinv[kGqG][8];                 // 2^(e - 15) of the P column maxima
  unsigned pmax[kGqG][8];
  int gsum[kGqG][8];
  float rowmax[kGqG][kGqWarps];
  SubItem sub[kSubRing];
  uint64_t full[kGqStages], empty[kGqStages];
  uint64_t wbar, wfree, g0bar, descfull[kSubRing];
  uint64_t afull[2], afree[2], sfull, pfull, yfull[2], yfree[2];
  uint32_t tmem;
};
static_assert(sizeof(GqSmem) <= 232448, "path-2 shared memory exceeds the 227 KB opt-in limit");

// stage geometry of path 2: K stages as path 1 (RK bond rows x all tiles); V stages of 8 bond
// rows (one M-block of (r, e)) x all tiles
__device__ __forceinline__ void gq_load_sub(SubItem& d, const dq_attn_args& a, int w) {
  load_sub<4>(d, a, w);
  const int nmb = (d.nbt + 1) / 2;
  int RK = (kStageBytes / (d.nbt * kI2Pad * 8)) & ~3;
  RK = min(RK, nmb == 2 ? 8 : 16);
  d.RK = RK;
  d.nK = (d.r + RK - 1) / RK;
  d.RV = 8;
  d.nslices = d.r / 8;
  d.stages = d.nK + d.nslices;
}

__device__ __forceinline__ void gq_issue_stage(const SubItem& d, int st, unsigned char* buf, uint64_t* bar) {
  if (st < d.nK) {
    issue_stage<4>(d, st, buf, bar);
    return;
  }
  const int mbv = st - d.nK;
  const int bt0 = d.wb0 / kI2Pad;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  mbar_expect_tx(bar, (uint32_t)(kGqVTileBytes * d.nbt));
  for (int t = 0; t < d.nbt; ++t) {
    const unsigned char* src = d.vc + ((size_t)(bt0 + t) * d.r + 8 * mbv) * 16 * kI2Pad / 2;
    bulk_g2s(buf + t * kGqVTileBytes, src, (uint32_t)kGqVTileBytes, bar);
  }
}

__device__ __forceinline__ void gq_issue_wimg(GqSmem& sm, const dq_attn_args& a, const SubItem& d) {
  const unsigned char* img = static_cast<const unsigned char*>(a.wimg) + (size_t)d.seg * a.wimg_stride;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  mbar_expect_tx(&sm.wbar, (uint32_t)(kWChunkBytes<kGqG> + sizeof(WMeta<kGqG>)));
  bulk_g2s(sm.w, img, (uint32_t)kWChunkBytes<kGqG>, &sm.wbar);
  bulk_g2s(&sm.wmeta, img + kWChunkBytes<kGqG>, (uint32_t)sizeof(WMeta<kGqG>), &sm.wbar);
}

__device__ __forceinline__ void tc_ld16(uint32_t taddr, int (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ unsigned redux_max(unsigned v) {
  unsigned r;
  asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ int redux_add(int v) {
  int r;
  asm volatile("redux.sync.add.s32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
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
      mbar_init(&sm.empty[s], kGqWarps);
    }
    for (int s = 0; s < kSubRing; ++s) mbar_init(&sm.descfull[s], 1);
    mbar_init(&sm.wbar, 1);
    mbar_init(&sm.wfree, 1);
    mbar_init(&sm.g0bar, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.afull[b], kGqWarps);
      mbar_init(&sm.afree[b], 1);
      mbar_init(&sm.yfull[b], 1);
      mbar_init(&sm.yfree[b], kGqWarps);
    }
    mbar_init(&sm.sfull, 1);
    mbar_init(&sm.pfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < kGqG * 8) {
    (&sm.pmax[0][0])[tid] = 0u;
    (&sm.gsum[0][0])[tid] = 0;
  }
  if (warp == kGqWarps + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  if (warp == kGqWarps) {
    // ---- producer: descriptors and code stages of this CTA's items (as paths 0 / 1) ---------
    if (lane == 0) {
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
        // W image of item k >= 1 once item k - 1 is done with its own (its K UMMAs completed
        // and the consumers read its metadata): by now the consumers are deep in item k - 1's
        // V phase, so the wait is short (item 0's image comes from consumer thread 0)
        if (k > 0) {
          mbar_wait(&sm.wfree, (uint32_t)((k - 1) & 1));
          gq_issue_wimg(sm, args, d);
        }
        bool nhave = false;
        for (int ls = 0; ls < d.stages; ++ls, ++g) {
          const int slot = g % kGqStages;
          if (g >= kGqStages) mbar_wait(&sm.empty[slot], (uint32_t)((g / kGqStages - 1) & 1));
          gq_issue_stage(d, ls, sm.ring[slot], &sm.full[slot]);
          if (ls == min(2, d.stages - 1)) {
            // the ticket counter is shared with the previous launch on these args: under
            // programmatic dependent launch, wait for that grid before drawing from it
            if (k == 0) asm volatile("griddepcontrol.wait;\n" ::: "memory");
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

  if (warp == kGqWarps + 1) {
    // ---- MMA warp: one elected lane issues every UMMA of the CTA ---------------------------
    if (lane == 0) {
      const uint32_t id_k = tc_idesc(128, 128, 0, 1);  // codes u8 x W limbs s8
      const uint32_t id_v = tc_idesc(128, 128, 0, 0);  // codes u8 x P limbs u8
      int na = 0;              // A-buffer uses
      int uy[2] = {0, 0};      // Y-buffer uses
      for (int j = 0;; ++j) {
        mbar_wait_spin(&sm.descfull[j % kSubRing], (uint32_t)((j / kSubRing) & 1));
        const SubItem d = sm.sub[j % kSubRing];
        if (d.nbt == 0) break;
        const int nmb = (d.nbt + 1) / 2;
        mbar_wait_spin(&sm.wbar, (uint32_t)(j & 1));  // W image of this item's segment
        // S occupies the Y columns: the previous item's epilogue must have read both buffers
        for (int b = 0; b < 2; ++b)
          if (uy[b] > 0) mbar_wait_spin(&sm.yfree[b], (uint32_t)((uy[b] - 1) & 1));
        tc_fence_after();
        for (int ks = 0; ks < d.nK; ++ks, ++na) {
          const int ab = na & 1;
          mbar_wait_spin(&sm.afull[ab], (uint32_t)((na >> 1) & 1));
          tc_fence_after();
          const int rk0 = ks * d.RK, nr = min(d.RK, d.r - rk0);
          for (int kk = 0; kk < nr / 2; ++kk) {  // UMMA k-step = 32 bytes = 2 bond rows
            const int rr = rk0 + 2 * kk;
            // N rows (h*2 + limb)*8 + a: 16 core-matrix groups r*128 bytes apart
            const uint64_t bdesc = tc_sdesc(&sm.w[rr * 8], 128, d.r * 128);
            for (int mb = 0; mb < nmb; ++mb)
              tc_mma_ts(tmem + kGqColSY + (uint32_t)(mb * 128),
                        tmem + kGqColA + (uint32_t)(ab * 64 + mb * d.RK * 4 + kk * 8), bdesc, id_k,
                        (ks | kk) ? 1u : 0u);
          }
          tc_commit(&sm.afree[ab]);
        }
        tc_commit(&sm.sfull);
        mbar_wait_spin(&sm.pfull, (uint32_t)(j & 1));  // P limbs in shared memory, S read
        tc_fence_after();
        for (int vs = 0; vs < d.nslices; ++vs, ++na) {
          const int ab = na & 1, yb = vs & 1;
          mbar_wait_spin(&sm.afull[ab], (uint32_t)((na >> 1) & 1));
          if (uy[yb] > 0) mbar_wait_spin(&sm.yfree[yb], (uint32_t)((uy[yb] - 1) & 1));
          tc_fence_after();
          for (int kk = 0; kk < 2 * d.nbt; ++kk) {  // 32 rows b per k-step
            const uint64_t bdesc = tc_sdesc(&sm.pr.pb[kk * 2 * 128], 128, (kCB / 16) * 128);
            tc_mma_ts(tmem + kGqColSY + (uint32_t)(yb * 128), tmem + kGqColA + (uint32_t)(ab * 64 + kk * 8), bdesc,
                      id_v, kk ? 1u : 0u);
          }
          tc_commit(&sm.afree[ab]);
          tc_commit(&sm.yfull[yb]);
          ++uy[yb];
        }
      }
    }
    __syncwarp();
    named_sync2(kGqCons + 32);  // the consumers' last TMEM reads are done
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    return;
  }

  // ---- consumer warps ----------------------------------------------------------------------
  const int q = warp & 3;                // TMEM lane quarter of this warp
  const int wg = warp >> 2;              // warpgroup: K / softmax M-block; V tiles 2wg, 2wg+1; heads 4wg..4wg+3
  const int lane_in = 32 * q + lane;     // TMEM lane
  const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
  int st = 0, na = 0;
  int uyc[2] = {0, 0};
  auto release = [&](int s) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s % kGqStages]);
  };

  if (tid == 0) {
    mbar_wait(&sm.descfull[0], 0);
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // the combine may be scheduled
    if (sm.sub[0].nbt > 0) gq_issue_wimg(sm, args, sm.sub[0]);
  }

  for (int j = 0;; ++j) {
    mbar_wait(&sm.descfull[j % kSubRing], (uint32_t)((j / kSubRing) & 1));
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

    // ---- K phase: widen this thread's row b of each stage into TMEM --------------------------
    const int jt = 2 * wg + (q >> 1);        // tile of this thread's row
    const int b_in = 32 * (q & 1) + lane;    // row inside the tile
    for (int ks = 0; ks < d.nK; ++ks, ++st, ++na) {
      const int slot = st % kGqStages, ab = na & 1;
      mbar_wait(&sm.full[slot], (uint32_t)((st / kGqStages) & 1));
      if (na >= 2) mbar_wait(&sm.afree[ab], (uint32_t)(((na >> 1) - 1) & 1));
      const int rk0 = ks * d.RK, nr = min(d.RK, d.r - rk0);
      if (wg < nmb) {
        const unsigned char* tile = sm.ring[slot] + jt * nr * kI2Pad * RB;
        const bool live = jt < nbt;
        for (int r4 = 0; r4 < nr; r4 += 4) {
          uint32_t v[16];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rl = r4 + i, rr = rk0 + rl;
            uint2 w2 = make_uint2(0u, 0u);
            if (live) w2 = *reinterpret_cast<const uint2*>(tile + (rl * kI2Pad + (b_in ^ ((rr & 3) * 4))) * RB);
            v[4 * i] = w2.x & 0x0F0F0F0Fu;
            v[4 * i + 1] = (w2.x >> 4) & 0x0F0F0F0Fu;
            v[4 * i + 2] = w2.y & 0x0F0F0F0Fu;
            v[4 * i + 3] = (w2.y >> 4) & 0x0F0F0F0Fu;
          }
          tc_st16(tmem + lane_addr + kGqColA + (uint32_t)(ab * 64 + wg * d.RK * 4 + r4 * 4), v);
        }
        tc_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.afull[ab]);
      release(st);
    }
    stamp(1);

    // ---- softmax of the item straight from S in TMEM (this thread = row b) -----------------
    mbar_wait(&sm.wbar, (uint32_t)(j & 1));  // W metadata
    mbar_wait(&sm.sfull, (uint32_t)(j & 1));
    tc_fence_after();
    const bool row_ok = wg < nmb && jt < nbt && d.wb0 + jt * kI2Pad + b_in < d.i2;
    const float kscale = d.kscale * args.sm_scale * 1.4426950408889634f;
    float s[kGqG][8];
    if (wg < nmb) {
#pragma unroll
      for (int h0 = 0; h0 < kGqG; h0 += 4) {
        int acc[4][16];
#pragma unroll
        for (int hh = 0; hh < 4; ++hh)
          tc_ld16(tmem + lane_addr + kGqColSY + (uint32_t)(wg * 128 + (h0 + hh) * 16), acc[hh]);
        tc_wait_ld();
#pragma unroll
        for (int hh = 0; hh < 4; ++hh)
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            const int h = h0 + hh;
            const float v = (float)(256 * acc[hh][a] + acc[hh][8 + a] - sm.wmeta.beta[h][a][0]) *
                            (kscale * sm.wmeta.cs[h][a][0]);
            s[h][a] = row_ok ? v : -INFINITY;
          }
      }
    } else {
#pragma unroll
      for (int h = 0; h < kGqG; ++h)
#pragma unroll
        for (int a = 0; a < 8; ++a) s[h][a] = -INFINITY;
    }
    tc_fence_before();
#pragma unroll
    for (int h = 0; h < kGqG; ++h) {
      float m = s[h][0];
#pragma unroll
      for (int a = 1; a < 8; ++a) m = fmaxf(m, s[h][a]);
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) sm.rowmax[h][warp] = m;
    }
    named_sync(kGqCons);
    // every K UMMA completed before sfull and every W-metadata read is done: W(j+1) may land
    if (tid == 0) mbar_arrive(&sm.wfree);
    float mh[kGqG];
#pragma unroll
    for (int h = 0; h < kGqG; ++h) {
      float m = sm.rowmax[h][0];
#pragma unroll
      for (int w = 1; w < kGqWarps; ++w) m = fmaxf(m, sm.rowmax[h][w]);
      mh[h] = m;
    }
    // P = exp2(s - m_h) and the per-column maxima over the item's rows
#pragma unroll
    for (int h = 0; h < kGqG; ++h)
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const float p = s[h][a] == -INFINITY ? 0.f : exp2f(s[h][a] - mh[h]);
        s[h][a] = p;
        const unsigned mx = redux_max(__float_as_uint(p));
        if (lane == ((h * 8 + a) & 31)) atomicMax(&sm.pmax[h][a], mx);
      }
    named_sync(kGqCons);
    // 15-bit fixed point per column; limbs hi (<= 128) and lo into the B operand of the V UMMAs
    {
      const int b_item = jt * kI2Pad + b_in;
      unsigned char* pcol = sm.pr.pb + (b_item >> 4) * 128 + inv_ord16<4>(b_item & 15);
      const bool write = wg < nmb && jt < nbt;
#pragma unroll
      for (int h = 0; h < kGqG; ++h)
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          const int pint = __float2int_rn(s[h][a] * pow2_sub_exp(__uint_as_float(sm.pmax[h][a]), kGqPBits));
          const int gs = redux_add(pint);
          if (lane == ((h * 8 + a) & 31)) atomicAdd(&sm.gsum[h][a], gs);
          if (write) {
            pcol[((h * 2 + 0) * (kCB / 16)) * 128 + a * 16] = (unsigned char)(pint >> 8);
            pcol[((h * 2 + 1) * (kCB / 16)) * 128 + a * 16] = (unsigned char)(pint & 0xFF);
          }
        }
    }
    if (tid < kGqG * 8) (&sm.pinv[0][0])[tid] = pow2_exp_sub(__uint_as_float((&sm.pmax[0][0])[tid]), kGqPBits);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // P read by the tensor cores
    named_sync(kGqCons);
    if (tid == 0) mbar_arrive(&sm.pfull);
    stamp(2);

    // ---- V phase: widen stage vs, fold Y of stage vs - 1 while its UMMAs run ------------------
    float o[4][8];  // [head 4wg + hl][c] for e = lane_in & 15, summed over this thread's bond rows
#pragma unroll
    for (int hl = 0; hl < 4; ++hl)
#pragma unroll
      for (int c = 0; c < 8; ++c) o[hl][c] = 0.f;
    auto widen_v = [&]() {
      const int slot = st % kGqStages, ab = na & 1;
      mbar_wait(&sm.full[slot], (uint32_t)((st / kGqStages) & 1));
      if (na >= 2) mbar_wait(&sm.afree[ab], (uint32_t)(((na >> 1) - 1) & 1));
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int t = 2 * wg + i;
        if (t < nbt) {
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
      if (lane == 0) mbar_arrive(&sm.afull[ab]);
      release(st);
      ++st;
      ++na;
    };
    auto fold_y = [&](int vs) {
      const int yb = vs & 1;
      mbar_wait(&sm.yfull[yb], (uint32_t)(uyc[yb] & 1));
      ++uyc[yb];
      tc_fence_after();
      float yf[4][8];
      {
        int y[4][16];
#pragma unroll
        for (int hl = 0; hl < 4; ++hl)
          tc_ld16(tmem + lane_addr + kGqColSY + (uint32_t)(yb * 128 + (4 * wg + hl) * 16), y[hl]);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.yfree[yb]);
#pragma unroll
        for (int hl = 0; hl < 4; ++hl) {
          const int h = 4 * wg + hl;
          const float4 pi0 = *reinterpret_cast<const float4*>(&sm.pinv[h][0]);
          const float4 pi1 = *reinterpret_cast<const float4*>(&sm.pinv[h][4]);
          const int4 gs0 = *reinterpret_cast<const int4*>(&sm.gsum[h][0]);
          const int4 gs1 = *reinterpret_cast<const int4*>(&sm.gsum[h][4]);
          const float pi[8] = {pi0.x, pi0.y, pi0.z, pi0.w, pi1.x, pi1.y, pi1.z, pi1.w};
          const int gs[8] = {gs0.x, gs0.y, gs0.z, gs0.w, gs1.x, gs1.y, gs1.z, gs1.w};
#pragma unroll
          for (int a = 0; a < 8; ++a)
            yf[hl][a] = (float)(256 * y[hl][a] + y[hl][8 + a] - X * gs[a]) * pi[a];
        }
      }
      // O[h, c, e] += sum_a G0v[a, c, r] Y[h, a, (r, e)] for this thread's (r, e)
      const int rr = 8 * vs + (lane_in >> 4);
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const float4 g_lo = sm.g0v[2 * (a * kMaxR + rr)], g_hi = sm.g0v[2 * (a * kMaxR + rr) + 1];
#pragma unroll
        for (int hl = 0; hl < 4; ++hl) {
          const float y = yf[hl][a];
          ffma2(o[hl][0], o[hl][1], g_lo.x, g_lo.y, y, y);
          ffma2(o[hl][2], o[hl][3], g_lo.z, g_lo.w, y, y);
          ffma2(o[hl][4], o[hl][5], g_hi.x, g_hi.y, y, y);
          ffma2(o[hl][6], o[hl][7], g_hi.z, g_hi.w, y, y);
        }
      }
    };
    mbar_wait(&sm.g0bar, (uint32_t)(j & 1));
    for (int vs = 0; vs < d.nslices; ++vs) {
      widen_v();
      if (vs > 0) fold_y(vs - 1);
    }
    fold_y(d.nslices - 1);
    stamp(3);

    // ---- reduce over bond rows: lanes l / l ^ 16, then the 4 warps of the warpgroup ----------
#pragma unroll
    for (int hl = 0; hl < 4; ++hl)
#pragma unroll
      for (int c = 0; c < 8; ++c) o[hl][c] += __shfl_xor_sync(0xffffffffu, o[hl][c], 16);
    named_sync(kGqCons);  // every V UMMA has completed (yfull): P is dead
    if (lane < 16) {
#pragma unroll
      for (int hl = 0; hl < 4; ++hl)
#pragma unroll
        for (int c = 0; c < 8; ++c) sm.pr.red[q][4 * wg + hl][c * 16 + lane] = o[hl][c];
    }
    named_sync(kGqCons);
    for (int i = tid; i < kGqG * kD; i += kGqCons) {
      const int h = i / kD, dd = i % kD;
      const float v = sm.pr.red[0][h][dd] + sm.pr.red[1][h][dd] + sm.pr.red[2][h][dd] + sm.pr.red[3][h][dd];
      args.part_o[((size_t)d.part * kGqG + h) * kD + dd] = v * d.vscale;
    }
    if (tid < kGqG) {
      float l = 0.f;
#pragma unroll
      for (int a = 0; a < 8; ++a) l += (float)sm.gsum[tid][a] * sm.pinv[tid][a];
      args.part_ml[((size_t)d.part * kGqG + tid) * 2 + 0] = mh[tid];  // log2 domain
      args.part_ml[((size_t)d.part * kGqG + tid) * 2 + 1] = l;
    }
    named_sync(kGqCons);  // red, pmax, gsum, pinv, g0v reusable
    if (tid < kGqG * 8) {
      (&sm.pmax[0][0])[tid] = 0u;
      (&sm.gsum[0][0])[tid] = 0;
    }
    stamp(5);
  }
  tc_fence_before();
  named_sync2(kGqCons + 32);  // with the MMA warp: TMEM may be freed
}

}  // namespace attn
}  // namespace dq

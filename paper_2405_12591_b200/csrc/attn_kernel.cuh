// The split kernel of the fused decode attention; see attention.cu for the math.
//
// Persistent and dynamically scheduled: a grid of (SMs x resident CTAs) CTAs draws work
// items from a global ticket counter (self-resetting: the last CTA to retire zeroes it for
// the next launch).  A work item (sub-item) is <= NT 64-row b tiles of one segment
// (dq_attention_plan).
//
// Warp roles: TEAMS consumer teams of 8 warps (MMA, softmax, epilogue; they issue their own
// W-image and G0v copies at their own barrier points) and 1 producer warp whose lane 0 issues
// every code stage (cp.async.bulk, completing on the slot's `full` mbarrier).
//
// TEAMS = 2 (one CTA per SM, opt-in: DQ_ATTN_TEAMS_G1=2): the two teams work on different items
// and share ONE pool of ring slots.  A team in its softmax or epilogue holds no more than
// kTeamPrefetch stages of its next phase (the producer reads the phase each team has begun,
// `started`), so the other team can keep up to S - kTeamPrefetch slots in flight: the SM
// keeps streaming at its share of HBM through either team's fixed per-item phases.  (With
// two CTAs of one team each, a CTA in its softmax sits on a full private ring, and the other
// CTA's 80 KB in flight cannot carry the SM's share: 32-36 of 44 GB/s.)  Slots
// are handed out from a free mask, so the producer publishes each team's n-th slot (and the
// parity of its `full` phase) in the team's stage queue `sq`, behind an mbarrier `sqbar`.
// TEAMS = 1 (the default): two CTAs per SM, each with its own FIFO ring of slots (stage n in slot
// n % S, no stage queue).  Measured on C2: 62.5 us per layer for TEAMS = 1 against 69 us for
// TEAMS = 2 -- the shared pool does not hide the fixed phases better than the sibling CTA does,
// and its per-stage queue costs the consumers an extra wait.
#pragma once

#include "attn_prepare.cuh"

namespace dq {
namespace attn {

#ifndef DQ_ATTN_WARPS
#define DQ_ATTN_WARPS 8
#endif
constexpr int kWarps = DQ_ATTN_WARPS;       // consumer warps per team
constexpr int kThreads = kWarps * 32;       // consumer threads per team
constexpr int kCtaThreads = kThreads + 32;  // one team + the producer warp
constexpr int kD = 128;
constexpr int kMaxR = 64;
constexpr int kCB = 256;              // b rows per sub-item (at most)
constexpr int kTiles = kCB / kI2Pad;  // 64-row tiles per sub-item (at most)
constexpr int kNG = kCB / 16;         // 16-row groups per sub-item
constexpr int kStageBytes = 16384;
// TEAMS = 1: ring depth and CTAs per SM: 2 CTAs x 5 x 16 KB stages for g = 1; g = 2 needs a
// 32 KB W image, so 2 CTAs x 3 stages
#ifndef DQ_ATTN_STAGES_G1
#define DQ_ATTN_STAGES_G1 5
#endif
#ifndef DQ_ATTN_CTAS_G1
#define DQ_ATTN_CTAS_G1 2
#endif
template <int G>
constexpr int kStagesOf = G == 1 ? DQ_ATTN_STAGES_G1 : 3;
template <int G, int TEAMS = 1>
constexpr int kCtasPerSm = TEAMS > 1 ? 1 : (G == 1 ? DQ_ATTN_CTAS_G1 : 2);
constexpr int kSubRing = 4;  // descriptor ring per team (in use: the current item, the next, one fetched)
constexpr int kQ = 32;       // per-team stage queue (>= ring slots)
// stages of a team's NEXT phase the producer issues while the team has not begun it
#ifndef DQ_TEAM_PREFETCH
#define DQ_TEAM_PREFETCH 3
#endif
constexpr int kTeamPrefetch = DQ_TEAM_PREFETCH;
constexpr int kSmemCap = 227 * 1024;  // dynamic shared memory per CTA (sm_100)
// Opt-in measurement build (-DDQ_INKERNEL_W=1): the W image computed inside the split kernel by
// the fetcher warp (g = 1, symmetric, one team per CTA, items of <= 256 rows), no prepare
// kernel; the W buffer then sits apart from an fp16 G0v buffer, and the fetcher writes item
// j + 1's W while item j is in its softmax / V phase.  Measured on C2: split kernel 86 us
// against 60 us, step 2.78 ms against 2.20 ms -- one warp computing 16 KB of W per item is too
// slow (a 2.5 us wait before each item) and the fp16 G0v fold lengthens the epilogue.
#ifndef DQ_INKERNEL_W
#define DQ_INKERNEL_W 0
#endif

template <int TEAMS>
constexpr int kCtaThreadsOf = TEAMS * kThreads + 32 * (TEAMS + 1);  // + a producer warp per team + the fetcher

template <int BITS>
constexpr int kPBits = 15;  // P / tile max in (0.5, 1] -> round(P * 2^(kPBits - e)); Y sums per 64-row tile

// one sub-item = (segment, b0, tiles): everything the producer and the consumers need,
// including the stage geometry (computed once when the descriptor is loaded)
struct SubItem {
  const unsigned char* kc;
  const unsigned char* vc;
  const float* vg0;  // fp32 G0v [a][rr][8 c] (normalised)
  float kscale, vscale;
  int seg, wb0, nbt, part;
  int r, i1, i2, item;
  int RK, nK, RV, nslices;  // K stages: RK bond rows x nbt tiles; V stages: (tile, slice of RV rows)
  int stages, pad_[3];      // nbt == 0: end of this team's items
};

// per-team state: descriptors, stage queue, W image / G0v, P, reductions
template <int G, int NT, bool ASYM, int QN = kQ>
struct TeamSmem {
  static constexpr bool kInW = DQ_INKERNEL_W && G == 1 && !ASYM && QN == 1 && NT <= kTiles;
  uint64_t wbar;   // W image (attn_prepare.cuh) by TMA, or by the fetcher warp (kInW); one phase per item
  uint64_t g0bar;  // G0v prefetch, one phase per sub-item
  uint64_t wfree;  // kInW: the consumers are past an item's K phase (its W buffer may be rewritten)
  uint64_t descfull[kSubRing];  // descriptor j written (producer arrival), phase j / kSubRing
  uint64_t sqbar[QN];           // stage n's slot published (producer arrival), phase n / kQ (TEAMS = 2)
  int sq[QN];                   // stage n of the team: ring slot | (full-barrier parity << 8)
  int started;                  // phase the consumers began: 2j = K of item j, 2j + 1 = V of item j
  int fetched;                  // descriptors the fetcher warp has written into `sub` (release / acquire)
  int taken;                    // descriptors the producer has made current
  int pad_;
  int kend[kSubRing], vend[kSubRing];  // producer: team stage index where item j's K / V phase ends
  SubItem sub[kSubRing];        // the team's j-th item lives in slot j % kSubRing
  alignas(16) WMeta<G> wmeta;  // per-column W scales and excess corrections (TMA target)
  int gamma[G][8][NT];     // excess correction of Y per 64-row tile: kExcess * sum_b Pint[a][b]
  float lsum[G][kWarps];   // probability mass per warp
  unsigned pmax[G][8][NT];  // largest probability per (h, a, tile), float bits
  // K phase: W limbs, 16-byte chunks [((h*2 + limb)*r + rr)*8 + (a ^ 2*(rr&3))];
  // V phase + epilogue (aliased, W is dead): fp32 G0v [a][rr][c] by TMA.  (Measured: separate
  // W and fp16 G0v buffers, the next W image loaded by the producer right after the K phase,
  // shorten the gap between items but lengthen the epilogue: C2 66 us against 62 us.)
  union {
    uint4 w[G * 2 * kMaxR * 8];
    float4 g0v[kInW ? 1 : 8 * (kMaxR * 2 + 1)];  // [a][rr][c] with a 16-byte pad per a (kG0vPad)
  } wg;
  // kInW: fp16 G0v [a][rr][8 c], r + 1 chunks per a (a 16-byte pad: the lanes tid4 = 0..3 read
  // a = 2 tid4 + aa four banks apart), loaded at the previous item's end; q of the item's unit
  uint4 g0v16[kInW ? 8 * (kMaxR + 1) : 1];
  float qs[kInW ? 128 : 1];
  // V phase: P limbs [((h*2 + limb)*8 + a)*(4 NT) + (bg ^ 4*(a&1))];
  // epilogue (aliased, P is dead): cross-warp reduction of the O partial
  union {
    uint4 p[G * 2 * 8 * 4 * NT];
    float red[kWarps][G][kD];
  } pr;
  float rowmax[G][kWarps];
  // asymmetric mode: the segment's V channel table [2][r][16] (scales, zero points; r <= kMaxR)
  alignas(16) float vch[ASYM ? 2 * kMaxR * 16 : 4];
};

template <int TEAMS>
constexpr int kQOf = TEAMS > 1 ? kQ : 1;  // a lone team reads its FIFO ring: no stage queue

template <int G, int NT, bool ASYM, int TEAMS>
constexpr int ring_stages() {
  constexpr int team = (int)sizeof(TeamSmem<G, NT, ASYM, kQOf<TEAMS>>);
  if constexpr (TEAMS == 1) {
    // as many stages (<= kStagesOf) as keep 2 CTAs per SM: 228 KB per SM, 1 KB reserved per CTA
    constexpr int s = (228 * 1024 / 2 - 1024 - team - 256) / (kStageBytes + 16);
    return s < kStagesOf<G> ? s : kStagesOf<G>;
  } else {
    const int s = (kSmemCap - TEAMS * team - 256) / (kStageBytes + 16);
    return s > 24 ? 24 : s;
  }
}

// NT: 64-row tiles per work item (4, or 8 for g = 1: twice the bytes per fixed per-item cost)
template <int G, int NT = kTiles, bool ASYM = false, int TEAMS = 1>
struct AttnSmem {
  static constexpr int kStages = ring_stages<G, NT, ASYM, TEAMS>();
  alignas(128) unsigned char ring[kStages][kStageBytes];
  uint64_t full[kStages];
  uint64_t empty[kStages];
  unsigned freemask;        // the slot pool: bit s set = slot s free (shared by the team producers)
  int slot_use[kStages];    // uses of each slot so far: the parity of its full / empty phases
  TeamSmem<G, NT, ASYM, kQOf<TEAMS>> team[TEAMS];
};

// stage geometry of a sub-item with r bond rows and nbt tiles
template <int BITS>
__device__ __forceinline__ void stage_geometry(SubItem& d) {
  constexpr int RB = 2 * BITS;
  int RK = (kStageBytes / (d.nbt * kI2Pad * RB)) & ~3;
  if (RK > d.r) RK = d.r;
  const int rw = d.r / kWarps;
  int kslice = kWarps;
  while (kslice > 1 && kslice * rw * 16 * kI2Pad * BITS / 8 > kStageBytes) kslice >>= 1;
  d.RK = RK;
  d.nK = (d.r + RK - 1) / RK;
  d.RV = kslice * rw;
  d.nslices = kWarps / kslice;
  d.stages = d.nK + d.nbt * d.nslices;
}

template <int BITS>
__device__ __forceinline__ void load_sub(SubItem& d, const dq_attn_args& a, int w) {
  const int sg = a.work[3 * w];
  const dq_segment& s = a.segs[sg];
  SubItem t;
  t.kc = s.k_codes;
  t.vc = s.v_codes;
  t.vg0 = static_cast<const float*>(s.v_g0);  // fp32, or fp16 under kInW (dq_attention_g0v_dtype)
  t.kscale = s.k_scale;
  t.vscale = s.v_scale;
  t.seg = sg;
  t.wb0 = a.work[3 * w + 1];
  t.nbt = a.work[3 * w + 2];
  t.part = a.work_part[w];
  t.r = s.r;
  t.i1 = s.i1;
  t.i2 = s.i2;
  t.item = w;
  stage_geometry<BITS>(t);
  d = t;
}

// the W image (limb chunks + metadata) of a sub-item's segment onto the team's wbar (one thread)
template <int G, int NT, bool ASYM, int QN>
__device__ __forceinline__ void issue_wimg(TeamSmem<G, NT, ASYM, QN>& tm, const dq_attn_args& a, const SubItem& d) {
  const unsigned char* img = static_cast<const unsigned char*>(a.wimg) + (size_t)d.seg * a.wimg_stride;
  const uint32_t wb = (uint32_t)(G * 2 * d.r * 8 * 16);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  mbar_expect_tx(&tm.wbar, wb + (uint32_t)sizeof(WMeta<G>));
  bulk_g2s(tm.wg.w, img, wb, &tm.wbar);
  bulk_g2s(&tm.wmeta, img + kWChunkBytes<G>, (uint32_t)sizeof(WMeta<G>), &tm.wbar);
}

// kInW: fp16 G0v (one copy per a into its padded block) and, asymmetric... (kInW is symmetric
// only) onto the team's g0bar (one thread)
template <int G, int NT, bool ASYM, int QN>
__device__ __forceinline__ void issue_g0v16(TeamSmem<G, NT, ASYM, QN>& tm, const SubItem& d) {
  mbar_expect_tx(&tm.g0bar, (uint32_t)(d.i1 * d.r * 16));
  const uint4* src = reinterpret_cast<const uint4*>(d.vg0);
  for (int aa = 0; aa < d.i1; ++aa)
    bulk_g2s(tm.g0v16 + aa * (d.r + 1), src + aa * d.r, (uint32_t)(d.r * 16), &tm.g0bar);
}

template <int NT>
__device__ __forceinline__ int p_chunk(int h, int limb, int a, int bg) {
  return ((h * 2 + limb) * 8 + a) * (4 * NT) + (bg ^ (4 * (a & 1)));
}

// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// named barrier (1 + team) over one team's consumer threads
__device__ __forceinline__ void team_sync(int team) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(1 + team), "r"(kThreads) : "memory");
}

// ---- the producer (lane 0 of the last warp) ---------------------------------------------
// Per team: the issue geometry of the item being streamed (registers) and the next item's
// descriptor, loaded into the team's descriptor ring as soon as its ticket is drawn.  Every
// iteration reclaims the slots the teams released (test_wait on `empty`, in each team's stage
// order), then issues one stage into a free slot for the eligible team with the fewest stages
// in flight.  A team is eligible while its next stage lies before the end of the phase its
// consumers have begun + kTeamPrefetch (TEAMS = 2; a lone team is never capped).
struct Issue {  // what issuing a stage needs, kept in registers
  const unsigned char* kc;
  const unsigned char* vc;
  int bt0, nbt, r, RK, nK, RV, nslices, stages;
};

__device__ __forceinline__ Issue issue_of(const SubItem& d) {
  Issue it;
  it.kc = d.kc;
  it.vc = d.vc;
  it.bt0 = d.wb0 / kI2Pad;
  it.nbt = d.nbt;
  it.r = d.r;
  it.RK = d.RK;
  it.nK = d.nK;
  it.RV = d.RV;
  it.nslices = d.nslices;
  it.stages = d.stages;
  return it;
}

// issue local stage `st` of an item into its ring slot (one thread)
// (no proxy fence: the slot's previous contents were only read by the consumers, whose release
// the producer observed on the slot's `empty` mbarrier before reissuing it)
template <int BITS>
__device__ __forceinline__ void issue_stage(const Issue& d, int st, unsigned char* slot_buf, uint64_t* bar) {
  constexpr int RB = 2 * BITS;
  if (st < d.nK) {
    const int rk0 = st * d.RK;
    const int nr = min(d.RK, d.r - rk0);
    const uint32_t chunk = (uint32_t)(nr * kI2Pad * RB);
    mbar_expect_tx(bar, chunk * d.nbt);
    const unsigned char* src = d.kc + ((size_t)d.bt0 * d.r + rk0) * kI2Pad * RB;
    for (int j = 0; j < d.nbt; ++j) bulk_g2s(slot_buf + j * chunk, src + (size_t)j * d.r * kI2Pad * RB, chunk, bar);
  } else {
    const int v = st - d.nK;
    const int btl = v / d.nslices, sl = v - btl * d.nslices;
    const uint32_t bytes = (uint32_t)(d.RV * 16 * kI2Pad * BITS / 8);
    mbar_expect_tx(bar, bytes);
    const unsigned char* src = d.vc + ((size_t)(d.bt0 + btl) * d.r + sl * d.RV) * 16 * kI2Pad * BITS / 8;
    bulk_g2s(slot_buf, src, bytes, bar);
  }
}

struct TeamProd {
  Issue cur;
  int ls;        // next local stage of cur
  int k;         // descriptors taken
  int issued, reclaimed;
  bool hc;       // streaming an item
};

__device__ __forceinline__ bool elect_lane() {
  uint32_t p;
  asm volatile("{\n.reg .pred P;\n.reg .b32 r;\nelect.sync r|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}" : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// ---- the fetcher (lane 0 of the warp after the producer) ----------------------------------
// Keeps each team's next descriptors ready in its ring (ticket from the global counter, then the
// work-list entry and the segment: dependent global loads of ~1 us that used to stall the
// producer once per item), at most kFetchAhead ahead of what the producer has taken.
// descriptors a team holds beyond its current item: 1 = the next item only (C2 62.5 us per layer;
// 2: 68 us -- tickets drawn early leave the last round unbalanced)
#ifndef DQ_FETCH_AHEAD
#define DQ_FETCH_AHEAD 1
#endif
constexpr int kFetchAhead = DQ_FETCH_AHEAD;

// W image of one item, computed by the whole fetcher warp straight into the team's W buffer: the
// prepare kernel's arithmetic (attn_prepare.cuh, path 0, g = 1, symmetric) one column a at a
// time -- lane l holds bond rows l and l + 32 (16 e each, ord16 order), the column's group
// maxima and beta are warp reductions.  Columns a >= i1 get beta 0 and the scale of a zero
// maximum, as in the prepare kernel (their scores are masked).
template <int BITS, int G, int NT, bool ASYM, int QN>
__device__ void compute_w(TeamSmem<G, NT, ASYM, QN>& tm, const dq_attn_args& args, const SubItem& d, int lane) {
  constexpr int X = kExcess<BITS>;
  const dq_segment& seg = args.segs[d.seg];
  const int r = seg.r, i1 = seg.i1;
  {  // q of the unit -> fp32 in shared memory (4 values per lane)
    const __half2* qh = reinterpret_cast<const __half2*>(args.q) + (size_t)seg.unit * 64;
    const float2 x0 = __half22float2(qh[2 * lane]), x1 = __half22float2(qh[2 * lane + 1]);
    reinterpret_cast<float4*>(tm.qs)[lane] = make_float4(x0.x, x0.y, x1.x, x1.y);
  }
  __syncwarp();
  const float4* g0k = reinterpret_cast<const float4*>(seg.k_g0);  // fp32 [a][rr][c], normalised
  for (int a = 0; a < 8; ++a) {
    float wv[2][16];
    float m[2] = {0.f, 0.f};
    bool live[2];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int rr = lane + 32 * h2;
      live[h2] = a < i1 && rr < r;
      float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
      if (live[h2]) {
        lo = g0k[2 * (a * r + rr)];
        hi = g0k[2 * (a * r + rr) + 1];
      }
      const float gk[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
      for (int i = 0; i < 16; ++i) wv[h2][i] = 0.f;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4* q4 = reinterpret_cast<const float4*>(&tm.qs[c * 16]);
        const float4 x0 = q4[0], x1 = q4[1], x2 = q4[2], x3 = q4[3];
        const float qc[16] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w,
                              x2.x, x2.y, x2.z, x2.w, x3.x, x3.y, x3.z, x3.w};
#pragma unroll
        for (int i = 0; i < 16; ++i) wv[h2][i] = fmaf(qc[ord16<BITS>(i)], gk[c], wv[h2][i]);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) m[h2] = fmaxf(m[h2], fabsf(wv[h2][i]));
    }
    // group 0: bond rows < kGroupR (lanes < 8, first row), group 1: the rest
    const unsigned g0 = live[0] && lane < kGroupR ? __float_as_uint(m[0]) : 0u;
    const unsigned g1 = __float_as_uint(fmaxf(live[0] && lane >= kGroupR ? m[0] : 0.f, live[1] ? m[1] : 0.f));
    const unsigned wmax[2] = {__reduce_max_sync(0xffffffffu, g0), __reduce_max_sync(0xffffffffu, g1)};
    int wsum[2] = {0, 0};
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      if (!live[h2]) continue;
      const int rr = lane + 32 * h2, grp = rr < kGroupR ? 0 : 1;
      const float wq = pow2_sub_exp(__uint_as_float(wmax[grp]), kWBits<BITS>);
      uint32_t hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int wint = __float2int_rn(wv[h2][i] * wq);
        wsum[grp] += wint;
        const int whi = wint >> 8;  // path 0: hi signed, lo unsigned
        hi[i >> 2] |= (uint32_t)(whi & 0xFF) << (8 * (i & 3));
        lo[i >> 2] |= (uint32_t)((wint - 256 * whi) & 0xFF) << (8 * (i & 3));
      }
      tm.wg.w[w_chunk(0, 0, r, rr, a, 0)] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      tm.wg.w[w_chunk(0, 1, r, rr, a, 0)] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    const int b0 = __reduce_add_sync(0xffffffffu, wsum[0]), b1 = __reduce_add_sync(0xffffffffu, wsum[1]);
    if (lane < 2) {
      tm.wmeta.beta[0][a][lane] = X * (lane == 0 ? b0 : b1);
      tm.wmeta.cs[0][a][lane] = pow2_exp_sub(__uint_as_float(wmax[lane]), kWBits<BITS>);
    }
  }
  __syncwarp();  // every lane's stores precede the leader's release on wbar
}

// ---- the fetcher (the warp after the producers) --------------------------------------------
// Lane 0 keeps each team's next descriptors ready in its ring (ticket from the global counter,
// then the work-list entry and the segment: dependent global loads of ~1 us that used to stall
// the producer once per item), at most kFetchAhead ahead of what the producer has taken.  With
// the in-kernel W image (kInW) the whole warp also computes item j + 1's W image as soon as the
// consumers are past item j's K phase, and releases it on the team's wbar.
template <int BITS, int G, int NT, bool ASYM, int TEAMS>
__device__ void fetch(AttnSmem<G, NT, ASYM, TEAMS>& sm, const dq_attn_args& args, int lane) {
  using TS = TeamSmem<G, NT, ASYM, kQOf<TEAMS>>;
  constexpr bool INW = TS::kInW;
  int fk[TEAMS];
  bool done[TEAMS];
  bool waited = false;  // griddepcontrol.wait before the first ticket (the counter is shared with
                        // the previous launch on these args) and before the first q read
  int left = TEAMS;
  int kw = 0;           // kInW (one team): the next item whose W image is due
  bool wdone = !INW;
#pragma unroll
  for (int t = 0; t < TEAMS; ++t) {
    const int first = (int)blockIdx.x + t * (int)gridDim.x;
    done[t] = first >= args.nwork;
    if (lane == 0) {
      if (done[t]) sm.team[t].sub[0].nbt = 0;
      else load_sub<BITS>(sm.team[t].sub[0], args, first);
      st_release(&sm.team[t].fetched, 1);
    }
    if (done[t]) --left;
    fk[t] = 1;
  }
  __syncwarp();
  while (left > 0 || !wdone) {
    bool idle = true;
#pragma unroll
    for (int t = 0; t < TEAMS; ++t) {
      if (done[t] || fk[t] - ld_acquire(&sm.team[t].taken) >= kFetchAhead) continue;
      idle = false;
      if (!waited) {
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        waited = true;
      }
      int nx = 0;
      if (lane == 0) nx = atomicAdd(args.sched, 1);
      nx = TEAMS * (int)gridDim.x + __shfl_sync(0xffffffffu, nx, 0);
      SubItem& dst = sm.team[t].sub[fk[t] & (kSubRing - 1)];
      if (nx < args.nwork) {
        if (lane == 0) load_sub<BITS>(dst, args, nx);
      } else {
        if (lane == 0) dst.nbt = 0;
        done[t] = true;
        --left;
      }
      ++fk[t];
      if (lane == 0) st_release(&sm.team[t].fetched, fk[t]);
      __syncwarp();
    }
    if constexpr (INW) {
      TS& tm = sm.team[0];
      if (!wdone && kw < fk[0]) {
        const SubItem& d = tm.sub[kw & (kSubRing - 1)];
        if (d.nbt == 0) {
          wdone = true;
        } else if (kw == 0 || mbar_test(&tm.wfree, (uint32_t)((kw - 1) & 1))) {
          if (!waited) {
            asm volatile("griddepcontrol.wait;\n" ::: "memory");  // q comes from the previous kernel
            waited = true;
          }
          compute_w<BITS>(tm, args, d, lane);
          if (lane == 0) mbar_arrive(&tm.wbar);
          ++kw;
          idle = false;
        }
      }
    }
    if (idle) __nanosleep(64);
  }
  // retire: the last CTA to finish drawing resets the counters for the next launch
  if (!waited) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(args.sched + 1, 1) == (int)gridDim.x - 1) {
      args.sched[0] = 0;
      args.sched[1] = 0;
    }
  }
}

// ---- the producers: one warp per team, converged --------------------------------------------
// Every lane holds the same (warp-uniform) state and one elected lane performs the stores,
// arrivals and copies (a lone `lane == 0` loop makes the compiler wrap each bulk copy's
// operands in a register-to-uniform broadcast loop).  Team t's producer claims slots from the
// CTA's pool (shared-memory atomics on `freemask`), publishes each one in the team's stage
// queue and issues the copies; it returns the slots its consumers released (test_wait on
// `empty`, in stage order).  Its issue limit is the end of the phase its consumers have begun
// + kTeamPrefetch (TEAMS = 1: none), so a team in its softmax or epilogue leaves the rest of
// the pool to the other team.
template <int BITS, int G, int NT, bool ASYM, int TEAMS>
__device__ void produce(AttnSmem<G, NT, ASYM, TEAMS>& sm, const dq_attn_args& args, int t) {
  using TS = TeamSmem<G, NT, ASYM, kQOf<TEAMS>>;
  static_assert((kQ & (kQ - 1)) == 0 && (kSubRing & (kSubRing - 1)) == 0, "power-of-two rings");
  TS& tm = sm.team[t];
  const bool leader = elect_lane();
  const int leader_lane = __ffs(__ballot_sync(0xffffffffu, leader)) - 1;
  TeamProd p;
  p.k = p.issued = p.reclaimed = 0;
  // descriptor p.k (from the fetcher) becomes current and is published to the consumers
  auto advance = [&]() {
    const int ds = p.k & (kSubRing - 1);
    while (ld_acquire(&tm.fetched) <= p.k) {
    }
    p.ls = 0;
    p.hc = tm.sub[ds].nbt > 0;
    if (p.hc) p.cur = issue_of(tm.sub[ds]);
    if (leader) {
      if (p.hc) {
        tm.kend[ds] = p.issued + p.cur.nK;
        tm.vend[ds] = p.issued + p.cur.stages;
      }
      mbar_arrive(&tm.descfull[ds]);  // release: the descriptor is visible to its waiters
      st_release(&tm.taken, p.k + 1);
    }
    ++p.k;
    __syncwarp();
  };
  auto reclaim = [&]() {
    uint32_t back = 0;
    while (p.reclaimed < p.issued) {
      const int e = tm.sq[p.reclaimed & (kQ - 1)];
      if (!mbar_test(&sm.empty[e & 0xFF], (uint32_t)(e >> 8))) break;
      back |= 1u << (e & 0xFF);
      ++p.reclaimed;
    }
    if (back && leader) atomicOr(&sm.freemask, back);
  };
  advance();
  if constexpr (TEAMS == 1) {  // a private FIFO ring: stage n in slot n % S, no queue needed
    constexpr int S = AttnSmem<G, NT, ASYM, TEAMS>::kStages;
    while (p.hc) {
      const int slot = p.issued % S;
      if (p.issued >= S) mbar_wait_spin(&sm.empty[slot], (uint32_t)((p.issued / S - 1) & 1));
      if (leader) issue_stage<BITS>(p.cur, p.ls, sm.ring[slot], &sm.full[slot]);
      ++p.issued;
      if (++p.ls == p.cur.stages) advance();
    }
    return;
  }
  for (;;) {
    reclaim();
    if (!p.hc) {
      if (p.reclaimed == p.issued) break;  // every slot of this team is back in the pool
      continue;
    }
    int lim = 0x7fffffff;
    if (TEAMS > 1) {
      const int ph = *reinterpret_cast<volatile int*>(&tm.started);
      const int jp = (ph >> 1) & (kSubRing - 1);
      lim = ((ph & 1) ? tm.vend[jp] : tm.kend[jp]) + kTeamPrefetch;
    }
    while (p.hc && p.issued < lim && p.issued - p.reclaimed < kQ) {
      int slot = -1, par = 0;
      if (leader) {
        unsigned m = *reinterpret_cast<volatile unsigned*>(&sm.freemask);
        while (m) {
          const int b = __ffs(m) - 1;
          const unsigned old = atomicAnd(&sm.freemask, ~(1u << b));
          if (old & (1u << b)) {
            slot = b;
            par = atomicAdd(&sm.slot_use[b], 1) & 1;
            break;
          }
          m = old & ~(1u << b);
        }
        if (slot >= 0) {
          tm.sq[p.issued & (kQ - 1)] = slot | (par << 8);
          mbar_arrive(&tm.sqbar[p.issued & (kQ - 1)]);
          issue_stage<BITS>(p.cur, p.ls, sm.ring[slot], &sm.full[slot]);
        }
      }
      slot = __shfl_sync(0xffffffffu, slot, leader_lane);
      if (slot < 0) break;
      ++p.issued;
      if (++p.ls == p.cur.stages) advance();  // item fully issued: the next one becomes current
    }
  }
}

template <int BITS, int G, int NT = kTiles, bool ASYM = false, int TEAMS = 1>
__global__ void __launch_bounds__(kCtaThreadsOf<TEAMS>, kCtasPerSm<G, TEAMS>) decode_attn_kernel(dq_attn_args args) {
  constexpr int RB = 2 * BITS;
  constexpr int X = kExcess<BITS>;
  constexpr bool SA = BITS == 8;  // A operand (codes) signed
  extern __shared__ __align__(128) unsigned char smem_raw[];
  AttnSmem<G, NT, ASYM, TEAMS>& sm = *reinterpret_cast<AttnSmem<G, NT, ASYM, TEAMS>*>(smem_raw);
  constexpr int S = AttnSmem<G, NT, ASYM, TEAMS>::kStages;

  const int warp_all = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp_all / kWarps;                 // == TEAMS for the producer / fetcher warps
  const int warp = warp_all - team * kWarps;          // warp within the team
  const int tid = (int)threadIdx.x - team * kThreads;  // thread within the team
  const int gid = lane >> 2, tid4 = lane & 3;

  // ---- prologue: barriers ---------------------------------------------------------------
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kWarps);
      sm.slot_use[s] = 0;
    }
    sm.freemask = S >= 32 ? ~0u : ((1u << S) - 1u);
    for (int t = 0; t < TEAMS; ++t) {
      for (int s = 0; s < kSubRing; ++s) mbar_init(&sm.team[t].descfull[s], 1);
      for (int s = 0; s < kQOf<TEAMS>; ++s) mbar_init(&sm.team[t].sqbar[s], 1);
      mbar_init(&sm.team[t].wbar, 1);
      mbar_init(&sm.team[t].wfree, 1);
      mbar_init(&sm.team[t].g0bar, 1);
      sm.team[t].started = 0;  // item 0's K phase: issue it whole before the consumers arrive
      sm.team[t].fetched = 0;
      sm.team[t].taken = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (team < TEAMS && tid < G * 8 * NT) {
    (&sm.team[team].gamma[0][0][0])[tid] = 0;
    (&sm.team[team].pmax[0][0][0])[tid] = 0u;
  }
  __syncthreads();  // barrier inits visible to every warp

  if (team == TEAMS) {
    // ---- producer: the code stages of this CTA's items (the code does not depend on the
    // prepare kernel, so no griddepcontrol.wait before the first stages); the next warp
    // fetches the work items
    if (warp < TEAMS) produce<BITS, G, NT, ASYM, TEAMS>(sm, args, warp);  // the whole warp, converged
    else fetch<BITS, G, NT, ASYM, TEAMS>(sm, args, lane);  // the whole warp
    return;
  }
  TeamSmem<G, NT, ASYM, kQOf<TEAMS>>& tm = sm.team[team];
  constexpr bool INW = TeamSmem<G, NT, ASYM, kQOf<TEAMS>>::kInW;

  if (tid == 0) {
    mbar_wait(&tm.descfull[0], 0);
    if constexpr (INW) {
      if (tm.sub[0].nbt > 0) issue_g0v16(tm, tm.sub[0]);
    }
    // programmatic dependent launch: everything above overlapped the prepare kernel; its
    // output (the per-segment W images) is read from here on
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // the combine may be scheduled
    if constexpr (!INW) {
      if (tm.sub[0].nbt > 0) issue_wimg(tm, args, tm.sub[0]);
    }
  }

  int st = 0;  // the team's running stage index (identical in every thread of the team)
  auto acquire = [&]() -> int {  // slot of stage st, once its codes have landed
    if constexpr (TEAMS == 1) {
      const int slot = st % S;
      mbar_wait(&sm.full[slot], (uint32_t)((st / S) & 1));
      return slot;
    }
    mbar_wait(&tm.sqbar[st % kQ], (uint32_t)((st / kQ) & 1));
    const int e = tm.sq[st % kQ];
    mbar_wait(&sm.full[e & 0xFF], (uint32_t)(e >> 8));
    return e & 0xFF;
  };
  auto release = [&](int slot) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[slot]);
  };
  auto begin_phase = [&](int ph) {
    if (tid == 0) *reinterpret_cast<volatile int*>(&tm.started) = ph;
  };

  for (int j = 0;; ++j) {
    mbar_wait(&tm.descfull[j % kSubRing], (uint32_t)((j / kSubRing) & 1));
    const SubItem d = tm.sub[j % kSubRing];
    if (d.nbt == 0) break;
    const int r = d.r, i1 = d.i1, i2 = d.i2, wb0 = d.wb0;
    const int nbt = d.nbt;
    begin_phase(2 * j);
    mbar_wait(&tm.wbar, (uint32_t)(j & 1));
#ifdef DQ_ATTN_TRACE  // measurement builds: per-item phase stamps [nwork][8] (global ns)
    auto stamp = [&](int k) {
      if (args.trace && tid == 0) args.trace[(size_t)d.item * 8 + k] = global_ns();
    };
    if (args.trace && tid == 0) {
      args.trace[(size_t)d.item * 8 + 5] = blockIdx.x;
      args.trace[(size_t)d.item * 8 + 6] = sm_id();
      args.trace[(size_t)d.item * 8 + 7] = team;
    }
#else
    auto stamp = [](int) {};
#endif
    stamp(0);

    // ---- phase 1: S = W . codes_k on the int8 tensor pipe ------------------------------
    constexpr int kWpt = kWarps / NT;       // warps per 64-row tile
    constexpr int MT = 4 / kWpt;            // 16-row m-tiles per warp
    const int jt = warp / kWpt;             // tile of this warp inside the sub-item
    const int bl_base = 16 * MT * (warp % kWpt);  // first row of this warp inside the tile
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
    const float kscale = d.kscale * args.sm_scale * 1.4426950408889634f;
    auto flush_group = [&](int grp) {
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float cs[2];
        int bt[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          cs[q] = kscale * tm.wmeta.cs[h][2 * tid4 + q][grp];
          bt[q] = tm.wmeta.beta[h][2 * tid4 + q][grp];
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int k = 0; k < 4; k += 2) {
            ffma2(sacc[mt][h][k], sacc[mt][h][k + 1], (float)(256 * acc_hi[mt][h][k] + acc_lo[mt][h][k] - bt[0]),
                  (float)(256 * acc_hi[mt][h][k + 1] + acc_lo[mt][h][k + 1] - bt[1]), cs[0], cs[1]);
            acc_hi[mt][h][k] = acc_lo[mt][h][k] = acc_hi[mt][h][k + 1] = acc_lo[mt][h][k + 1] = 0;
          }
      }
    };
    // per-thread constant parts of the fragment addresses: the K-tile swizzle and the W
    // chunk swizzle depend on rr & 3 = tid4 only (stages and q0 steps are multiples of 4)
    const int swz = tid4 * (16 / BITS);
    int row_off[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int b0 = bl_base + mt * 16 + gid;
      row_off[mt][0] = (tid4 * kI2Pad + (b0 ^ swz)) * RB;
      row_off[mt][1] = (tid4 * kI2Pad + ((b0 + 8) ^ swz)) * RB;
    }
    const uint4* wthr = tm.wg.w + tid4 * 8 + (gid ^ (2 * tid4));
    const int wl = r * 8;  // chunks per (head, limb)
    for (int ks = 0; ks < d.nK; ++ks, ++st) {
      const int slot = acquire();
#ifdef DQ_ATTN_NULL_CONSUMER  // measurement only: the memory pipeline without the contractions
      release(slot);
      continue;
#endif
      const int rk0 = ks * d.RK;
      const int nr = min(d.RK, r - rk0);
      if (jt < nbt) {
        const unsigned char* tile = sm.ring[slot] + jt * nr * kI2Pad * RB;
        const uint4* wp = wthr + rk0 * 8;
        for (int q0 = 0; q0 < nr; q0 += 4, tile += 4 * kI2Pad * RB, wp += 32) {
          uint4 bh[G], bl[G];
#pragma unroll
          for (int h = 0; h < G; ++h) {
            bh[h] = wp[(2 * h) * wl];
            bl[h] = wp[(2 * h + 1) * wl];
          }
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            uint32_t x0[4], x1[4];
            row_bytes<BITS>(lds_row<BITS>(tile + row_off[mt][0]), x0);
            row_bytes<BITS>(lds_row<BITS>(tile + row_off[mt][1]), x1);
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
      release(slot);
    }
    if (r > kGroupR) flush_group(1);
    stamp(1);
#ifdef DQ_ATTN_NULL_STREAM  // measurement only: the producer / ring / scheduler alone
    begin_phase(2 * j + 1);
    for (int vs = 0; vs < nbt * d.nslices; ++vs, ++st) release(acquire());
    team_sync(team);
    if (tid == 0) {
      const int jn = j + 1;
      if constexpr (INW) {
        mbar_arrive(&tm.wfree);
        mbar_wait(&tm.g0bar, (uint32_t)(j & 1));
      }
      mbar_wait(&tm.descfull[jn % kSubRing], (uint32_t)((jn / kSubRing) & 1));
      if (tm.sub[jn % kSubRing].nbt > 0) {
        if constexpr (INW) issue_g0v16(tm, tm.sub[jn % kSubRing]);
        else issue_wimg(tm, args, tm.sub[jn % kSubRing]);
      }
    }
    continue;
#endif

    // ---- phase 2: softmax of the sub-item straight from the accumulators --------------
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
          const bool ok = (a < i1) && (wb0 + bl < i2) && (jt < nbt);
          sv[mt][h][k] = ok ? sacc[mt][h][k] : -INFINITY;
          m = fmaxf(m, sv[mt][h][k]);
        }
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) tm.rowmax[h][warp] = m;
    }
    team_sync(team);  // every warp is past phase 1: the W buffer is dead
    if (INW && tid == 0) mbar_arrive(&tm.wfree);  // the fetcher may write the next item's W image
    if (!INW && lane == 0 && warp < i1) {  // prefetch the fp32 G0v for the epilogue into it (+ the V channel table)
      // one copy per a, issued by warp a, into blocks of 2r + 1 float4s: the epilogue's lanes
      // tid4 = 0..3 read a = 2 tid4 + aa, and the pad puts their blocks 32 bytes apart in the
      // banks (an unpadded 2r-float4 stride maps all four onto the same banks: a 4-way
      // conflict per load, 10 us of a C2 layer).  A copy completing before warp 0's expect_tx
      // only takes the transaction count negative; the phase needs that arrival.
      const uint32_t cb = ASYM ? (uint32_t)(2 * r * 16 * 4) : 0u;
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      if (warp == 0) {
        mbar_expect_tx(&tm.g0bar, (uint32_t)(i1 * r * 32) + cb);
        if (ASYM) bulk_g2s(tm.vch, args.segs[d.seg].v_ch, cb, &tm.g0bar);
      }
      bulk_g2s(tm.wg.g0v + warp * (2 * r + 1), reinterpret_cast<const float4*>(d.vg0) + warp * 2 * r,
               (uint32_t)(r * 32), &tm.g0bar);
    }
    unsigned char* pb = reinterpret_cast<unsigned char*>(tm.pr.p);
    // P = exp2(s - m) in fixed point with one scale per (h, a, 64-row tile), set by that
    // tile's largest probability: small probabilities far from the peak keep their
    // relative precision (the V side combines its accumulators per tile anyway)
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float m = tm.rowmax[h][0];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) m = fmaxf(m, tm.rowmax[h][w]);
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
      for (int q = 0; q < 2; ++q) {
        float v = tmax[q];
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
        if (gid == 0 && jt < nbt) atomicMax(&tm.pmax[h][2 * tid4 + q][jt], __float_as_uint(v));
      }
    }
    team_sync(team);  // per-tile probability maxima complete
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float lsum = 0.f;
      int gsum[2] = {0, 0};  // per a of this thread (a = 2*tid4, 2*tid4+1), this warp's tile
      float pq[2], pinv[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float pm = __uint_as_float(tm.pmax[h][2 * tid4 + q][min(jt, NT - 1)]);
        pq[q] = pow2_sub_exp(pm, kPBits<BITS>);
        pinv[q] = pow2_exp_sub(pm, kPBits<BITS>);
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
          if (jt < nbt) {
            const int pos = inv_ord16<BITS>(bl & 15);
            pb[p_chunk<NT>(h, 0, a, bl >> 4) * 16 + pos] = (unsigned char)(pint >> 8);
            pb[p_chunk<NT>(h, 1, a, bl >> 4) * 16 + pos] = (unsigned char)(pint & 0xFF);
          }
        }
      // per (a, tile) sums: reduce over the 8 gid lanes sharing tid4 (same a, same tile)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        int v = gsum[q];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        // gamma = X sum_b Pint (symmetric), sum_b Pint (asymmetric: the zero point is per channel)
        if (X && gid == 0 && jt < nbt) atomicAdd(&tm.gamma[h][2 * tid4 + q][jt], ASYM ? v : X * v);
      }
      for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
      if (lane == 0) tm.lsum[h][warp] = lsum;
    }
    team_sync(team);  // P limbs, gamma and lsum complete
    begin_phase(2 * j + 1);
    stamp(2);

    // ---- phase 3: Y = codes_v . P^T on the int8 tensor pipe ----------------------------
    // warp w owns bond rows w*rw .. w*rw+rw-1 (an m-tile = one bond row x 16 e)
    const int rw = r / kWarps;
    const int kslice = kWarps / d.nslices;
    const int my_slice = warp / kslice;
    const int rbase_in_slice = (warp % kslice) * rw;
    constexpr int kRw = kMaxR / kWarps;  // bond rows per warp at r = 64
    float accv[kRw][G][4];
#pragma unroll
    for (int t = 0; t < kRw; ++t)
#pragma unroll
      for (int h = 0; h < G; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) accv[t][h][k] = 0.f;
    const int nV = nbt * d.nslices;
    if (ASYM) mbar_wait(&tm.g0bar, (uint32_t)(j & 1));  // the V zero points seed the accumulators
    for (int vs = 0, btl = 0, sl = 0; vs < nV; ++vs, ++st) {
      const int slot = acquire();
#ifdef DQ_ATTN_NULL_CONSUMER
      if (++sl == d.nslices) sl = 0, ++btl;
      release(slot);
      continue;
#endif
      if (sl == my_slice) {
        uint4 ph[G], pl_[G];
        int gam[G][2];
        float pinv[G][2];
#pragma unroll
        for (int h = 0; h < G; ++h) {
          ph[h] = tm.pr.p[p_chunk<NT>(h, 0, gid, btl * 4 + tid4)];
          pl_[h] = tm.pr.p[p_chunk<NT>(h, 1, gid, btl * 4 + tid4)];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            gam[h][q] = tm.gamma[h][2 * tid4 + q][btl];
            pinv[h][q] = pow2_exp_sub(__uint_as_float(tm.pmax[h][2 * tid4 + q][btl]), kPBits<BITS>);
          }
        }
        const unsigned char* buf = sm.ring[slot];
#pragma unroll
        for (int t = 0; t < kRw; ++t) {
          if (t < rw) {
            const int rl = rbase_in_slice + t;
            uint32_t x0[4], x1[4];
            row_bytes<BITS>(lds_row<BITS>(buf + (rl * 16 + gid) * 8 * BITS + RB * tid4), x0);
            row_bytes<BITS>(lds_row<BITS>(buf + (rl * 16 + gid + 8) * 8 * BITS + RB * tid4), x1);
            int z0 = 1, z1 = 1;  // asymmetric: zero points of (bond row, e = gid / gid + 8)
            if (ASYM) {
              const int rr = warp * rw + t;
              z0 = (int)tm.vch[r * 16 + rr * 16 + gid];  // zero points follow the scales
              z1 = (int)tm.vch[r * 16 + rr * 16 + gid + 8];
            }
#pragma unroll
            for (int h = 0; h < G; ++h) {
              // the excess (or zero-point) correction seeds the low-limb accumulator
              int yh[4] = {0, 0, 0, 0};
              int yl[4] = {-z0 * gam[h][0], -z0 * gam[h][1], -z1 * gam[h][0], -z1 * gam[h][1]};
              imma<SA, false>(yh, x0[0], x1[0], x0[1], x1[1], ph[h].x, ph[h].y);
              imma<SA, false>(yl, x0[0], x1[0], x0[1], x1[1], pl_[h].x, pl_[h].y);
              imma<SA, false>(yh, x0[2], x1[2], x0[3], x1[3], ph[h].z, ph[h].w);
              imma<SA, false>(yl, x0[2], x1[2], x0[3], x1[3], pl_[h].z, pl_[h].w);
#pragma unroll
              for (int k = 0; k < 4; k += 2)
                ffma2(accv[t][h][k], accv[t][h][k + 1], (float)(256 * yh[k] + yl[k]),
                      (float)(256 * yh[k + 1] + yl[k + 1]), pinv[h][0], pinv[h][1]);
            }
          }
        }
      }
      release(slot);
      if (++sl == d.nslices) sl = 0, ++btl;
    }

    stamp(3);
    // ---- phase 4: O = scale_v * G0v . Y on CUDA cores, reduce, write the partial -------
    // accv[t][h]: rows e = gid (k 0,1) / gid+8 (k 2,3); cols a = 2*tid4 + (k & 1)
    float part[G][16];  // [h][c*2 + (e == gid+8)]
#pragma unroll
    for (int h = 0; h < G; ++h)
#pragma unroll
      for (int k = 0; k < 16; ++k) part[h][k] = 0.f;
    mbar_wait(&tm.g0bar, (uint32_t)(j & 1));  // G0v [a][rr][c] (normalised): fp32 in the W buffer, or fp16 (kInW)
    const float4* g0v = tm.wg.g0v;
#ifdef DQ_ATTN_NULL_FOLD  // measurement only: no G0v fold (wrong results), Y still consumed
#pragma unroll
    for (int t = 0; t < kRw; ++t)
#pragma unroll
      for (int h = 0; h < G; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) part[h][(t * 4 + k) & 15] += accv[t][h][k];
    if (tid < 0)
#endif
#pragma unroll
    for (int t = 0; t < kRw; ++t) {
      if (t < rw) {
        const int rr = warp * rw + t;
        // asymmetric: the per-(bond row, e) channel scales of V
        const float s0 = ASYM ? tm.vch[rr * 16 + gid] : 1.f, s1 = ASYM ? tm.vch[rr * 16 + gid + 8] : 1.f;
#pragma unroll
        for (int aa = 0; aa < 2; ++aa) {
          const int a = 2 * tid4 + aa;
          if (a < i1) {
            float gc[8];
            if constexpr (INW) {
              const uint4 gh = tm.g0v16[a * (r + 1) + rr];
              const float2 g01 = __half22float2(*reinterpret_cast<const __half2*>(&gh.x));
              const float2 g23 = __half22float2(*reinterpret_cast<const __half2*>(&gh.y));
              const float2 g45 = __half22float2(*reinterpret_cast<const __half2*>(&gh.z));
              const float2 g67 = __half22float2(*reinterpret_cast<const __half2*>(&gh.w));
              gc[0] = g01.x, gc[1] = g01.y, gc[2] = g23.x, gc[3] = g23.y;
              gc[4] = g45.x, gc[5] = g45.y, gc[6] = g67.x, gc[7] = g67.y;
            } else {
              const float4 g_lo = g0v[a * (2 * r + 1) + 2 * rr], g_hi = g0v[a * (2 * r + 1) + 2 * rr + 1];
              gc[0] = g_lo.x, gc[1] = g_lo.y, gc[2] = g_lo.z, gc[3] = g_lo.w;
              gc[4] = g_hi.x, gc[5] = g_hi.y, gc[6] = g_hi.z, gc[7] = g_hi.w;
            }
#pragma unroll
            for (int h = 0; h < G; ++h) {
              const float y0 = ASYM ? accv[t][h][aa] * s0 : accv[t][h][aa];
              const float y1 = ASYM ? accv[t][h][2 + aa] * s1 : accv[t][h][2 + aa];
#pragma unroll
              for (int c = 0; c < 8; ++c) ffma2(part[h][2 * c], part[h][2 * c + 1], gc[c], gc[c], y0, y1);
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
    team_sync(team);  // every warp is past the V stages and G0v: P and W/G0v buffers are free
    if (tid == 0) {
      const int jn = j + 1;
      mbar_wait(&tm.descfull[jn % kSubRing], (uint32_t)((jn / kSubRing) & 1));
      if (tm.sub[jn % kSubRing].nbt > 0) {
        if constexpr (INW) issue_g0v16(tm, tm.sub[jn % kSubRing]);  // the fetcher writes W
        else issue_wimg(tm, args, tm.sub[jn % kSubRing]);
      }
    }
    if (tid < G * 8 * NT) {
      (&tm.gamma[0][0][0])[tid] = 0;
      (&tm.pmax[0][0][0])[tid] = 0u;
    }
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
        tm.pr.red[warp][h][c * 16 + gid] = v0;
        tm.pr.red[warp][h][c * 16 + gid + 8] = v1;
      }
    team_sync(team);
    for (int i = tid; i < G * kD; i += kThreads) {
      const int h = i / kD, dd = i % kD;
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) v += tm.pr.red[w][h][dd];
      args.part_o[((size_t)d.part * G + h) * kD + dd] = v * d.vscale;
    }
    if (tid < G) {
      float l = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) l += tm.lsum[tid][w];
      args.part_ml[((size_t)d.part * G + tid) * 2 + 0] = mh[tid];  // log2 domain
      args.part_ml[((size_t)d.part * G + tid) * 2 + 1] = l;
    }
    stamp(4);
  }
}

}  // namespace attn
}  // namespace dq

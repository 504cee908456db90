// K5: fused DecoQuant dequantisation + decode attention for D = 128 (j = (8,16)).
//
// Reference semantics (kvcache.py:188-217 scores, compress.py:159-231 fused reads):
// for one unit (sequence, kv head) with segments of T_s tokens (plan i=(i1,i2),
// bond r) and g query rows q[h] (GQA group), the output is
//     softmax_t(q.K^T * sm_scale) V        over all segments and the fp16 tail,
// with K[a*i2+b, c*16+e] = sum_r G0k[a,c,r] * scale_k * code_k[r,b,e] (same for V).
//
// Factored order: per segment
//   W[h,a,r,e] = sum_c q[h,c*16+e] G0k[a,c,r]                  (CUDA cores, per CTA)
//   S[h,a,b]   = scale_k * sum_{r,e} W[h,a,r,e] code_k[r,b,e]   (int8 tensor cores)
//   P          = exp(S*sm_scale - m)                           (split-T softmax)
//   Y[h,a,r,e] = sum_b P[h,a,b] code_v[r,b,e]                  (int8 tensor cores)
//   O[h,c,e]   = scale_v * sum_{a,r} G0v[a,c,r] Y[h,a,r,e]     (CUDA cores, epilogue)
//
// Data movement (path 0, attn_kernel.cuh): a persistent grid of (SMs x resident CTAs) CTAs
// draws work items (<= 256 rows of one segment, or 512 for g = 1 with 2- / 4-bit codes;
// dq_attention_plan; one partial each) from a self-resetting ticket counter.  A producer
// warp streams the packed K codes (DQ_LAYOUT_KTILE) and V codes (DQ_LAYOUT_VTILE) through a
// 5-stage x 16 KB shared-memory ring by cp.async.bulk (TMA bulk copies completing on
// mbarriers), running ahead across item boundaries (2 CTAs/SM -> 160 KB in flight per SM).
// Eight consumer warps read bank-conflict-free fragments (K tile rows are XOR-swizzled by r
// in HBM) and widen codes to bytes (int4: one AND per 4 even codes, one SHF+AND per 4 odd
// codes).  The codes multiply fixed-point W and P split into two 8-bit limbs (hi*256 + lo) on
// the int8 tensor pipe (mma.sync m16n8k32, exact s32 accumulation); the excess-code offset is
// removed exactly in integers.  The reduction index is permuted identically on both
// operands, which is free.  Full-precision K/V never exist anywhere.  Paths 1 and 2
// (attn_tc.cuh, attn_gqa.cuh) run the same contractions as tcgen05 UMMAs with TMEM
// accumulators.  The prepare (W image), split and combine kernels are chained with
// programmatic dependent launch.
#include "attn_gqa.cuh"
#include "attn_combine.cuh"

#include <algorithm>
#include <vector>

namespace dq {

namespace {

using namespace attn;

// ---- combine: one CTA per kv head unit; see attn_combine.cuh --------------------------
// Launched with programmatic dependent launch behind the split kernel.  Everything before
// griddepcontrol.wait overlaps the split kernel: this grid is scheduled only once the split
// kernel has passed its own wait, so the prepare kernel, the producers of q and every earlier
// step have completed; the dense fp16 tail (written by earlier steps) is read here, the split
// kernel's partials only after the wait.
constexpr int kCombineThreads = 256;

template <int G>
__global__ void __launch_bounds__(kCombineThreads) combine_kernel(dq_attn_args args) {
  extern __shared__ float tail_s[];  // [tail_cap]
  __shared__ __align__(16) float red[(kCombineThreads / 32) * 130];
  const int u = blockIdx.x, d = threadIdx.x;
  const int hg = args.head_groups > 1 ? args.head_groups : 1;
  auto sync = [] { __syncthreads(); };
  if (G == 1 && hg == 1) {  // tail partial first (overlapping the split kernel), then the merge
    const int tl = args.tail_len ? args.tail_len[u] : 0;
    float Mt = -INFINITY, Lt = 0.f, Ot = 0.f;
    if (tl > 0) tail_partial<1>(args, u, u, 0, d, kCombineThreads, tl, tail_s, red, sync, Mt, Lt, Ot);
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    merge_head<1>(args, u, 0, d, Mt, Lt, Ot);
    if (args.app_k) {
      sync();
      combine_append(args, u, d, tl);
    }
    return;
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  combine_unit<G>(args, u, d, kCombineThreads, tail_s, red, sync);
}

// combine for the GQA kernel's 8 heads: one 128-thread group per head (named barrier 1 + group);
// the tail partials overlap the split kernel (see combine_kernel), the merges follow its wait
// and the fused append comes once every group has read the tail
#ifndef DQ_COMB_GQ_MINB
#define DQ_COMB_GQ_MINB 2
#endif
__global__ void __launch_bounds__(kGqG * 128, DQ_COMB_GQ_MINB) combine_gqa_kernel(dq_attn_args args) {
  extern __shared__ float tail_sg[];  // [kGqG][tail_cap]
  __shared__ __align__(16) float red[kGqG][4 * 130];
  const int u = blockIdx.x, grp = threadIdx.x >> 7, d = threadIdx.x & 127;
  const int hg = args.head_groups > 1 ? args.head_groups : 1;
  const int tl = args.tail_len ? args.tail_len[u] : 0;
  const int cap = args.tail_cap > 0 ? args.tail_cap : 1;
  auto gsync = [grp] { asm volatile("bar.sync %0, 128;\n" ::"r"(1 + grp) : "memory"); };
  if (hg == 1) {
    float Mt = -INFINITY, Lt = 0.f, Ot = 0.f;
    if (tl > 0) {  // the whole tail partial with K / V rows shared by the heads (tail_gq)
      __shared__ __align__(16) float qs[kGqG][128];
      __shared__ float gred[kGqG][8];
      tail_gq<kGqG * 128>(args, u, tl, cap, tail_sg, qs, &red[0][0], gred[grp], gsync, Mt, Lt, Ot);
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    merge_head<kGqG>(args, u, grp, d, Mt, Lt, Ot);
  } else {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    for (int vv = 0; vv < hg; ++vv)
      combine_head<kGqG>(args, u, u * hg + vv, grp, d, 128, tl, tail_sg + (size_t)grp * cap, red[grp], gsync);
  }
  if (args.app_k) {
    __syncthreads();  // every group has read tail_len[u] and the tail
    if (grp == 0) combine_append(args, u, d, tl);
  }
}

__global__ void tail_append_kernel(const __half* __restrict__ k_rows, const __half* __restrict__ v_rows,
                                   __half* __restrict__ tail_k, __half* __restrict__ tail_v, int32_t* tail_len,
                                   int tail_cap) {
  const int u = blockIdx.x;
  const int pos = tail_len[u];
  if (pos < tail_cap) {
    tail_k[((size_t)u * tail_cap + pos) * kD + threadIdx.x] = k_rows[(size_t)u * kD + threadIdx.x];
    tail_v[((size_t)u * tail_cap + pos) * kD + threadIdx.x] = v_rows[(size_t)u * kD + threadIdx.x];
  }
  __syncthreads();
  if (threadIdx.x == 0) tail_len[u] = pos + 1;
}


// consumer teams of the mma.sync split kernel: 1 = two CTAs per SM, each a FIFO ring (the default:
// C2 62.5 us per layer); 2 = one CTA per SM, two teams sharing a slot pool (DQ_ATTN_TEAMS_G1=2,
// g = 1 only: measured 69 us)
#ifndef DQ_ATTN_TEAMS_G1
#define DQ_ATTN_TEAMS_G1 1
#endif
template <int G>
constexpr int kTeamsOf = G == 1 ? DQ_ATTN_TEAMS_G1 : 1;

// the split kernel computes the W image itself (no prepare kernel) and folds an fp16 G0v
bool in_kernel_w(int g, int path, int asym, int chunk_b) {
  return DQ_INKERNEL_W && path == 0 && g == 1 && !asym && kTeamsOf<1> == 1 && chunk_b <= kCB;
}

template <int BITS, int G, int NT = kTiles, bool ASYM = false>
int set_attrs() {
  constexpr int T = kTeamsOf<G>;
  static bool attr = false;
  if (!attr) {
    const int smem = (int)sizeof(AttnSmem<G, NT, ASYM, T>);
    DQ_CUDA_TRY(cudaFuncSetAttribute(decode_attn_kernel<BITS, G, NT, ASYM, T>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    DQ_CUDA_TRY(cudaFuncSetAttribute(decode_attn_kernel<BITS, G, NT, ASYM, T>,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    attr = true;
  }
  return DQ_OK;
}

// launch the mma.sync split kernel instance (BITS, G, NT, ASYM) with its team count
template <int BITS, int G, int NT, bool ASYM>
int launch_split(cudaLaunchConfig_t cfg, const dq_attn_args& a) {
  constexpr int T = kTeamsOf<G>;
  const int rc = set_attrs<BITS, G, NT, ASYM>();
  if (rc != DQ_OK) return rc;
  cfg.blockDim = dim3(kCtaThreadsOf<T>);
  cfg.dynamicSmemBytes = sizeof(AttnSmem<G, NT, ASYM, T>);
  DQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, decode_attn_kernel<BITS, G, NT, ASYM, T>, a));
  return DQ_OK;
}

template <int BITS, int G>
int occupancy(int* per_sm) {
  constexpr int T = kTeamsOf<G>;
  const int rc = set_attrs<BITS, G>();
  if (rc != DQ_OK) return rc;
  DQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, decode_attn_kernel<BITS, G, kTiles, false, T>,
                                                            kCtaThreadsOf<T>, sizeof(AttnSmem<G, kTiles, false, T>)));
  return DQ_OK;
}

// one CTA per SM: the tcgen05 kernels allocate all 512 TMEM columns
template <class Kernel>
int launch_tc(Kernel kernel, size_t smem, int threads, const dq_attn_args& a, cudaStream_t s) {
  int sms = 0, dev = 0;
  DQ_CUDA_TRY(cudaGetDevice(&dev));
  DQ_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.nwork < sms ? a.nwork : sms));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = (a.phases & 8) ? 0 : 1;  // phases bit 3: no PDL edge (back-to-back timing)
  DQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, a));
  return DQ_OK;
}

template <int BITS, int G>
int launch_attn(const dq_attn_args& a, cudaStream_t s) {
  if constexpr (G <= 2) {
    const int rc = set_attrs<BITS, G>();
    if (rc != DQ_OK) return rc;
  } else {
    if (a.path != 2 || BITS != 4) return fail(DQ_ERR_UNSUPPORTED, "g = %d runs on the tcgen05 GQA path (4-bit codes)", G);
  }
  const int phases = a.phases ? a.phases : 7;
  if (a.nwork > 0 && (phases & 5)) {
    if (!a.wimg || a.wimg_stride < kWImageBytes<G>) return fail(DQ_ERR_INVALID_ARG, "W image workspace too small");
  }
  if (a.nseg > 0 && a.nwork > 0 && (phases & 4) && a.path == 2) {
    if constexpr (BITS == 4 && G == kGqG) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)a.nseg);
      cfg.blockDim = dim3(kPrepGqThreads);
      cfg.stream = s;
      cudaLaunchAttribute attr_pdl[1];
      attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr_pdl;
      cfg.numAttrs = 1;
      DQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn_prepare_gqa_kernel, a));
    }
  } else if (a.nseg > 0 && a.nwork > 0 && (phases & 4) && !in_kernel_w(G, a.path, a.asym, a.chunk_b)) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)a.nseg, kPrepSplit);
    cfg.blockDim = dim3(kPrepThreadsOf<G>);
    cfg.stream = s;
    cudaLaunchAttribute attr_pdl[1];
    attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr_pdl;
    cfg.numAttrs = 1;
    if (a.asym) {
      if constexpr (BITS <= 4 && G <= 2) DQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn_prepare_kernel<BITS, G, true>, a));
    } else {
      DQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn_prepare_kernel<BITS, G>, a));
    }
  }
  if (a.path == 1 && a.nwork > 0 && (phases & 1)) {
    if constexpr (BITS == 4 && G == 1) {
      static bool tc_attr = false;
      if (!tc_attr) {
        DQ_CUDA_TRY(cudaFuncSetAttribute(decode_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(TcSmem)));
        tc_attr = true;
      }
      const int rc = launch_tc(decode_attn_tc_kernel, sizeof(TcSmem), kTcThreads, a, s);
      if (rc != DQ_OK) return rc;
    } else {
      return fail(DQ_ERR_UNSUPPORTED, "the tcgen05 path 1 covers 4-bit codes with g = 1");
    }
  } else if (a.path == 2 && a.nwork > 0 && (phases & 1)) {
    if constexpr (BITS == 4 && G == kGqG) {
      static bool gq_attr = false;
      if (!gq_attr) {
        DQ_CUDA_TRY(cudaFuncSetAttribute(decode_attn_gqa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(GqSmem)));
        gq_attr = true;
      }
      const int rc = launch_tc(decode_attn_gqa_kernel, sizeof(GqSmem), kGqThreads, a, s);
      if (rc != DQ_OK) return rc;
    } else {
      return fail(DQ_ERR_UNSUPPORTED, "the tcgen05 GQA path covers 4-bit codes with g = 8");
    }
  } else if (a.nwork > 0 && (phases & 1)) {
    if constexpr (G <= 2) {
      // programmatic dependent launch: the split kernel's prologue and first code copies
      // overlap the prepare kernel; it waits (griddepcontrol.wait) only for the W images
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(a.nctas > 0 && a.nctas < a.nwork ? a.nctas : a.nwork));
      cfg.stream = s;
      cudaLaunchAttribute attr_pdl[1];
      attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr_pdl;
      cfg.numAttrs = (phases & 8) ? 0 : 1;  // bit 3: no PDL edge (back-to-back timing of the split kernel)
      if (a.asym && BITS == 8) return fail(DQ_ERR_UNSUPPORTED, "the asymmetric mode covers 2- and 4-bit codes");
      int rc = DQ_OK;
      if (a.chunk_b > kCB) {  // 8-tile work items (g = 1, 2- and 4-bit codes)
        if constexpr (G == 1 && BITS <= 4) {
          rc = a.asym ? launch_split<BITS, G, 2 * kTiles, true>(cfg, a) : launch_split<BITS, G, 2 * kTiles, false>(cfg, a);
        } else {
          return fail(DQ_ERR_UNSUPPORTED, "work items of more than %d rows need g = 1 and 2- or 4-bit codes", kCB);
        }
      } else if (a.asym) {
        if constexpr (BITS <= 4) rc = launch_split<BITS, G, kTiles, true>(cfg, a);
      } else {
        rc = launch_split<BITS, G, kTiles, false>(cfg, a);
      }
      if (rc != DQ_OK) return rc;
    }
  }
  if (phases & 2) {
    const bool gq = G == kGqG;  // one 128-thread group per head
    const size_t csmem = sizeof(float) * (a.tail_cap > 0 ? a.tail_cap : 1) * (gq ? kGqG : 1);
    const int hg = a.head_groups > 1 ? a.head_groups : 1;
    if (gq) {  // static reduction buffers + 8 tail buffers exceed the default 48 KB
      static bool cg_attr = false;
      if (!cg_attr) {
        DQ_CUDA_TRY(cudaFuncSetAttribute(combine_gqa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        cg_attr = true;
      }
      if (csmem > 160 * 1024) return fail(DQ_ERR_UNSUPPORTED, "tail capacity %d too large for the GQA combine", a.tail_cap);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.units / hg));
    cfg.blockDim = dim3(gq ? kGqG * 128 : kCombineThreads);
    cfg.dynamicSmemBytes = csmem;
    cfg.stream = s;
    cudaLaunchAttribute attr_pdl[1];
    attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr_pdl;
    // the combine reads q and the tail before its griddepcontrol.wait, which is safe only behind
    // the split kernel (it triggers after its own wait); with no split kernel in front (a
    // tail-only layer, or a combine-only launch) the predecessor may be q's producer: no PDL edge
    cfg.numAttrs = (a.nwork > 0 && (phases & 1)) ? 1 : 0;
    if (gq) {
      DQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, combine_gqa_kernel, a));
    } else {
      DQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, combine_kernel<G>, a));
    }
  }
  return DQ_OK;
}

template <int BITS>
int dispatch_g(const dq_attn_args& a, cudaStream_t s) {
  if (a.asym && a.path != 0) return fail(DQ_ERR_UNSUPPORTED, "the asymmetric mode runs on the mma.sync split kernel");
  if (a.chunk_b <= 0 || a.chunk_b > 2 * kCB || a.chunk_b % kI2Pad || (a.chunk_b > kCB && a.path != 0))
    return fail(DQ_ERR_UNSUPPORTED, "chunk_b must be a multiple of %d in %d..%d (%d off path 0; got %d)", kI2Pad, kI2Pad,
                2 * kCB, kCB, a.chunk_b);
  switch (a.g) {
    case 1: return launch_attn<BITS, 1>(a, s);
    case 2: return launch_attn<BITS, 2>(a, s);
    case kGqG: return launch_attn<BITS, kGqG>(a, s);
  }
  return fail(DQ_ERR_UNSUPPORTED, "g must be 1, 2 or %d in this build (got %d)", kGqG, a.g);
}

}  // namespace

}  // namespace dq


using namespace dq;

extern "C" int dq_attention_plan(const dq_segment* segs, int32_t nseg, int32_t units, int32_t chunk_b, int32_t max_work,
                                 int32_t* work, int32_t* nwork, int32_t* work_part, int32_t* unit_part0,
                                 int32_t* unit_nparts, int32_t* total_parts) {
  if (nseg < 0 || units < 0 || chunk_b <= 0 || chunk_b % kI2Pad) return fail(DQ_ERR_INVALID_ARG, "bad plan arguments");
  if (!nwork || !total_parts || !unit_part0 || !unit_nparts) return fail(DQ_ERR_INVALID_ARG, "null output");
  const int maxt = chunk_b / kI2Pad;
  for (int u = 0; u < units; ++u) unit_nparts[u] = 0;
  int n = 0;
  for (int s = 0; s < nseg; ++s) {
    const dq_segment& g = segs[s];
    if (g.unit < 0 || g.unit >= units) return fail(DQ_ERR_INVALID_ARG, "segment %d has unit %d", s, g.unit);
    if (g.r > kMaxR || g.r % 8 || g.i1 > 8 || g.i2p % kI2Pad || g.i2p < g.i2)
      return fail(DQ_ERR_UNSUPPORTED, "segment %d plan unsupported", s);
    // ceil(tiles / maxt) near-equal items per segment
    const int nt = (g.i2 + kI2Pad - 1) / kI2Pad, k = (nt + maxt - 1) / maxt;
    for (int i = 0, t = 0; i < k; ++i) {
      const int len = nt / k + (i < nt % k ? 1 : 0);
      if (work) {
        if (n >= max_work) return fail(DQ_ERR_INVALID_ARG, "work list exceeds max_work = %d", max_work);
        work[3 * n] = s;
        work[3 * n + 1] = t * kI2Pad;
        work[3 * n + 2] = len;
      }
      unit_nparts[g.unit]++;
      ++n;
      t += len;
    }
  }
  int acc = 0;
  for (int u = 0; u < units; ++u) {
    unit_part0[u] = acc;
    acc += unit_nparts[u];
  }
  if (work && work_part) {
    // partial slots per unit, in work-list order
    std::vector<int> cursor(unit_part0, unit_part0 + units);
    for (int i = 0; i < n; ++i) work_part[i] = cursor[segs[work[3 * i]].unit]++;
  }
  *nwork = n;
  *total_parts = acc;
  return DQ_OK;
}

extern "C" int dq_attention_ctas(int32_t g, int32_t bits, int32_t* ctas) {
  if (!ctas) return fail(DQ_ERR_INVALID_ARG, "null output");
  int dev = 0, sms = 0, per_sm = 0;
  DQ_CUDA_TRY(cudaGetDevice(&dev));
  DQ_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int rc = DQ_OK;
  switch (bits * 16 + g) {
    case 2 * 16 + 1: rc = occupancy<2, 1>(&per_sm); break;
    case 2 * 16 + 2: rc = occupancy<2, 2>(&per_sm); break;
    case 4 * 16 + 1: rc = occupancy<4, 1>(&per_sm); break;
    case 4 * 16 + 2: rc = occupancy<4, 2>(&per_sm); break;
    case 8 * 16 + 1: rc = occupancy<8, 1>(&per_sm); break;
    case 8 * 16 + 2: rc = occupancy<8, 2>(&per_sm); break;
    case 4 * 16 + kGqG: per_sm = 1; break;  // the tcgen05 GQA kernel: one CTA per SM
    default: return fail(DQ_ERR_UNSUPPORTED, "no split kernel for bits %d, g %d", bits, g);
  }
  if (rc != DQ_OK) return rc;
  *ctas = sms * per_sm;
  return DQ_OK;
}

extern "C" int dq_attention_g0v_dtype(int32_t g, int32_t path, int32_t asym, int32_t chunk_b, int32_t* dtype) {
  if (!dtype) return fail(DQ_ERR_INVALID_ARG, "null output");
  *dtype = in_kernel_w(g, path, asym, chunk_b) ? DQ_F16 : DQ_F32;
  return DQ_OK;
}

extern "C" int dq_attention_wimg_bytes(int32_t g, int64_t* bytes) {
  if (!bytes) return fail(DQ_ERR_INVALID_ARG, "null output");
  if (g == 1) *bytes = kWImageBytes<1>;
  else if (g == 2) *bytes = kWImageBytes<2>;
  else if (g == kGqG) *bytes = kWImageBytes<kGqG>;
  else return fail(DQ_ERR_UNSUPPORTED, "g must be 1, 2 or %d in this build (got %d)", kGqG, g);
  return DQ_OK;
}

extern "C" int dq_decode_attention(const dq_attn_args* h, void* stream) {
  if (!h) return fail(DQ_ERR_INVALID_ARG, "null args");
  const dq_attn_args& a = *h;
  if (a.units <= 0) return DQ_OK;
  if (!a.q || !a.out ||
      (a.nwork > 0 && (!a.segs || !a.work || !a.work_part || !a.sched || !a.part_o || !a.part_ml)))
    return fail(DQ_ERR_INVALID_ARG, "dq_decode_attention: null pointer");
  if (!a.unit_part0 || !a.unit_nparts) return fail(DQ_ERR_INVALID_ARG, "dq_decode_attention: missing unit tables");
  if (a.head_groups > 1 && a.units % a.head_groups)
    return fail(DQ_ERR_INVALID_ARG, "dq_decode_attention: units (%d) not a multiple of head_groups (%d)", a.units,
                a.head_groups);
  if (a.app_k && (!a.app_v || !a.tail_k || !a.tail_v || !a.tail_len || a.tail_cap <= 0))
    return fail(DQ_ERR_INVALID_ARG, "dq_decode_attention: append needs app_v and the tail buffers");
  cudaStream_t s = (cudaStream_t)stream;
  switch (a.bits) {
    case 2: return dispatch_g<2>(a, s);
    case 4: return dispatch_g<4>(a, s);
    case 8: return dispatch_g<8>(a, s);
  }
  return fail(DQ_ERR_UNSUPPORTED_BITS, "bits must be one of (2, 4, 8), got %d", a.bits);
}

extern "C" int dq_tail_append(const uint16_t* k_rows, const uint16_t* v_rows, int32_t units, uint16_t* tail_k,
                              uint16_t* tail_v, int32_t* tail_len, int32_t tail_cap, void* stream) {
  if (units <= 0) return DQ_OK;
  if (!k_rows || !v_rows || !tail_k || !tail_v || !tail_len) return fail(DQ_ERR_INVALID_ARG, "null pointer");
  tail_append_kernel<<<units, kD, 0, (cudaStream_t)stream>>>((const __half*)k_rows, (const __half*)v_rows,
                                                            (__half*)tail_k, (__half*)tail_v, tail_len, tail_cap);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

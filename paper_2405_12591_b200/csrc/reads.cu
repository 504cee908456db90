// K4 reconstruct, the generic fused reads, layout conversion and small helpers.
//
//   reconstruct  : compress.py:105-107 -> mpo.py:181-198   (dequantize, contract, de-interleave)
//   fused_matmul_t: compress.py:195-231   x @ W^T without materialising W
//   fused_matmul : compress.py:159-192   x @ W   without materialising W
//
// These serve the reference-mirroring API for any n=2 plan.  The decode hot path
// uses the specialised D=128 kernel in attention.cu instead.
#include <algorithm>

#include "common.cuh"

namespace dq {

namespace {

constexpr int kThreads = 256;

// ---- K4: out[a*i2+b, c*j2+e] = sum_r core0[a,c,r] * f32(code[r,b,e]) * scale ----
// grid (nblk, b-tiles of kBT rows).  The dequantized codes of the b-tile and the
// whole core0 are staged in shared memory; each thread produces output elements
// with consecutive (c,e) so the stores are coalesced.
constexpr int kBT = 8;

__global__ void __launch_bounds__(kThreads) reconstruct_kernel(const float* __restrict__ core0,
                                                               const uint8_t* __restrict__ payload,
                                                               int64_t payload_stride, CoreGeom geom,
                                                               const float* __restrict__ scale, int i1, int j1,
                                                               int cols, void* __restrict__ out, int out_dtype) {
  extern __shared__ float smem[];
  const int r = geom.r, i2 = geom.i2, j2 = geom.j2;
  const int m = i1 * j1;
  float* g0 = smem;               // [m][r]
  float* dq = smem + m * r;       // [r][kBT][j2]
  const int64_t blk = blockIdx.x;
  const int b0 = blockIdx.y * kBT;
  const int nb = min(kBT, i2 - b0);
  const float s = scale[blk];
  const float* c0 = core0 + blk * (int64_t)m * r;
  const uint8_t* pl = payload + blk * payload_stride;
  for (int i = threadIdx.x; i < m * r; i += kThreads) g0[i] = c0[i];
  for (int i = threadIdx.x; i < r * kBT * j2; i += kThreads) {
    const int rr = i / (kBT * j2), rem = i - rr * kBT * j2;
    const int bb = rem / j2, e = rem - bb * j2;
    float v = 0.f;
    if (bb < nb) v = __fmul_rn((float)geom_read(pl, geom, rr, b0 + bb, e), s);
    dq[i] = v;
  }
  __syncthreads();
  const int rows_per_tile = i1 * nb;
  const int64_t total = (int64_t)rows_per_tile * cols;
  for (int64_t o = threadIdx.x; o < total; o += kThreads) {
    const int row = (int)(o / cols), col = (int)(o - (int64_t)row * cols);
    const int a = row / nb, bb = row - a * nb;
    const int c = col / j2, e = col - c * j2;
    const float* gp = g0 + (a * j1 + c) * r;
    double acc = 0.0;
    for (int rr = 0; rr < r; ++rr) acc = fma((double)gp[rr], (double)dq[(rr * kBT + bb) * j2 + e], acc);
    const int64_t orow = (int64_t)a * i2 + b0 + bb;
    const int64_t oidx = blk * (int64_t)i1 * i2 * cols + orow * cols + col;
    if (out_dtype == DQ_F16)
      ((__half*)out)[oidx] = __float2half_rn((float)acc);
    else
      ((float*)out)[oidx] = (float)acc;
  }
}

// ---- K4 for 128-wide rows (j = (8, 16)) on the fp64 tensor pipe ---------------------------
// Per CTA: one block x 8 b values.  D[(a, c)][(b, e)] = sum_r G0[(a, c)][r] dq[r][(b, e)] is a
// (64 x 64) . (64 x 128) GEMM: DMMA m8n8k4, warp w owns the 8 rows (a, c) = 8w.. x 128 columns.
// Operands are staged as fp32 (G0 as stored, dq = f32(code) * f32(scale): quantize.py:154-157)
// and widened exactly to fp64 in the fragments: the same f64 accumulation of the same f32
// values as the reference's reconstruct (mpo.py:181-198).
constexpr int kK4Pitch = 68;  // floats per row of the operand tiles (conflict-light fragment reads)

__device__ __forceinline__ void dmma64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kThreads) reconstruct128_kernel(const float* __restrict__ core0,
                                                                  const uint8_t* __restrict__ payload,
                                                                  int64_t payload_stride, CoreGeom geom,
                                                                  const float* __restrict__ scale, int i1,
                                                                  void* __restrict__ out, int out_dtype) {
  extern __shared__ __align__(16) float k4s[];
  float* g0 = k4s;                   // [p = (a, c)][r]
  float* dq = k4s + 64 * kK4Pitch;   // [(b, e)][r]
  const int r = geom.r, i2 = geom.i2;
  const int64_t blk = blockIdx.x;
  const int b0 = blockIdx.y * 8;
  const float s = scale[blk];
  const float* c0 = core0 + blk * (int64_t)i1 * 8 * r;
  const uint8_t* pl = payload + blk * payload_stride;
  for (int i = threadIdx.x; i < 64 * 64; i += kThreads) {
    const int p = i / 64, rr = i % 64;
    g0[p * kK4Pitch + rr] = (p < i1 * 8 && rr < r) ? c0[p * r + rr] : 0.f;
  }
  for (int i = threadIdx.x; i < 128 * 64; i += kThreads) {
    const int rr = i / 128, be = i % 128, bl = be / 16, e = be % 16;
    float v = 0.f;
    if (rr < r && b0 + bl < i2) v = __fmul_rn((float)geom_read(pl, geom, rr, b0 + bl, e), s);
    dq[be * kK4Pitch + rr] = v;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  double acc[16][2];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j][0] = acc[j][1] = 0.0;
  const float* arow = g0 + (w * 8 + g) * kK4Pitch + t4;
  for (int k = 0; k < r; k += 4) {
    const double a = (double)arow[k];
#pragma unroll
    for (int j = 0; j < 16; ++j) dmma64(acc[j][0], acc[j][1], a, (double)dq[(j * 8 + g) * kK4Pitch + k + t4]);
  }
  const int p = w * 8 + g, aa = p / 8, c = p % 8;
  if (aa >= i1) return;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int be = j * 8 + 2 * t4, bl = be / 16, e = be % 16;
    if (b0 + bl >= i2) continue;
    const int64_t o = blk * (int64_t)i1 * i2 * 128 + ((int64_t)aa * i2 + b0 + bl) * 128 + c * 16 + e;
    if (out_dtype == DQ_F16) {
      *reinterpret_cast<__half2*>(static_cast<__half*>(out) + o) =
          __halves2half2(__float2half_rn((float)acc[j][0]), __float2half_rn((float)acc[j][1]));
    } else {
      *reinterpret_cast<float2*>(static_cast<float*>(out) + o) = make_float2((float)acc[j][0], (float)acc[j][1]);
    }
  }
}

// WorkingSetMeter (compress.py:23-33), measured by the kernels: meter[0] = the most dequantized
// codes one CTA holds at once (atomicMax), meter[1] = codes dequantized in total (atomicAdd)
__device__ __forceinline__ void meter_report(unsigned long long* meter, long long held, long long unpacked) {
  if (!meter) return;
  for (int o = 16; o; o >>= 1) {
    held += __shfl_xor_sync(0xffffffffu, held, o);
    unpacked += __shfl_xor_sync(0xffffffffu, unpacked, o);
  }
  __shared__ unsigned long long red[2];
  if (threadIdx.x == 0) red[0] = red[1] = 0ull;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&red[0], (unsigned long long)held);
    atomicAdd(&red[1], (unsigned long long)unpacked);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMax(&meter[0], red[0]);
    atomicAdd(&meter[1], red[1]);
  }
}

// Both fused reads stage tiles of at most TILE_ELEMENTS = 64 x 64 codes (compress.py:20, the
// reference's working-set bound) in shared memory with every thread's loads in flight at once,
// then contract from shared memory; the staged tile is the CTA's whole working set.
constexpr int kTileCodes = 64 * 64;

// ---- x @ W^T: CTA (query row p, tile of kFT rows b, group of kFR bond rows) -------
//   Wt[a][r][e] = sum_c x[p, c*j2+e] * core0[a,c,r]   (the group's bond rows, in shared memory)
//   part[p][grp][a*i2+b] = sum_{r in grp, e} Wt[a][r][e] * code[r,b,e]   (fp64, workspace)
//   out[p, a*i2+b] = scale * sum_grp part[p][grp][a*i2+b]   (fused_t_sum_kernel, fixed order)
//   lane = b within the tile, warp w = bond row w of the group
constexpr int kFT = 32;
constexpr int kFR = 8;

__global__ void __launch_bounds__(kThreads) fused_t_kernel(const float* __restrict__ x, const float* __restrict__ core0,
                                                           const uint8_t* __restrict__ payload, CoreGeom geom, int i1,
                                                           int j1, int cols, int fr, double* __restrict__ part,
                                                           unsigned long long* meter) {
  // fr <= kFR bond rows per group: fr * j2 * kFT codes stay within one 64 x 64 tile
  extern __shared__ double smem_d[];
  const int r = geom.r, i2 = geom.i2, j2 = geom.j2;
  float* xs = reinterpret_cast<float*>(smem_d);               // [cols]
  float* wt = xs + cols;                                      // [i1][kFR][j2]
  int8_t* cs = reinterpret_cast<int8_t*>(wt + i1 * kFR * j2);  // [kFR][j2][kFT]
  const int p = blockIdx.x, b0 = blockIdx.y * kFT, r0 = blockIdx.z * fr;
  const int rows = i1 * i2, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int live = min(kFT, i2 - b0), nr = min(fr, r - r0);
  for (int i = tid; i < cols; i += kThreads) xs[i] = x[(int64_t)p * cols + i];
  for (int i = tid; i < nr * j2 * kFT; i += kThreads) {  // code (r0 + rl, b0 + bl, e)
    const int bl = i % kFT, re = i / kFT, rl = re / j2, e = re - rl * j2;
    cs[i] = (int8_t)(bl < live ? geom_read(payload, geom, r0 + rl, b0 + bl, e) : 0);
  }
  __syncthreads();
  for (int i = tid; i < i1 * nr * j2; i += kThreads) {
    const int a = i / (nr * j2), rem = i - a * nr * j2;
    const int rl = rem / j2, e = rem - rl * j2;
    double acc = 0.0;
    for (int c = 0; c < j1; ++c) acc = fma((double)xs[c * j2 + e], (double)core0[(a * j1 + c) * r + r0 + rl], acc);
    wt[(a * kFR + rl) * j2 + e] = (float)acc;
  }
  __syncthreads();
  double acc[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) acc[a] = 0.0;
  if (w < nr)
    for (int e = 0; e < j2; ++e) {
      const double cv = (double)cs[(w * j2 + e) * kFT + lane];
#pragma unroll
      for (int a = 0; a < 8; ++a)
        if (a < i1) acc[a] = fma((double)wt[(a * kFR + w) * j2 + e], cv, acc[a]);
    }
  meter_report(meter, tid == 0 ? (long long)nr * j2 * live : 0, tid == 0 ? (long long)nr * j2 * live : 0);
  // the group's partial: the warps' bond rows added in a fixed order through shared memory
  __syncthreads();
  double* red = smem_d;  // [kFR][8 a][kFT] (reuses xs / wt / codes: every read is done)
#pragma unroll
  for (int a = 0; a < 8; ++a)
    if (w < kFR) red[(w * 8 + a) * kFT + lane] = acc[a];
  __syncthreads();
  double* dst = part + ((int64_t)p * gridDim.z + blockIdx.z) * rows;
  for (int i = tid; i < i1 * kFT; i += kThreads) {
    const int a = i / kFT, bl = i - a * kFT;
    if (bl >= live) continue;
    double v = 0.0;
    for (int ww = 0; ww < nr; ++ww) v += red[(ww * 8 + a) * kFT + bl];
    dst[a * i2 + b0 + bl] = v;
  }
}

__global__ void fused_t_sum_kernel(const double* __restrict__ part, int groups, int64_t rows,
                                   const float* __restrict__ scale, float* __restrict__ out) {
  const int p = blockIdx.y;
  const double s = (double)*scale;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int g = 0; g < groups; ++g) v += part[((int64_t)p * groups + g) * rows + i];
    out[(int64_t)p * rows + i] = (float)(v * s);
  }
}

// ---- x @ W: CTA (query row p, chunk of b rows) ------------------------------
//   part[p][chunk][a][r][e] = sum_{b in chunk} x[p, a*i2+b] * code[r,b,e]   (thread per (r,e),
//   tiles of at most TILE_ELEMENTS codes; fp64, workspace)
//   out[p, c*j2+e] = scale * sum_{a,r} core0[a,c,r] * f32(sum_chunk part[...])   (fused_n_out_kernel)
constexpr int kFNThreads = 1024;
constexpr int kFNChunk = 32;  // b rows per CTA

__global__ void __launch_bounds__(kFNThreads) fused_n_kernel(const float* __restrict__ x,
                                                             const uint8_t* __restrict__ payload, CoreGeom geom, int i1,
                                                             double* __restrict__ part, unsigned long long* meter) {
  extern __shared__ float smem[];
  const int r = geom.r, i2 = geom.i2, j2 = geom.j2;
  const int pairs = r * j2, tid = threadIdx.x;
  const int p = blockIdx.x, c0 = blockIdx.y * kFNChunk, cn = min(kFNChunk, i2 - c0);
  float* xs = smem;                                       // [i1][kFNChunk]
  int8_t* cs = reinterpret_cast<int8_t*>(xs + i1 * kFNChunk);  // [kfn][r][j2]
  const int kfn = max(1, kTileCodes / pairs);             // b rows per tile
  for (int i = tid; i < i1 * kFNChunk; i += kFNThreads) {
    const int a = i / kFNChunk, bl = i - a * kFNChunk;
    xs[i] = bl < cn ? x[(int64_t)p * i1 * i2 + (int64_t)a * i2 + c0 + bl] : 0.f;
  }
  constexpr int kPer = 2;  // (r, e) pairs per thread: r * j2 <= 2048
  double acc[kPer][8];
#pragma unroll
  for (int k = 0; k < kPer; ++k)
#pragma unroll
    for (int a = 0; a < 8; ++a) acc[k][a] = 0.0;
  for (int t0 = 0; t0 < cn; t0 += kfn) {
    __syncthreads();  // the previous tile's codes are read (and xs is loaded)
    const int nb = min(kfn, cn - t0);
    for (int i = tid; i < nb * pairs; i += kFNThreads) {  // code (rr, c0 + t0 + bl, e)
      const int bl = i / pairs, re = i - bl * pairs, rr = re / j2, e = re - rr * j2;
      cs[i] = (int8_t)geom_read(payload, geom, rr, c0 + t0 + bl, e);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int re = tid + k * kFNThreads;
      if (re < pairs)
        for (int bl = 0; bl < nb; ++bl) {
          const double cv = (double)cs[bl * pairs + re];
#pragma unroll
          for (int a = 0; a < 8; ++a)
            if (a < i1) acc[k][a] = fma((double)xs[a * kFNChunk + t0 + bl], cv, acc[k][a]);
        }
    }
  }
  double* dst = part + ((int64_t)p * gridDim.y + blockIdx.y) * i1 * pairs;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int re = tid + k * kFNThreads;
#pragma unroll
    for (int a = 0; a < 8; ++a)
      if (re < pairs && a < i1) dst[a * pairs + re] = acc[k][a];
  }
  meter_report(meter, tid == 0 ? (long long)min(kfn, cn) * pairs : 0, tid == 0 ? (long long)cn * pairs : 0);
}

__global__ void __launch_bounds__(kFNThreads) fused_n_out_kernel(const double* __restrict__ part, int chunks,
                                                                 const float* __restrict__ core0, CoreGeom geom, int i1,
                                                                 int j1, int cols, const float* __restrict__ scale,
                                                                 float* __restrict__ out) {
  extern __shared__ float y[];  // [i1][r][j2]
  const int r = geom.r, j2 = geom.j2, pairs = r * j2, p = blockIdx.x, tid = threadIdx.x;
  // Y = the chunks' partials summed in chunk order: 8 independent sums per thread in flight
  const int n = i1 * pairs;
  for (int i0 = 0; i0 < n; i0 += 8 * kFNThreads) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = 0.0;
    for (int g = 0; g < chunks; ++g) {
      const double* src = part + ((int64_t)p * chunks + g) * n;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k * kFNThreads + tid;
        if (i < n) v[k] += src[i];
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + k * kFNThreads + tid;
      if (i < n) y[i] = (float)v[k];
    }
  }
  __syncthreads();
  // out[c, e] = scale * sum_a sum_r core0[a,c,r] y[a,r,e]: 8 lanes per output (lane & 7 = a
  // residue), combined by a fixed butterfly
  const double s = (double)*scale;
  for (int o0 = 0; o0 < cols * 8; o0 += kFNThreads) {
    const int o = o0 + tid, i = o >> 3, k = o & 7;
    double v = 0.0;
    if (i < cols) {
      const int c = i / j2, e = i - c * j2;
      for (int a = k; a < i1; a += 8)
        for (int rr = 0; rr < r; ++rr)
          v = fma((double)core0[(a * j1 + c) * r + rr], (double)y[(a * r + rr) * j2 + e], v);
    }
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    if (i < cols && k == 0) out[(int64_t)p * cols + i] = (float)(v * s);
  }
}

// ---- packed-core relayout: one thread per destination byte ------------------
__global__ void relayout_kernel(const uint8_t* __restrict__ src, CoreGeom gs, int64_t src_stride,
                                uint8_t* __restrict__ dst, CoreGeom gd, int64_t dst_stride, int64_t dst_bytes) {
  const int bits = gd.bits;
  const int per = 8 / bits;
  const int64_t blk = blockIdx.y;
  const uint8_t* s = src + blk * src_stride;
  uint8_t* d = dst + blk * dst_stride;
  const int64_t nslots = geom_slots(gd);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dst_bytes; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned v = 0;
    for (int k = 0; k < per; ++k) {
      const int64_t slot = i * per + k;
      if (slot >= nslots) break;
      int rr, b, e;
      const int code = geom_coords(gd, slot, rr, b, e) ? geom_read(s, gs, rr, b, e) : 0;
      v |= geom_encode(code, gd) << (k * bits);
    }
    d[i] = (uint8_t)v;
  }
}

// core0 (1,i1,j1,r) f32 -> fp16 [a][r][c], divided by a per-block power of two so that
// max|g0h| lies in [0.5, 1): keeps W = q.G0 inside fp16 range whatever the K scale.
// One CTA per block.
__global__ void core0_f16_kernel(const float* __restrict__ core0, int i1, int j1, int r, void* __restrict__ out,
                                 int out_dtype, float* __restrict__ norm) {
  __shared__ float red[32];
  const int per = i1 * j1 * r;
  const int64_t blk = blockIdx.x;
  const float* src = core0 + blk * per;
  float m = 0.f;
  for (int i = threadIdx.x; i < per; i += blockDim.x) m = fmaxf(m, fabsf(src[i]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
  // f = 2^(e) with m / f in [0.5, 1); exact power of two, f = 1 for an all-zero core
  float f = 1.f;
  if (norm) {
    if (m > 0.f) {
      int e;
      frexpf(m, &e);
      f = ldexpf(1.f, e);
    }
    if (threadIdx.x == 0) norm[blk] = f;
  }
  const float inv = 1.f / f;
  for (int i = threadIdx.x; i < per; i += blockDim.x) {
    const int a = i / (r * j1), t = i - a * r * j1;
    const int rr = t / j1, c = t - rr * j1;
    const float v = src[(a * j1 + c) * r + rr] * inv;
    if (out_dtype == DQ_F16)
      static_cast<__half*>(out)[blk * per + i] = __float2half_rn(v);
    else
      static_cast<float*>(out)[blk * per + i] = v;
  }
}

int check_geom(const dq_plan2& p, int bits, int layout) {
  if (!bits_ok(bits)) return fail(DQ_ERR_UNSUPPORTED_BITS, "bits must be one of (2, 4, 8), got %d", bits);
  if (layout != DQ_LAYOUT_REF && layout != DQ_LAYOUT_KTILE && layout != DQ_LAYOUT_VTILE)
    return fail(DQ_ERR_INVALID_ARG, "unknown layout %d", layout);
  if (p.i1 * p.j1 > 64) return fail(DQ_ERR_UNSUPPORTED, "i1*j1 > 64");
  return DQ_OK;
}

// the fused reads' partial sums live in stream-ordered workspace from the device's default
// memory pool; keep freed blocks in the pool (the default threshold returns them to the driver
// at every synchronisation, a cudaMalloc per call)
int keep_pool_memory() {
  static bool done[64] = {};  // per device
  int dev = 0;
  DQ_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 64 && done[dev]) return DQ_OK;
  cudaMemPool_t pool;
  DQ_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = UINT64_MAX;
  DQ_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  if (dev < 64) done[dev] = true;
  return DQ_OK;
}

}  // namespace

}  // namespace dq

using namespace dq;

extern "C" int dq_deco_dequantize_batched(const float* core0, const uint8_t* payload, int64_t payload_stride,
                                          int32_t layout, const float* scale, int64_t nblk, int64_t rows,
                                          int64_t cols, int32_t bits, void* out, int32_t out_dtype, void* stream) {
  if (rows < 1 || cols < 1) return fail(DQ_ERR_SHAPE_MISMATCH, "dimensions must be >= 1");
  dq_plan2 p = make_plan2(rows, cols);
  int st = check_geom(p, bits, layout);
  if (st) return st;
  if (nblk == 0) return DQ_OK;
  if (!core0 || !payload || !scale || !out) return fail(DQ_ERR_INVALID_ARG, "null pointer");
  CoreGeom g = make_geom(p, bits, layout);
  if (cols == 128 && p.j1 == 8 && p.j2 == 16 && p.r <= 64) {  // every KV block: the tensor-pipe kernel
    dim3 grid((unsigned)nblk, (unsigned)ceil_div(p.i2, 8));
    constexpr int k4smem = (int)sizeof(float) * 192 * kK4Pitch;
    static bool attr = false;
    if (!attr) {
      DQ_CUDA_TRY(cudaFuncSetAttribute(reconstruct128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, k4smem));
      attr = true;
    }
    reconstruct128_kernel<<<grid, kThreads, k4smem, (cudaStream_t)stream>>>(core0, payload, payload_stride, g, scale,
                                                                       (int)p.i1, out, out_dtype);
    DQ_LAUNCH_CHECK();
    return DQ_OK;
  }
  const size_t smem = sizeof(float) * ((size_t)p.i1 * p.j1 * p.r + (size_t)p.r * kBT * p.j2);
  if (smem > 200 * 1024) return fail(DQ_ERR_UNSUPPORTED, "plan too large for the reconstruct kernel");
  DQ_CUDA_TRY(cudaFuncSetAttribute(reconstruct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)nblk, (unsigned)ceil_div(p.i2, kBT));
  reconstruct_kernel<<<grid, kThreads, smem, (cudaStream_t)stream>>>(core0, payload, payload_stride, g, scale,
                                                                    (int)p.i1, (int)p.j1, (int)cols, out, out_dtype);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_fused_matmul_t(const float* x, int64_t np, const float* core0, const uint8_t* payload,
                                 int32_t layout, const float* scale, int64_t rows, int64_t cols, int32_t bits,
                                 float* out, uint64_t* meter, void* stream) {
  if (rows < 1 || cols < 1) return fail(DQ_ERR_SHAPE_MISMATCH, "dimensions must be >= 1");
  dq_plan2 p = make_plan2(rows, cols);
  int st = check_geom(p, bits, layout);
  if (st) return st;
  if (np == 0) return DQ_OK;
  if (!x || !core0 || !payload || !scale || !out) return fail(DQ_ERR_INVALID_ARG, "null pointer");
  if (p.i1 > 8) return fail(DQ_ERR_UNSUPPORTED, "i1 > 8");
  if (np > 65535) return fail(DQ_ERR_UNSUPPORTED, "more than 65535 query rows");
  CoreGeom g = make_geom(p, bits, layout);
  const size_t smem = std::max(sizeof(float) * ((size_t)cols + (size_t)p.i1 * kFR * p.j2) + (size_t)kFR * p.j2 * kFT,
                               sizeof(double) * kFR * 8 * kFT);
  if (smem > 200 * 1024) return fail(DQ_ERR_UNSUPPORTED, "plan too large for the fused kernel");
  cudaStream_t s = (cudaStream_t)stream;
  const int fr = std::max(1, std::min(kFR, kTileCodes / (int)(p.j2 * kFT)));  // bond rows per group
  const int groups = (int)ceil_div(p.r, fr);
  if (int rc = keep_pool_memory()) return rc;
  double* part = nullptr;  // the bond-row groups' partial sums (stream-ordered workspace)
  DQ_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * np * groups * rows, s));
  DQ_CUDA_TRY(cudaFuncSetAttribute(fused_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)np, (unsigned)ceil_div(p.i2, kFT), (unsigned)groups);
  fused_t_kernel<<<grid, kThreads, smem, s>>>(x, core0, payload, g, (int)p.i1, (int)p.j1, (int)cols, fr, part,
                                              (unsigned long long*)meter);
  DQ_LAUNCH_CHECK();
  fused_t_sum_kernel<<<dim3((unsigned)std::min<int64_t>(ceil_div(rows, kThreads), 64), (unsigned)np), kThreads, 0, s>>>(
      part, groups, rows, scale, out);
  DQ_LAUNCH_CHECK();
  DQ_CUDA_TRY(cudaFreeAsync(part, s));
  return DQ_OK;
}

extern "C" int dq_fused_matmul(const float* x, int64_t np, const float* core0, const uint8_t* payload,
                               int32_t layout, const float* scale, int64_t rows, int64_t cols, int32_t bits,
                               float* out, uint64_t* meter, void* stream) {
  if (rows < 1 || cols < 1) return fail(DQ_ERR_SHAPE_MISMATCH, "dimensions must be >= 1");
  dq_plan2 p = make_plan2(rows, cols);
  int st = check_geom(p, bits, layout);
  if (st) return st;
  if (np == 0) return DQ_OK;
  if (!x || !core0 || !payload || !scale || !out) return fail(DQ_ERR_INVALID_ARG, "null pointer");
  if (p.i1 > 8) return fail(DQ_ERR_UNSUPPORTED, "i1 > 8");
  if ((int64_t)p.r * p.j2 > 2 * kFNThreads) return fail(DQ_ERR_UNSUPPORTED, "plan too large for the fused kernel");
  if (np > 65535) return fail(DQ_ERR_UNSUPPORTED, "more than 65535 query rows");
  CoreGeom g = make_geom(p, bits, layout);
  cudaStream_t s = (cudaStream_t)stream;
  const int chunks = (int)ceil_div(p.i2, kFNChunk);
  const int64_t ysz = (int64_t)p.i1 * p.r * p.j2;
  if (int rc = keep_pool_memory()) return rc;
  double* part = nullptr;  // the b chunks' partial Y (stream-ordered workspace)
  DQ_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * np * chunks * ysz, s));
  const size_t smem = sizeof(float) * p.i1 * kFNChunk + (size_t)kTileCodes;
  fused_n_kernel<<<dim3((unsigned)np, (unsigned)chunks), kFNThreads, smem, s>>>(x, payload, g, (int)p.i1, part,
                                                                              (unsigned long long*)meter);
  DQ_LAUNCH_CHECK();
  const size_t smem2 = sizeof(float) * ysz;
  if (smem2 > 200 * 1024) return fail(DQ_ERR_UNSUPPORTED, "plan too large for the fused kernel");
  DQ_CUDA_TRY(cudaFuncSetAttribute(fused_n_out_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
  fused_n_out_kernel<<<(unsigned)np, kFNThreads, smem2, s>>>(part, chunks, core0, g, (int)p.i1, (int)p.j1, (int)cols,
                                                           scale, out);
  DQ_LAUNCH_CHECK();
  DQ_CUDA_TRY(cudaFreeAsync(part, s));
  return DQ_OK;
}

extern "C" int dq_relayout(const uint8_t* src, int32_t src_layout, int64_t src_stride, uint8_t* dst,
                           int32_t dst_layout, int64_t dst_stride, int64_t nblk, const dq_plan2* hp, int32_t bits,
                           void* stream) {
  if (!hp) return fail(DQ_ERR_INVALID_ARG, "null plan");
  int st = check_geom(*hp, bits, src_layout);
  if (st) return st;
  st = check_geom(*hp, bits, dst_layout);
  if (st) return st;
  if (nblk == 0) return DQ_OK;
  if (!src || !dst) return fail(DQ_ERR_INVALID_ARG, "null pointer");
  int64_t dbytes;
  st = dq_layout_bytes(hp, bits, dst_layout, &dbytes);
  if (st) return st;
  CoreGeom gs = make_geom(*hp, bits, src_layout), gd = make_geom(*hp, bits, dst_layout);
  int64_t gx = ceil_div(dbytes, kThreads);
  if (gx > 256) gx = 256;
  relayout_kernel<<<dim3((unsigned)gx, (unsigned)nblk), kThreads, 0, (cudaStream_t)stream>>>(src, gs, src_stride, dst,
                                                                                            gd, dst_stride, dbytes);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_core0_relayout(const float* core0, int64_t nblk, const dq_plan2* hp, void* out, int32_t out_dtype,
                                 float* norm, void* stream) {
  if (!hp || (nblk && (!core0 || !out))) return fail(DQ_ERR_INVALID_ARG, "null pointer");
  if (out_dtype != DQ_F16 && out_dtype != DQ_F32) return fail(DQ_ERR_INVALID_ARG, "unknown dtype %d", out_dtype);
  if (nblk == 0) return DQ_OK;
  core0_f16_kernel<<<(unsigned)nblk, kThreads, 0, (cudaStream_t)stream>>>(core0, (int)hp->i1, (int)hp->j1, (int)hp->r,
                                                                         out, out_dtype, norm);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

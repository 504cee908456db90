// K4 reconstruct, the generic fused reads, layout conversion and small helpers.
//
//   reconstruct  : compress.py:105-107 -> mpo.py:181-198   (dequantize, contract, de-interleave)
//   fused_matmul_t: compress.py:195-231   x @ W^T without materialising W
//   fused_matmul : compress.py:159-192   x @ W   without materialising W
//
// These serve the reference-mirroring API for any n=2 plan.  The decode hot path
// uses the specialised D=128 kernel in attention.cu instead.
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

// ---- x @ W^T: one CTA per (query row p, tile of 256 b) ----------------------
//   Wt[a][r][e] = sum_c x[p, c*j2+e] * core0[a,c,r]   (staged in shared memory)
//   out[p, a*i2+b] = scale * sum_{r,e} Wt[a][r][e] * code[r,b,e]
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

__global__ void __launch_bounds__(kThreads) fused_t_kernel(const float* __restrict__ x, const float* __restrict__ core0,
                                                           const uint8_t* __restrict__ payload, CoreGeom geom,
                                                           const float* __restrict__ scale, int i1, int j1, int cols,
                                                           float* __restrict__ out, unsigned long long* meter) {
  extern __shared__ float smem[];
  const int r = geom.r, i2 = geom.i2, j2 = geom.j2;
  float* xs = smem;             // [cols]
  float* wt = smem + cols;      // [i1][r][j2]
  const int p = blockIdx.x;
  const int rows = i1 * i2;
  for (int i = threadIdx.x; i < cols; i += kThreads) xs[i] = x[(int64_t)p * cols + i];
  __syncthreads();
  for (int i = threadIdx.x; i < i1 * r * j2; i += kThreads) {
    const int a = i / (r * j2), rem = i - a * r * j2;
    const int rr = rem / j2, e = rem - rr * j2;
    double acc = 0.0;
    for (int c = 0; c < j1; ++c) acc = fma((double)xs[c * j2 + e], (double)core0[(a * j1 + c) * r + rr], acc);
    wt[i] = (float)acc;
  }
  __syncthreads();
  const int b = blockIdx.y * kThreads + threadIdx.x;
  const bool live = b < i2;
  double acc[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) acc[a] = 0.0;
  if (live) {
    for (int rr = 0; rr < r; ++rr)
      for (int e = 0; e < j2; ++e) {
        const double cv = (double)geom_read(payload, geom, rr, b, e);  // one code at a time per thread
        if (cv == 0.0) continue;
#pragma unroll
        for (int a = 0; a < 8; ++a)
          if (a < i1) acc[a] = fma((double)wt[(a * r + rr) * j2 + e], cv, acc[a]);
      }
  }
  meter_report(meter, live ? 1 : 0, live ? (long long)r * j2 : 0);
  if (!live) return;
  const double s = (double)*scale;
  for (int a = 0; a < i1; ++a) out[(int64_t)p * rows + a * i2 + b] = (float)(acc[a] * s);
}

// ---- x @ W: one CTA per query row p ---------------------------------------
//   Y[a][r][e] = sum_b x[p, a*i2+b] * code[r,b,e]        (thread per (r,e))
//   out[p, c*j2+e] = scale * sum_{a,r} core0[a,c,r] * Y[a][r][e]
__global__ void __launch_bounds__(kThreads) fused_n_kernel(const float* __restrict__ x, const float* __restrict__ core0,
                                                           const uint8_t* __restrict__ payload, CoreGeom geom,
                                                           const float* __restrict__ scale, int i1, int j1, int cols,
                                                           float* __restrict__ out, unsigned long long* meter) {
  extern __shared__ float smem[];
  const int r = geom.r, i2 = geom.i2, j2 = geom.j2;
  const int rows = i1 * i2;
  float* xs = smem;          // [rows]
  float* y = smem + rows;    // [i1][r][j2]
  const int p = blockIdx.x;
  for (int i = threadIdx.x; i < rows; i += kThreads) xs[i] = x[(int64_t)p * rows + i];
  __syncthreads();
  long long held = 0, unpacked = 0;
  for (int i = threadIdx.x; i < r * j2; i += kThreads) {
    const int rr = i / j2, e = i - rr * j2;
    double acc[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) acc[a] = 0.0;
    held = 1;  // one code at a time per thread
    unpacked += i2;
    for (int b = 0; b < i2; ++b) {
      const double cv = (double)geom_read(payload, geom, rr, b, e);
      if (cv == 0.0) continue;
#pragma unroll
      for (int a = 0; a < 8; ++a)
        if (a < i1) acc[a] = fma((double)xs[a * i2 + b], cv, acc[a]);
    }
    for (int a = 0; a < i1; ++a) y[(a * r + rr) * j2 + e] = (float)acc[a];
  }
  meter_report(meter, held, unpacked);
  __syncthreads();
  const double s = (double)*scale;
  for (int i = threadIdx.x; i < cols; i += kThreads) {
    const int c = i / j2, e = i - c * j2;
    double acc = 0.0;
    for (int a = 0; a < i1; ++a)
      for (int rr = 0; rr < r; ++rr)
        acc = fma((double)core0[(a * j1 + c) * r + rr], (double)y[(a * r + rr) * j2 + e], acc);
    out[(int64_t)p * cols + i] = (float)(acc * s);
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
  CoreGeom g = make_geom(p, bits, layout);
  const size_t smem = sizeof(float) * ((size_t)cols + (size_t)p.i1 * p.r * p.j2);
  if (smem > 200 * 1024) return fail(DQ_ERR_UNSUPPORTED, "plan too large for the fused kernel");
  DQ_CUDA_TRY(cudaFuncSetAttribute(fused_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)np, (unsigned)ceil_div(p.i2, kThreads));
  fused_t_kernel<<<grid, kThreads, smem, (cudaStream_t)stream>>>(x, core0, payload, g, scale, (int)p.i1, (int)p.j1,
                                                                (int)cols, out, (unsigned long long*)meter);
  DQ_LAUNCH_CHECK();
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
  CoreGeom g = make_geom(p, bits, layout);
  const size_t smem = sizeof(float) * ((size_t)rows + (size_t)p.i1 * p.r * p.j2);
  if (smem > 200 * 1024) return fail(DQ_ERR_UNSUPPORTED, "plan too large for the fused kernel");
  DQ_CUDA_TRY(cudaFuncSetAttribute(fused_n_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fused_n_kernel<<<(unsigned)np, kThreads, smem, (cudaStream_t)stream>>>(x, core0, payload, g, scale, (int)p.i1,
                                                                        (int)p.j1, (int)cols, out,
                                                                        (unsigned long long*)meter);
  DQ_LAUNCH_CHECK();
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

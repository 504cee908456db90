// Decode-harness kernels (the reference has no model, its toy analogue is
// kvcache.py:234-309): the elementwise work around the cuBLAS projections of the LLaMA-shaped
// decoder in model.py, fused so that one layer is ~10 launches (norm, QKV GEMM, RoPE, the three
// attention kernels, O GEMM, norm, gate/up GEMM, SwiGLU, down GEMM) instead of ~70 torch
// elementwise launches.  Rounding follows the torch expressions they replace (model.py
// _rms / _rope / silu * up) step for step: fp32 arithmetic, bf16 rounding where torch
// materialises a bf16 tensor, no FMA contraction where torch rounds a product.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

constexpr int kNormThreads = 256;
constexpr int kNormVec = 4;  // 8-element vectors per thread: hidden <= 8 * 256 * 4 = 8192

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ float bf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// x_out = bf16(x + y) (y optional); h = bf16(bf16(x_out * rsqrt(mean(x_out^2) + eps)) * w).
// One CTA per row; the row stays in registers between the reduction and the scaling.
__global__ void __launch_bounds__(kNormThreads) add_rmsnorm_kernel(const bf16* x,  // may alias x_out
                                                                   const bf16* __restrict__ y,
                                                                   const bf16* __restrict__ w, bf16* x_out,
                                                                   bf16* __restrict__ h, int hidden, float eps) {
  const int row = blockIdx.x, tid = threadIdx.x, nv = hidden / 8;
  const size_t base = (size_t)row * hidden;
  float v[kNormVec][8];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kNormVec; ++i) {
    const int c = tid + i * kNormThreads;
    if (c < nv) {
      uint4 xa = reinterpret_cast<const uint4*>(x + base)[c];
      const bf16* xe = reinterpret_cast<const bf16*>(&xa);
      if (y) {
        uint4 ya = reinterpret_cast<const uint4*>(y + base)[c];
        const bf16* ye = reinterpret_cast<const bf16*>(&ya);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[i][e] = bf(__bfloat162float(xe[e]) + __bfloat162float(ye[e]));
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[i][e] = __bfloat162float(xe[e]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) ss = fmaf(v[i][e], v[i][e], ss);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  __shared__ float red[kNormThreads / 32];
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < kNormThreads / 32; ++i) tot += red[i];
  const float rs = rsqrtf(tot / (float)hidden + eps);
#pragma unroll
  for (int i = 0; i < kNormVec; ++i) {
    const int c = tid + i * kNormThreads;
    if (c < nv) {
      uint4 wa = reinterpret_cast<const uint4*>(w)[c];
      const bf16* we = reinterpret_cast<const bf16*>(&wa);
      uint4 xo, ho;
      bf16* xoe = reinterpret_cast<bf16*>(&xo);
      bf16* hoe = reinterpret_cast<bf16*>(&ho);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xoe[e] = __float2bfloat16_rn(v[i][e]);
        hoe[e] = __float2bfloat16_rn(__fmul_rn(bf(__fmul_rn(v[i][e], rs)), __bfloat162float(we[e])));
      }
      if (y) reinterpret_cast<uint4*>(x_out + base)[c] = xo;
      reinterpret_cast<uint4*>(h + base)[c] = ho;
    }
  }
}

// Rotary embedding (half-split, model.py _rope) of the q and k heads of one fused QKV row at
// decode position *pos, written as fp16 in the attention's layouts; v is converted to fp16.
// CTA (row b, group of kRopeHeads heads); thread (head, i) owns the pair (i, i + 64) of one head.
constexpr int kRopeHeads = 8;

__global__ void __launch_bounds__(kRopeHeads * 64) qkv_rope_kernel(const bf16* __restrict__ qkv, int heads,
                                                                   int kv_heads, const int64_t* __restrict__ pos,
                                                                   float theta, __half* __restrict__ q,
                                                                   __half* __restrict__ k, __half* __restrict__ v) {
  const int b = blockIdx.x, ht = heads + 2 * kv_heads;
  const float p = (float)*pos;
  const bf16* row = qkv + (size_t)b * ht * 128;
  {
    const int hh = blockIdx.y * kRopeHeads + (threadIdx.x >> 6), i = threadIdx.x & 63;
    if (hh >= ht) return;
    const bf16* src = row + hh * 128;
    const float x1 = __bfloat162float(src[i]), x2 = __bfloat162float(src[i + 64]);
    __half* dst;
    if (hh < heads) {
      dst = q + ((size_t)b * heads + hh) * 128;
    } else if (hh < heads + kv_heads) {
      dst = k + ((size_t)b * kv_heads + hh - heads) * 128;
    } else {
      dst = v + ((size_t)b * kv_heads + hh - heads - kv_heads) * 128;
      dst[i] = __float2half_rn(x1);
      dst[i + 64] = __float2half_rn(x2);
      return;
    }
    const float inv = powf(theta, -(float)(2 * i) / 128.f);
    const float ang = __fmul_rn(p, inv);
    const float c = cosf(ang), s = sinf(ang);
    const float o1 = bf(__fsub_rn(__fmul_rn(x1, c), __fmul_rn(x2, s)));
    const float o2 = bf(__fadd_rn(__fmul_rn(x1, s), __fmul_rn(x2, c)));
    dst[i] = __float2half_rn(o1);
    dst[i + 64] = __float2half_rn(o2);
  }
}

// SwiGLU of a fused gate/up row (gate = columns [0, ffn), up = [ffn, 2 ffn)):
// out = bf16(bf16(silu(gate)) * up), 8 elements per thread.
__global__ void silu_mul_kernel(const bf16* __restrict__ gu, int ffn, bf16* __restrict__ out) {
  const int row = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ffn / 8) return;
  const uint4 ga = reinterpret_cast<const uint4*>(gu + (size_t)row * 2 * ffn)[c];
  const uint4 ua = reinterpret_cast<const uint4*>(gu + (size_t)row * 2 * ffn + ffn)[c];
  const bf16* ge = reinterpret_cast<const bf16*>(&ga);
  const bf16* ue = reinterpret_cast<const bf16*>(&ua);
  uint4 o;
  bf16* oe = reinterpret_cast<bf16*>(&o);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float g = __bfloat162float(ge[e]);
    const float sg = bf(__fdiv_rn(g, __fadd_rn(1.f, expf(-g))));
    oe[e] = __float2bfloat16_rn(__fmul_rn(sg, __bfloat162float(ue[e])));
  }
  reinterpret_cast<uint4*>(out + (size_t)row * ffn)[c] = o;
}

}  // namespace

using dq::fail;

extern "C" int dq_model_add_rmsnorm(const uint16_t* x, const uint16_t* y, const uint16_t* w, uint16_t* x_out,
                                    uint16_t* h, int32_t rows, int32_t hidden, float eps, void* stream) {
  if (rows <= 0) return DQ_OK;
  if (!x || !w || !h || (y && !x_out)) return fail(DQ_ERR_INVALID_ARG, "null pointer");
  if (hidden <= 0 || hidden % 8 || hidden > 8 * kNormThreads * kNormVec)
    return fail(DQ_ERR_SHAPE_MISMATCH, "hidden must be a positive multiple of 8 up to %d, got %d",
                8 * kNormThreads * kNormVec, hidden);
  add_rmsnorm_kernel<<<rows, kNormThreads, 0, (cudaStream_t)stream>>>(
      (const bf16*)x, (const bf16*)y, (const bf16*)w, (bf16*)x_out, (bf16*)h, hidden, eps);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_model_qkv_rope(const uint16_t* qkv, int32_t batch, int32_t heads, int32_t kv_heads,
                                 const int64_t* pos, float theta, uint16_t* q, uint16_t* k, uint16_t* v,
                                 void* stream) {
  if (batch <= 0) return DQ_OK;
  if (!qkv || !pos || !q || !k || !v) return fail(DQ_ERR_INVALID_ARG, "null pointer");
  if (heads <= 0 || kv_heads <= 0 || heads % kv_heads)
    return fail(DQ_ERR_SHAPE_MISMATCH, "heads (%d) must be a positive multiple of kv_heads (%d)", heads, kv_heads);
  const dim3 grid((unsigned)batch, (unsigned)((heads + 2 * kv_heads + kRopeHeads - 1) / kRopeHeads));
  qkv_rope_kernel<<<grid, kRopeHeads * 64, 0, (cudaStream_t)stream>>>((const bf16*)qkv, heads, kv_heads, pos, theta,
                                                               (__half*)q, (__half*)k, (__half*)v);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_model_silu_mul(const uint16_t* gate_up, int32_t rows, int32_t ffn, uint16_t* out, void* stream) {
  if (rows <= 0) return DQ_OK;
  if (!gate_up || !out) return fail(DQ_ERR_INVALID_ARG, "null pointer");
  if (ffn <= 0 || ffn % 8) return fail(DQ_ERR_SHAPE_MISMATCH, "ffn must be a positive multiple of 8, got %d", ffn);
  const dim3 grid((unsigned)((ffn / 8 + 255) / 256), (unsigned)rows);
  silu_mul_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((const bf16*)gate_up, ffn, (bf16*)out);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

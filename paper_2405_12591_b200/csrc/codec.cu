// K1 pack/unpack and K2 symmetric RTN quantizer (bit-exact with quantize.py:66-157).
//
// All three are HBM-bound byte/integer kernels: one thread per OUTPUT byte
// (pack, quantize) or per output code (unpack), grid-stride loops sized to a
// multiple of the SM count, no shared memory needed.
#include "common.cuh"

namespace dq {

namespace {

constexpr int kThreads = 256;

int grid_for(int64_t work) {
  int64_t blocks = ceil_div(work, kThreads);
  const int64_t cap = 148 * 16;
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

// quantize.py:66-82: two's complement in `bits`, earliest code in the low bits,
// last byte zero-padded.  RangeOverflow (quantize.py:71-72) goes to the flags word.
__global__ void pack_kernel(const int8_t* __restrict__ codes, int64_t count, int bits, uint8_t* __restrict__ out,
                            int32_t* flags) {
  const int per = 8 / bits;
  const int qmax = (1 << (bits - 1)) - 1;
  const unsigned mask = (1u << bits) - 1u;
  const int64_t nbytes = payload_bytes(count, bits);
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbytes; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned v = 0;
    for (int k = 0; k < per; ++k) {
      const int64_t idx = i * per + k;
      if (idx < count) {
        const int c = codes[idx];
        bad |= (c < -qmax) | (c > qmax);
        v |= ((unsigned)c & mask) << (k * bits);
      }
    }
    out[i] = (uint8_t)v;
  }
  if (bad && flags) atomicOr(flags, (int)DQ_FLAG_RANGE_OVERFLOW);
}

// quantize.py:95-120 (unpack == unpack_range with start 0)
__global__ void unpack_kernel(const uint8_t* __restrict__ payload, int64_t start, int64_t count, int bits,
                              int8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int8_t)read_code(payload, start + i, bits);
}

// max |t| as the bit pattern of a non-negative float (monotone as uint32) + finiteness
__global__ void amax_kernel(const float* __restrict__ t, int64_t count, unsigned* amax_bits, int32_t* flags) {
  float m = 0.f;
  bool nonfinite = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = t[i];
    nonfinite |= !isfinite(v);
    m = fmaxf(m, fabsf(v));
  }
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(amax_bits, __float_as_uint(m));
    if (nonfinite && flags) atomicOr(flags, (int)DQ_FLAG_NONFINITE);
  }
}

// quantize.py:133-151: codes computed in fp64 exactly as the reference, packed on the fly
__global__ void quantize_pack_kernel(const float* __restrict__ t, int64_t count, int bits,
                                     const unsigned* __restrict__ amax_bits, float* scale_out,
                                     uint8_t* __restrict__ out) {
  const int per = 8 / bits;
  const int qmax = (1 << (bits - 1)) - 1;
  const unsigned mask = (1u << bits) - 1u;
  const double amax = (double)__uint_as_float(*amax_bits);
  bool degenerate;
  const float scale = rtn_scale(amax, qmax, &degenerate);
  if (blockIdx.x == 0 && threadIdx.x == 0) *scale_out = scale;
  const int64_t nbytes = payload_bytes(count, bits);
  const double rinv = amax > 0.0 ? 1.0 / amax : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbytes; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned v = 0;
    if (!degenerate) {
      for (int k = 0; k < per; ++k) {
        const int64_t idx = i * per + k;
        if (idx < count) v |= ((unsigned)rtn_code_fast(t[idx], qmax, amax, rinv) & mask) << (k * bits);
      }
    }
    out[i] = (uint8_t)v;
  }
}

// fp64 input (quantize.py:131-145 on a float64 array): max |t| as the bits of a non-negative
// double (monotone as uint64) + finiteness
__global__ void amax_f64_kernel(const double* __restrict__ t, int64_t count, unsigned long long* amax_bits,
                                int32_t* flags) {
  double m = 0.0;
  bool nonfinite = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = t[i];
    nonfinite |= !isfinite(v);
    m = fmax(m, fabs(v));
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(amax_bits, (unsigned long long)__double_as_longlong(m));
    if (nonfinite && flags) atomicOr(flags, (int)DQ_FLAG_NONFINITE);
  }
}

__global__ void quantize_pack_f64_kernel(const double* __restrict__ t, int64_t count, int bits,
                                         const unsigned long long* __restrict__ amax_bits, float* scale_out,
                                         uint8_t* __restrict__ out) {
  const int per = 8 / bits;
  const int qmax = (1 << (bits - 1)) - 1;
  const unsigned mask = (1u << bits) - 1u;
  const double amax = __longlong_as_double((long long)*amax_bits);
  bool degenerate;
  const float scale = rtn_scale(amax, qmax, &degenerate);
  if (blockIdx.x == 0 && threadIdx.x == 0) *scale_out = scale;
  const int64_t nbytes = payload_bytes(count, bits);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbytes; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned v = 0;
    if (!degenerate) {
      for (int k = 0; k < per; ++k) {
        const int64_t idx = i * per + k;
        if (idx < count) v |= ((unsigned)rtn_code_f64(t[idx], qmax, amax) & mask) << (k * bits);
      }
    }
    out[i] = (uint8_t)v;
  }
}

// quantize.py:154-157: f32(code) * f32(scale)
__global__ void dequant_kernel(const uint8_t* __restrict__ payload, int64_t count, int bits,
                               const float* __restrict__ scale, float* __restrict__ out) {
  const float s = *scale;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __fmul_rn((float)read_code(payload, i, bits), s);
}

}  // namespace

}  // namespace dq

using namespace dq;

extern "C" int dq_pack(const int8_t* codes, int64_t count, int32_t bits, uint8_t* payload, int32_t* flags,
                       void* stream) {
  if (!bits_ok(bits)) return fail(DQ_ERR_UNSUPPORTED_BITS, "bits must be one of (2, 4, 8), got %d", bits);
  if (count < 0 || (count && (!codes || !payload))) return fail(DQ_ERR_INVALID_ARG, "dq_pack: bad arguments");
  if (count == 0) return DQ_OK;
  pack_kernel<<<grid_for(payload_bytes(count, bits)), kThreads, 0, (cudaStream_t)stream>>>(codes, count, bits,
                                                                                           payload, flags);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_unpack(const uint8_t* payload, int64_t payload_len, int64_t start, int64_t count, int32_t bits,
                         int8_t* codes, void* stream) {
  if (!bits_ok(bits)) return fail(DQ_ERR_UNSUPPORTED_BITS, "bits must be one of (2, 4, 8), got %d", bits);
  const int per = 8 / bits;
  if (start < 0 || count < 0 || (start + count + per - 1) / per > payload_len)
    return fail(DQ_ERR_CORRUPT_PAYLOAD, "requested element range exceeds payload");
  if (count == 0) return DQ_OK;
  unpack_kernel<<<grid_for(count), kThreads, 0, (cudaStream_t)stream>>>(payload, start, count, bits, codes);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_quantize_workspace_size(int64_t, size_t* bytes) {
  if (!bytes) return fail(DQ_ERR_INVALID_ARG, "null output");
  *bytes = 256;
  return DQ_OK;
}

extern "C" int dq_quantize_rtn(const float* t, int64_t count, int32_t bits, float* scale, uint8_t* payload,
                               int32_t* flags, void* ws, size_t ws_bytes, void* stream) {
  if (!bits_ok(bits)) return fail(DQ_ERR_UNSUPPORTED_BITS, "bits must be one of (2, 4, 8), got %d", bits);
  if (count < 0 || !scale || (count && (!t || !payload)) || !ws || ws_bytes < 256)
    return fail(DQ_ERR_INVALID_ARG, "dq_quantize_rtn: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned* amax = (unsigned*)ws;
  DQ_CUDA_TRY(cudaMemsetAsync(amax, 0, sizeof(unsigned), s));
  if (count) {
    amax_kernel<<<grid_for(count), kThreads, 0, s>>>(t, count, amax, flags);
    DQ_LAUNCH_CHECK();
  }
  quantize_pack_kernel<<<grid_for(payload_bytes(count, bits)), kThreads, 0, s>>>(t, count, bits, amax, scale,
                                                                                 payload);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_quantize_rtn_f64(const double* t, int64_t count, int32_t bits, float* scale, uint8_t* payload,
                                   int32_t* flags, void* ws, size_t ws_bytes, void* stream) {
  if (!bits_ok(bits)) return fail(DQ_ERR_UNSUPPORTED_BITS, "bits must be one of (2, 4, 8), got %d", bits);
  if (count < 0 || !scale || (count && (!t || !payload)) || !ws || ws_bytes < 256)
    return fail(DQ_ERR_INVALID_ARG, "dq_quantize_rtn_f64: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* amax = (unsigned long long*)ws;
  DQ_CUDA_TRY(cudaMemsetAsync(amax, 0, sizeof(unsigned long long), s));
  if (count) {
    amax_f64_kernel<<<grid_for(count), kThreads, 0, s>>>(t, count, amax, flags);
    DQ_LAUNCH_CHECK();
  }
  quantize_pack_f64_kernel<<<grid_for(payload_bytes(count, bits)), kThreads, 0, s>>>(t, count, bits, amax, scale,
                                                                                     payload);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_dequantize(const uint8_t* payload, int64_t count, int32_t bits, const float* scale, float* out,
                             void* stream) {
  if (!bits_ok(bits)) return fail(DQ_ERR_UNSUPPORTED_BITS, "bits must be one of (2, 4, 8), got %d", bits);
  if (count < 0 || (count && (!payload || !scale || !out))) return fail(DQ_ERR_INVALID_ARG, "dq_dequantize: bad arguments");
  if (count == 0) return DQ_OK;
  dequant_kernel<<<grid_for(count), kThreads, 0, (cudaStream_t)stream>>>(payload, count, bits, scale, out);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

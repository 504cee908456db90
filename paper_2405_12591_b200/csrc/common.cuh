// Shared helpers for the DecoQuant sm_100a kernels (see include/dquant_b200.h).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/dquant_b200.h"

namespace dq {

// ---- error plumbing (thread-local message behind dq_last_error) ----------
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

#define DQ_CUDA_TRY(expr)                                                              \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return ::dq::fail(DQ_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,        \
                        cudaGetErrorString(e_));                                       \
  } while (0)

#define DQ_LAUNCH_CHECK() DQ_CUDA_TRY(cudaGetLastError())

inline bool bits_ok(int bits) { return bits == 2 || bits == 4 || bits == 8; }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// The device layouts pad i2 to a multiple of this many rows (include/dquant_b200.h).
constexpr int kI2Pad = 64;

// mpo.py:66-70 / 73-96 with n=2
int64_t largest_divisor_le(int64_t x, int64_t cap = 8);
dq_plan2 make_plan2(int64_t rows, int64_t cols);

// ---- element addressing of packed large cores ---------------------------
struct CoreGeom {
  int32_t r, i2, j2, i2p;  // i2p == i2 for DQ_LAYOUT_REF
  int32_t layout;
  int32_t bits;
};

inline CoreGeom make_geom(const dq_plan2& p, int bits, int layout) {
  CoreGeom g;
  g.r = (int32_t)p.r;
  g.i2 = (int32_t)p.i2;
  g.j2 = (int32_t)p.j2;
  g.i2p = layout == DQ_LAYOUT_REF ? (int32_t)p.i2 : (int32_t)round_up(p.i2, kI2Pad);
  g.layout = layout;
  g.bits = bits;
  return g;
}

// number of code slots (including padding) of one packed core
__host__ __device__ inline int64_t geom_slots(const CoreGeom& g) { return (int64_t)g.r * g.i2p * g.j2; }

// Device layouts (include/dquant_b200.h): b is split into 64-row tiles bt, and
// the K rows of a tile are XOR-swizzled by r so that the mma fragment reads of
// 4 consecutive r hit distinct shared-memory banks.
__host__ __device__ inline int ktile_swizzle(int rr, int bits) { return (rr & 3) * (16 / bits); }

// linear code slot of logical element (rr, b, e)
__host__ __device__ inline int64_t geom_slot(const CoreGeom& g, int rr, int b, int e) {
  if (g.layout == DQ_LAYOUT_REF) return ((int64_t)rr * g.i2 + b) * g.j2 + e;
  const int bt = b / kI2Pad, bl = b % kI2Pad;
  if (g.layout == DQ_LAYOUT_VTILE) return (((int64_t)bt * g.r + rr) * g.j2 + e) * kI2Pad + bl;
  return (((int64_t)bt * g.r + rr) * kI2Pad + (bl ^ ktile_swizzle(rr, g.bits))) * g.j2 + e;
}

// inverse: logical element of a slot; returns false for padding slots
__host__ __device__ inline bool geom_coords(const CoreGeom& g, int64_t slot, int& rr, int& b, int& e) {
  if (g.layout == DQ_LAYOUT_REF) {
    e = (int)(slot % g.j2);
    const int64_t t = slot / g.j2;
    b = (int)(t % g.i2);
    rr = (int)(t / g.i2);
    return true;
  }
  if (g.layout == DQ_LAYOUT_VTILE) {
    const int bl = (int)(slot % kI2Pad);
    int64_t t = slot / kI2Pad;
    e = (int)(t % g.j2);
    t /= g.j2;
    rr = (int)(t % g.r);
    b = (int)(t / g.r) * kI2Pad + bl;
  } else {
    e = (int)(slot % g.j2);
    int64_t t = slot / g.j2;
    const int bsw = (int)(t % kI2Pad);
    t /= kI2Pad;
    rr = (int)(t % g.r);
    b = (int)(t / g.r) * kI2Pad + (bsw ^ ktile_swizzle(rr, g.bits));
  }
  return b < g.i2;
}

__host__ __device__ inline int64_t payload_bytes(int64_t count, int bits) { return (count * bits + 7) / 8; }

// signed code at slot (two's complement in `bits`, earliest element in the low bits)
// bits divides 8, so a code never spans two bytes: its bit offset slot * bits splits into a byte
// index and a shift without any (64-bit) division
__device__ __forceinline__ int read_code(const uint8_t* p, int64_t slot, int bits) {
  const int64_t bit = slot * bits;
  const unsigned raw = ((unsigned)p[bit >> 3] >> (unsigned)(bit & 7)) & ((1u << bits) - 1u);
  const int sign = 1 << (bits - 1);
  return (int)(raw ^ sign) - sign;
}

// Device layouts store codes in excess-2^(bits-1) form (code + 2^(bits-1), unsigned),
// which the attention kernel turns into fp16 with one LOP3 per pair of codes.
__device__ __forceinline__ int geom_read(const uint8_t* p, const CoreGeom& g, int rr, int b, int e) {
  const int64_t slot = geom_slot(g, rr, b, e);
  if (g.layout == DQ_LAYOUT_REF) return read_code(p, slot, g.bits);
  const int64_t bit = slot * g.bits;
  const unsigned raw = ((unsigned)p[bit >> 3] >> (unsigned)(bit & 7)) & ((1u << g.bits) - 1u);
  return (int)raw - (1 << (g.bits - 1));
}

// lane bits of `code` in layout g
__host__ __device__ inline unsigned geom_encode(int code, const CoreGeom& g) {
  const unsigned mask = (1u << g.bits) - 1u;
  return g.layout == DQ_LAYOUT_REF ? ((unsigned)code & mask) : ((unsigned)(code + (1 << (g.bits - 1))) & mask);
}

// ---- bit-exact replica of quantize.py:144-145 ---------------------------
// y = t * qmax / amax in fp64 (product first), code = copysign(floor(|y| + 0.5), y), clipped.
__device__ __forceinline__ int rtn_code(float t, int qmax, double amax) {
  const double y = __ddiv_rn(__dmul_rn((double)t, (double)qmax), amax);
  double c = floor(__dadd_rn(fabs(y), 0.5));
  if (c > (double)qmax) c = (double)qmax;
  return y < 0.0 ? -(int)c : (int)c;
}

// the same on an fp64 value (float64 input arrays: quantize.py:144 multiplies the original values)
__device__ __forceinline__ int rtn_code_f64(double t, int qmax, double amax) {
  const double y = __ddiv_rn(__dmul_rn(t, (double)qmax), amax);
  double c = floor(__dadd_rn(fabs(y), 0.5));
  if (c > (double)qmax) c = (double)qmax;
  return y < 0.0 ? -(int)c : (int)c;
}

// rtn_code without the fp64 division on the common path: y ~ RN(t*qmax) * RN(1/amax) is within
// ~2^-51 relative of RN(RN(t*qmax)/amax) (|y| <= 127), so whenever |y| + 1/2 lies more than 1e-9
// from an integer the rounded code is the same; near a rounding boundary (exact ties
// included) the exact division decides
__device__ __forceinline__ int rtn_code_fast(float t, int qmax, double amax, double rinv) {
  const double yt = __dmul_rn((double)t, (double)qmax);
  const double ya = yt * rinv;
  const double f = fabs(ya) + 0.5;
  const double fl = floor(f);
  if (f - fl > 1e-9 && fl + 1.0 - f > 1e-9) {
    const int c = min((int)fl, qmax);
    return ya < 0.0 ? -c : c;
  }
  return rtn_code(t, qmax, amax);
}

// quantize.py:135-140: f32(amax/qmax), or 1.0 when amax == 0 or the step underflows
__host__ __device__ inline float rtn_scale(double amax, int qmax, bool* degenerate) {
  float s = amax > 0.0 ? (float)(amax / (double)qmax) : 1.0f;
  const bool deg = (amax == 0.0) || (s == 0.0f);
  if (deg) s = 1.0f;
  if (degenerate) *degenerate = deg;
  return s;
}

}  // namespace dq

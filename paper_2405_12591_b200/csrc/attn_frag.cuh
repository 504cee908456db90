// Building blocks of the fused decode-attention kernel (attention.cu):
// TMA bulk copies + mbarriers, int8 tensor-core MMA, and the packed-code ->
// MMA-fragment unpacking with its element orders.
#pragma once

#include "common.cuh"

namespace dq {
namespace attn {

// ---- PTX wrappers ---------------------------------------------------------------
__device__ __forceinline__ int64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (int64_t)t;
}

__device__ __forceinline__ int sm_id() {
  int s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

#ifndef DQ_WAIT_HINT
#define DQ_WAIT_HINT 0x989680
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if DQ_WAIT_HINT
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(DQ_WAIT_HINT)  // suspend-time hint (ns): sleep in the wait, not spin
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}

// (c0, c1) += (a0, a1) * (b0, b1) as one packed fp32x2 FMA (FFMA2, sm_100); a scalar
// operand repeated in both halves is encoded as a broadcast, not a move
__device__ __forceinline__ uint64_t pack2(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void ffma2(float& c0, float& c1, float a0, float a1, float b0, float b1) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pack2(a0, a1)), "l"(pack2(b0, b1)), "l"(pack2(c0, c1)));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(d));
}

// spin variant (no suspend hint) for a single latency-critical thread
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// plain arrival (release semantics at CTA scope)
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// n arrivals at once (release semantics at CTA scope)
__device__ __forceinline__ void mbar_arrive_n(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}

// named barrier 1 over the first `threads` threads (the consumer warps)
__device__ __forceinline__ void named_sync(int threads) {
  asm volatile("bar.sync 1, %0;\n" ::"r"(threads) : "memory");
}

// named barrier 2 over `threads` threads (consumer warps + the MMA warp of the tcgen05 path)
__device__ __forceinline__ void named_sync2(int threads) {
  asm volatile("bar.sync 2, %0;\n" ::"r"(threads) : "memory");
}

// TMA bulk copy global -> shared, completing `bytes` on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// D += A . B on the int8 tensor pipe: m16n8k32, A row-major 16x32 (u8 or s8),
// B column-major 32x8 (u8 or s8), exact s32 accumulation.
template <bool A_SIGNED, bool B_SIGNED>
__device__ __forceinline__ void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
  if constexpr (A_SIGNED && B_SIGNED) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else if constexpr (A_SIGNED) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else if constexpr (B_SIGNED) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
}

// 2^(k - e) and 2^(e - k) for e = frexp exponent of a non-negative float x (x = m * 2^e,
// m in [0.5, 1)), by exponent-field arithmetic; x is clamped below to 2^-100 (0 included)
__device__ __forceinline__ float pow2_sub_exp(float x, int k) {  // 2^(k - e)
  const int E = max((int)((__float_as_uint(x) >> 23) & 0xFF), 27);
  return __uint_as_float((uint32_t)(k + 253 - E) << 23);
}
__device__ __forceinline__ float pow2_exp_sub(float x, int k) {  // 2^(e - k)
  const int E = max((int)((__float_as_uint(x) >> 23) & 0xFF), 27);
  return __uint_as_float((uint32_t)(E - 126 - k + 127) << 23);
}

// ---- packed code rows -----------------------------------------------------------------
// A row is 16 codes of one (r, b) [K side] or of one (r, e) x 16 b [V side]: 2*BITS bytes,
// excess-coded (code + 2^(bits-1)) as the device layouts store them.
template <int BITS>
struct Row {
  uint32_t w[BITS == 8 ? 4 : (BITS == 4 ? 2 : 1)];
};

template <int BITS>
__device__ __forceinline__ Row<BITS> lds_row(const unsigned char* p) {
  Row<BITS> r;
  if constexpr (BITS == 4) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    r.w[0] = v.x;
    r.w[1] = v.y;
  } else if constexpr (BITS == 2) {
    r.w[0] = *reinterpret_cast<const uint32_t*>(p);
  } else {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    r.w[0] = v.x;
    r.w[1] = v.y;
    r.w[2] = v.z;
    r.w[3] = v.w;
  }
  return r;
}

// Integer code offset seen by the MMA (int4/int2 stay excess-coded as u8; int8 is
// flipped to two's complement s8 and carries no offset).
template <int BITS>
constexpr int kExcess = BITS == 8 ? 0 : (1 << (BITS - 1));

// One row -> the four A-fragment words of two k32 MMAs (a0/a2 of MMA 0, a0/a2 of MMA 1).
// int4: nibbles -> bytes is one AND for the even and one SHF+AND for the odd codes;
// int2: crumbs -> bytes, three shifts and four ANDs; int8: one XOR per 4 codes.
template <int BITS>
__device__ __forceinline__ void row_bytes(const Row<BITS>& r, uint32_t (&o)[4]) {
  if constexpr (BITS == 4) {
    o[0] = r.w[0] & 0x0F0F0F0Fu;
    o[1] = (r.w[0] >> 4) & 0x0F0F0F0Fu;
    o[2] = r.w[1] & 0x0F0F0F0Fu;
    o[3] = (r.w[1] >> 4) & 0x0F0F0F0Fu;
  } else if constexpr (BITS == 2) {
    o[0] = r.w[0] & 0x03030303u;
    o[1] = (r.w[0] >> 2) & 0x03030303u;
    o[2] = (r.w[0] >> 4) & 0x03030303u;
    o[3] = (r.w[0] >> 6) & 0x03030303u;
  } else {
    o[0] = r.w[0] ^ 0x80808080u;
    o[1] = r.w[1] ^ 0x80808080u;
    o[2] = r.w[2] ^ 0x80808080u;
    o[3] = r.w[3] ^ 0x80808080u;
  }
}

// Element of the 16-group held at byte position i of those four words (i = 4*word + byte);
// the B operand of the same MMAs is laid out in 16-byte chunks with the same order, so
// every k slot pairs equal elements.
template <int BITS>
__host__ __device__ constexpr int ord16(int i) {
  if (BITS == 4) return (i >> 3) * 8 + 2 * (i & 3) + ((i >> 2) & 1);  // 0,2,4,6 | 1,3,5,7 | 8,..,14 | 9,..,15
  if (BITS == 2) return 4 * (i & 3) + (i >> 2);                        // 0,4,8,12 | 1,5,9,13 | ...
  return i;
}

template <int BITS>
__host__ __device__ constexpr int inv_ord16(int e) {
  if (BITS == 4) return 8 * (e >> 3) + 4 * (e & 1) + ((e & 7) >> 1);
  if (BITS == 2) return 4 * (e & 3) + (e >> 2);
  return e;
}

}  // namespace attn
}  // namespace dq

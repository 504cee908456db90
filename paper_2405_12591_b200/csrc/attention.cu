// K5: fused DecoQuant dequantisation + decode attention for D = 128 (j = (8,16)).
//
// Reference semantics (kvcache.py:188-217 scores, compress.py:159-231 fused reads):
// for one unit (sequence, kv head) with segments s of T_s tokens (plan i=(i1,i2),
// bond r) and g query rows q[h] (GQA group), the output is
//     softmax_t(q.K^T * sm_scale) V        over all segments and the fp16 tail,
// with K[a*i2+b, c*16+e] = sum_r G0k[a,c,r] * scale_k * code_k[r,b,e] (same for V).
//
// Factored order: per segment
//   W[h,a,r,e] = sum_c q[h,c*16+e] G0k[a,c,r]                  (CUDA cores, per CTA)
//   S[h,a,b]   = scale_k * sum_{r,e} W[h,a,r,e] code_k[r,b,e]   (tensor cores)
//   P          = exp(S*sm_scale - m)                           (online softmax, split-T)
//   Y[h,a,r,e] = sum_b P[h,a,b] code_v[r,b,e]                  (tensor cores)
//   O[h,c,e]   = scale_v * sum_{a,r} G0v[a,c,r] Y[h,a,r,e]     (CUDA cores, epilogue)
// Codes never leave registers as anything but fp16 MMA fragments: packed words are
// loaded with 4/8/16-byte coalesced loads straight into the fragment layout (the
// reduction index is permuted identically on both MMA operands, which is free),
// converted with the 0x6400 magic-number trick (exact: |code| <= 127 < 1024), and
// fed to mma.sync m16n8k16 (f16 x f16 -> f32).  Full-precision K/V never exist.
//
// Work item = (segment, 64*k-row slice of b) -> one CTA; partial (m, l, O) per item,
// merged with the dense fp16 tail by combine_kernel (flash-decoding split).
#include "common.cuh"

namespace dq {

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kD = 128;
constexpr int kMaxR = 64;

// ---- MMA ---------------------------------------------------------------------
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ---- packed rows of 16 codes ------------------------------------------------
// BITS=4: 8 bytes, BITS=2: 4 bytes, BITS=8: 16 bytes.  Stored pre-biased
// (xor with the sign bit of every lane) so each lane is code + 2^(bits-1).
template <int BITS>
struct Row {
  uint32_t w[BITS == 8 ? 4 : (BITS == 4 ? 2 : 1)];
};

template <int BITS>
__device__ __forceinline__ Row<BITS> load_row(const uint8_t* p) {
  Row<BITS> r;
  if constexpr (BITS == 4) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    r.w[0] = v.x ^ 0x88888888u;
    r.w[1] = v.y ^ 0x88888888u;
  } else if constexpr (BITS == 2) {
    r.w[0] = __ldg(reinterpret_cast<const uint32_t*>(p)) ^ 0xAAAAAAAAu;
  } else {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    r.w[0] = v.x ^ 0x80808080u;
    r.w[1] = v.y ^ 0x80808080u;
    r.w[2] = v.z ^ 0x80808080u;
    r.w[3] = v.w ^ 0x80808080u;
  }
  return r;
}

template <int BITS>
__device__ __forceinline__ Row<BITS> zero_row() {
  Row<BITS> r;
#pragma unroll
  for (int i = 0; i < (int)(sizeof(r.w) / 4); ++i) r.w[i] = BITS == 4 ? 0x88888888u : (BITS == 2 ? 0xAAAAAAAAu : 0x80808080u);
  return r;
}

// half2 pairs for sub-MMA c: lo -> k slots (2t, 2t+1), hi -> (2t+8, 2t+9).
// The element of the 16-group that lands in each slot is perm<BITS>(4c + {0,1,2,3}).
template <int BITS, int C>
__device__ __forceinline__ void row_pairs(const Row<BITS>& r, uint32_t& lo, uint32_t& hi) {
  uint32_t l, h;
  if constexpr (BITS == 4) {
    l = ((r.w[0] >> (4 * C)) & 0x000F000Fu) | 0x64006400u;
    h = ((r.w[1] >> (4 * C)) & 0x000F000Fu) | 0x64006400u;
  } else if constexpr (BITS == 2) {
    l = ((r.w[0] >> (2 * C)) & 0x00030003u) | 0x64006400u;
    h = ((r.w[0] >> (2 * C + 8)) & 0x00030003u) | 0x64006400u;
  } else {
    l = (r.w[C] & 0x00FF00FFu) | 0x64006400u;
    h = ((r.w[C] >> 8) & 0x00FF00FFu) | 0x64006400u;
  }
  constexpr uint32_t bias = BITS == 4 ? 0x64086408u : (BITS == 2 ? 0x64026402u : 0x64806480u);  // 1024+2^(b-1)
  const __half2 hb = *reinterpret_cast<const __half2*>(&bias);
  __half2 hl = __hsub2(*reinterpret_cast<__half2*>(&l), hb);
  __half2 hh = __hsub2(*reinterpret_cast<__half2*>(&h), hb);
  lo = *reinterpret_cast<uint32_t*>(&hl);
  hi = *reinterpret_cast<uint32_t*>(&hh);
}

// element of the 16-group held in permuted position q (must match row_pairs)
template <int BITS>
__host__ __device__ constexpr int perm16(int q) {
  const int c = q >> 2, j = q & 3;
  if (BITS == 4) return c + 4 * j;                       // c, c+4, c+8, c+12
  if (BITS == 2) return c + (j == 1 ? 8 : j == 2 ? 4 : j == 3 ? 12 : 0);  // c, c+8, c+4, c+12
  return 4 * c + (j == 1 ? 2 : j == 2 ? 1 : j);           // 4c, 4c+2, 4c+1, 4c+3
}

template <int BITS>
__device__ __forceinline__ int inv_perm16(int e) {
#pragma unroll
  for (int q = 0; q < 16; ++q)
    if (perm16<BITS>(q) == e) return q;
  return 0;
}

template <int G, int CB>
struct AttnSmem {
  float q[G][kD];
  // W in fragment order: 16-byte chunks [(h*r + rr)*2 + j][a ^ 2*(rr&3)]
  uint4 w[G * kMaxR * 2 * 8];
  // G0v fp16 [a][r][c] (16 bytes per (a, r))
  uint4 g0v[8 * kMaxR];
  float s[G][8][CB];
  // P in fragment order: 16-byte chunks [((h*8 + a)*NG + bg)*2 + (j ^ (a&1))]
  uint4 p[G * 8 * (CB / 16) * 2];
  float red[kWarps][G][kD];
  float wmax;
  float rowmax[G][kWarps];
  float rowsum[G][kWarps];
};

template <int BITS, int G, int MT>
__global__ void __launch_bounds__(kThreads) decode_attn_kernel(dq_attn_args args) {
  constexpr int CB = MT * 16 * kWarps;  // b rows per work item
  constexpr int NG = CB / 16;
  constexpr int RB = 2 * BITS;          // bytes per 16-code row
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AttnSmem<G, CB>& sm = *reinterpret_cast<AttnSmem<G, CB>*>(smem_raw);

  const int wi = blockIdx.x;
  const int seg_id = args.work[2 * wi];
  const int wb0 = args.work[2 * wi + 1];
  const dq_segment seg = args.segs[seg_id];
  const int unit = seg.unit;
  const int r = seg.r, i1 = seg.i1, i2 = seg.i2, i2p = seg.i2p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tid4 = lane & 3;

  // ---- phase 0: q, W = q . G0k (fp32 -> fp16 fragments), G0v ------------------
  const __half* qh = reinterpret_cast<const __half*>(args.q) + (size_t)unit * G * kD;
  for (int i = tid; i < G * kD; i += kThreads) sm.q[i / kD][i % kD] = __half2float(qh[i]);
  if (tid == 0) sm.wmax = 0.f;
  {
    const uint4* src = reinterpret_cast<const uint4*>(seg.v_g0);
    for (int i = tid; i < i1 * r; i += kThreads) sm.g0v[i] = src[i];
  }
  __syncthreads();
  // load the G0k row of bond index rr (8 values of c), zeros for a >= i1
  const uint4* g0k = reinterpret_cast<const uint4*>(seg.k_g0);
  auto g0k_row = [&](int a, int rr, float (&gk)[8]) {
    if (a < i1) {
      const uint4 gv = g0k[a * r + rr];
      const __half2* g2 = reinterpret_cast<const __half2*>(&gv);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __half22float2(g2[k]);
        gk[2 * k] = f.x;
        gk[2 * k + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) gk[k] = 0.f;
    }
  };
  float lmax = 0.f;
  for (int item = tid; item < G * 8 * r; item += kThreads) {
    const int h = item / (8 * r), rem = item - h * 8 * r;
    const int a = rem / r, rr = rem - a * r;
    float gk[8];
    g0k_row(a, rr, gk);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < 8; ++c) acc = fmaf(sm.q[h][c * 16 + e], gk[c], acc);
      lmax = fmaxf(lmax, fabsf(acc));
    }
  }
  for (int o = 16; o; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  if (lane == 0) atomicMax(reinterpret_cast<unsigned*>(&sm.wmax), __float_as_uint(lmax));
  __syncthreads();
  // power-of-two prescale keeps |W| inside fp16 range (exact, undone in the score scale)
  float wscale = 1.f;
  {
    const float wm = sm.wmax;
    while (wm * wscale > 16384.f) wscale *= 0.5f;
  }
  for (int item = tid; item < G * 8 * r; item += kThreads) {
    const int h = item / (8 * r), rem = item - h * 8 * r;
    const int a = rem / r, rr = rem - a * r;
    float gk[8];
    g0k_row(a, rr, gk);
    float wv[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < 8; ++c) acc = fmaf(sm.q[h][c * 16 + e], gk[c], acc);
      wv[e] = acc * wscale;
    }
    __half hv[16];
#pragma unroll
    for (int qi = 0; qi < 16; ++qi) hv[qi] = __float2half_rn(wv[perm16<BITS>(qi)]);
    const int sw = a ^ (2 * (rr & 3));
    sm.w[((h * r + rr) * 2 + 0) * 8 + sw] = *reinterpret_cast<uint4*>(&hv[0]);
    sm.w[((h * r + rr) * 2 + 1) * 8 + sw] = *reinterpret_cast<uint4*>(&hv[8]);
  }
  __syncthreads();

  // ---- phase 1: S = W . codes_k (tensor cores) ---------------------------------
  const int wbase = wb0 + warp * MT * 16;  // first b row of this warp
  float acc[MT][G][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int h = 0; h < G; ++h)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[mt][h][k] = 0.f;
  {
    const uint8_t* kc = seg.k_codes;
    bool valid[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      valid[mt][0] = wbase + mt * 16 + gid < i2p;
      valid[mt][1] = wbase + mt * 16 + gid + 8 < i2p;
    }
    auto load_step = [&](int rr0, Row<BITS> (&dst)[MT][2]) {
      const int rr = rr0 + tid4;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int b = wbase + mt * 16 + gid + 8 * hh;
          dst[mt][hh] = valid[mt][hh] ? load_row<BITS>(kc + ((size_t)rr * i2p + b) * RB) : zero_row<BITS>();
        }
    };
    Row<BITS> cur[MT][2], nxt[MT][2];
    load_step(0, cur);
    for (int rr0 = 0; rr0 < r; rr0 += 4) {
      if (rr0 + 4 < r) load_step(rr0 + 4, nxt);
      uint4 bw[G][2];
#pragma unroll
      for (int h = 0; h < G; ++h)
#pragma unroll
        for (int j = 0; j < 2; ++j) bw[h][j] = sm.w[((h * r + rr0 + tid4) * 2 + j) * 8 + (gid ^ (2 * tid4))];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        uint32_t a[4][4];
        row_pairs<BITS, 0>(cur[mt][0], a[0][0], a[0][2]);
        row_pairs<BITS, 0>(cur[mt][1], a[0][1], a[0][3]);
        row_pairs<BITS, 1>(cur[mt][0], a[1][0], a[1][2]);
        row_pairs<BITS, 1>(cur[mt][1], a[1][1], a[1][3]);
        row_pairs<BITS, 2>(cur[mt][0], a[2][0], a[2][2]);
        row_pairs<BITS, 2>(cur[mt][1], a[2][1], a[2][3]);
        row_pairs<BITS, 3>(cur[mt][0], a[3][0], a[3][2]);
        row_pairs<BITS, 3>(cur[mt][1], a[3][1], a[3][3]);
#pragma unroll
        for (int h = 0; h < G; ++h) {
          mma16816(acc[mt][h], a[0][0], a[0][1], a[0][2], a[0][3], bw[h][0].x, bw[h][0].y);
          mma16816(acc[mt][h], a[1][0], a[1][1], a[1][2], a[1][3], bw[h][0].z, bw[h][0].w);
          mma16816(acc[mt][h], a[2][0], a[2][1], a[2][2], a[2][3], bw[h][1].x, bw[h][1].y);
          mma16816(acc[mt][h], a[3][0], a[3][1], a[3][2], a[3][3], bw[h][1].z, bw[h][1].w);
        }
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        cur[mt][0] = nxt[mt][0];
        cur[mt][1] = nxt[mt][1];
      }
    }
  }
  // scores (already in log2 domain): s = acc * scale_k * sm_scale / wscale * log2(e)
  const float kscale = seg.k_scale * args.sm_scale / wscale * 1.4426950408889634f;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int h = 0; h < G; ++h)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int bl = warp * MT * 16 + mt * 16 + gid + (k >= 2 ? 8 : 0);
        const int a = 2 * tid4 + (k & 1);
        const bool ok = (a < i1) && (wb0 + bl < i2);
        sm.s[h][a][bl] = ok ? acc[mt][h][k] * kscale : -INFINITY;
      }
  __syncthreads();

  // ---- phase 2: local softmax of this work item ---------------------------------
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float m = -INFINITY;
    for (int i = tid; i < 8 * CB; i += kThreads) m = fmaxf(m, sm.s[h][i / CB][i % CB]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) sm.rowmax[h][warp] = m;
  }
  __syncthreads();
  float mh[G];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float m = sm.rowmax[h][0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) m = fmaxf(m, sm.rowmax[h][w]);
    mh[h] = m;
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float l = 0.f;
    __half* pbase = reinterpret_cast<__half*>(sm.p);
    for (int i = tid; i < 8 * CB; i += kThreads) {
      const int a = i / CB, bl = i % CB;
      const float sv = sm.s[h][a][bl];
      const float pv = sv == -INFINITY ? 0.f : exp2f(sv - mh[h]);
      const __half ph = __float2half_rn(pv);
      l += __half2float(ph);  // sum what the PV product actually uses
      const int bg = bl >> 4, q = inv_perm16<BITS>(bl & 15);
      const int j = q >> 3, within = q & 7;
      const int chunk = ((h * 8 + a) * NG + bg) * 2 + (j ^ (a & 1));
      pbase[chunk * 8 + within] = ph;
    }
    for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) sm.rowsum[h][warp] = l;
  }
  __syncthreads();

  // ---- phase 3: Y = codes_v . P^T (tensor cores) ---------------------------------
  // warp w owns bond rows rr = w*rw .. w*rw+rw-1 (rw = r/8 <= 8); m-tile = one rr x 16 e
  const int rw = r / kWarps;
  constexpr int HG = G < 2 ? G : 2;  // heads per V pass (register budget)
  const int nsteps = min(CB, i2p - wb0) / 64;
  float part[G][16];  // O partial: [h][c*2 + (e == gid+8)]
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int k = 0; k < 16; ++k) part[h][k] = 0.f;
  const uint8_t* vc = seg.v_codes;
#pragma unroll
  for (int hg = 0; hg < G; hg += HG) {
    float accv[8][HG][4];
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int h = 0; h < HG; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) accv[t][h][k] = 0.f;
    for (int st = 0; st < nsteps; ++st) {
      const int bstart = wb0 + st * 64 + 16 * tid4;
      Row<BITS> rows[8][2];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (t < rw) {
          const int rr = warp * rw + t;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int e = gid + 8 * hh;
            rows[t][hh] = load_row<BITS>(vc + (((size_t)rr * 16 + e) * i2p + bstart) * BITS / 8);
          }
        }
      }
      uint4 pf[HG][2];
#pragma unroll
      for (int h = 0; h < HG; ++h)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int bg = st * 4 + tid4;
          pf[h][j] = sm.p[(((hg + h) * 8 + gid) * NG + bg) * 2 + (j ^ (gid & 1))];
        }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (t < rw) {
          uint32_t a[4][4];
          row_pairs<BITS, 0>(rows[t][0], a[0][0], a[0][2]);
          row_pairs<BITS, 0>(rows[t][1], a[0][1], a[0][3]);
          row_pairs<BITS, 1>(rows[t][0], a[1][0], a[1][2]);
          row_pairs<BITS, 1>(rows[t][1], a[1][1], a[1][3]);
          row_pairs<BITS, 2>(rows[t][0], a[2][0], a[2][2]);
          row_pairs<BITS, 2>(rows[t][1], a[2][1], a[2][3]);
          row_pairs<BITS, 3>(rows[t][0], a[3][0], a[3][2]);
          row_pairs<BITS, 3>(rows[t][1], a[3][1], a[3][3]);
#pragma unroll
          for (int h = 0; h < HG; ++h) {
            mma16816(accv[t][h], a[0][0], a[0][1], a[0][2], a[0][3], pf[h][0].x, pf[h][0].y);
            mma16816(accv[t][h], a[1][0], a[1][1], a[1][2], a[1][3], pf[h][0].z, pf[h][0].w);
            mma16816(accv[t][h], a[2][0], a[2][1], a[2][2], a[2][3], pf[h][1].x, pf[h][1].y);
            mma16816(accv[t][h], a[3][0], a[3][1], a[3][2], a[3][3], pf[h][1].z, pf[h][1].w);
          }
        }
      }
    }
    // ---- phase 4a: contract Y with G0v on CUDA cores ---------------------------
    // accv[t][h]: rows e = gid (k 0,1) / gid+8 (k 2,3); cols a = 2*tid4 + (k & 1)
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (t < rw) {
        const int rr = warp * rw + t;
#pragma unroll
        for (int aa = 0; aa < 2; ++aa) {
          const int a = 2 * tid4 + aa;
          if (a < i1) {
            const uint4 gv = sm.g0v[a * r + rr];
            const __half2* g2 = reinterpret_cast<const __half2*>(&gv);
            float gc[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 f = __half22float2(g2[k]);
              gc[2 * k] = f.x;
              gc[2 * k + 1] = f.y;
            }
#pragma unroll
            for (int h = 0; h < HG; ++h)
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                part[hg + h][2 * c] = fmaf(gc[c], accv[t][h][aa], part[hg + h][2 * c]);
                part[hg + h][2 * c + 1] = fmaf(gc[c], accv[t][h][2 + aa], part[hg + h][2 * c + 1]);
              }
          }
        }
      }
    }
  }
  // reduce over the 4 threads of a quad (different a), then over warps (different rr)
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float v = part[h][k];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      part[h][k] = v;
    }
  // thread tid4 writes c = 2*tid4, 2*tid4+1 for e = gid, gid+8
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
      sm.red[warp][h][c * 16 + gid] = v0;
      sm.red[warp][h][c * 16 + gid + 8] = v1;
    }
  __syncthreads();
  const int slot = args.work_part[wi];
  for (int i = tid; i < G * kD; i += kThreads) {
    const int h = i / kD, d = i % kD;
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) v += sm.red[w][h][d];
    args.part_o[((size_t)slot * G + h) * kD + d] = v * seg.v_scale;
  }
  if (tid < G) {
    float l = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) l += sm.rowsum[tid][w];
    args.part_ml[((size_t)slot * G + tid) * 2 + 0] = mh[tid];  // log2 domain
    args.part_ml[((size_t)slot * G + tid) * 2 + 1] = l;
  }
}

// ---- combine: merge work-item partials with the dense fp16 tail ------------------
// one CTA (128 threads) per unit; thread d owns output dim d.
template <int G>
__global__ void __launch_bounds__(128) combine_kernel(dq_attn_args args) {
  extern __shared__ float tail_s[];  // [tail_cap]
  __shared__ float red[4];
  const int u = blockIdx.x;
  const int d = threadIdx.x, lane = d & 31, warp = d >> 5;
  const int p0 = args.unit_part0[u], np = args.unit_nparts[u];
  const int tl = args.tail_len ? args.tail_len[u] : 0;
  const float l2e = 1.4426950408889634f;
  for (int h = 0; h < G; ++h) {
    // dense tail scores (log2 domain)
    float tm = -INFINITY;
    if (tl > 0) {
      const __half* qh = reinterpret_cast<const __half*>(args.q) + ((size_t)u * G + h) * kD;
      const uint2 qv = reinterpret_cast<const uint2*>(qh)[lane];
      const __half2* q2 = reinterpret_cast<const __half2*>(&qv);
      const float2 qa = __half22float2(q2[0]), qb = __half22float2(q2[1]);
      const __half* tk = reinterpret_cast<const __half*>(args.tail_k) + (size_t)u * args.tail_cap * kD;
      for (int t = warp; t < tl; t += 4) {
        const uint2 kv = reinterpret_cast<const uint2*>(tk + (size_t)t * kD)[lane];
        const __half2* k2 = reinterpret_cast<const __half2*>(&kv);
        const float2 ka = __half22float2(k2[0]), kb = __half22float2(k2[1]);
        float dot = qa.x * ka.x + qa.y * ka.y + qb.x * kb.x + qb.y * kb.y;
        for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (lane == 0) tail_s[t] = dot * args.sm_scale * l2e;
      }
      __syncthreads();
      for (int t = d; t < tl; t += 128) tm = fmaxf(tm, tail_s[t]);
      for (int o = 16; o; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
      if (lane == 0) red[warp] = tm;
      __syncthreads();
      tm = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
      __syncthreads();
    }
    float M = tm;
    for (int i = 0; i < np; ++i) M = fmaxf(M, args.part_ml[((size_t)(p0 + i) * G + h) * 2]);
    float L = 0.f, O = 0.f;
    for (int i = 0; i < np; ++i) {
      const size_t s = (size_t)(p0 + i) * G + h;
      const float m = args.part_ml[s * 2];
      if (m == -INFINITY) continue;
      const float f = exp2f(m - M);
      L += f * args.part_ml[s * 2 + 1];
      O += f * args.part_o[s * kD + d];
    }
    if (tl > 0) {
      const __half* tv = reinterpret_cast<const __half*>(args.tail_v) + (size_t)u * args.tail_cap * kD;
      float lt = 0.f, ot = 0.f;
      for (int t = 0; t < tl; ++t) {
        const float p = exp2f(tail_s[t] - M);
        lt += p;
        ot = fmaf(p, __half2float(tv[(size_t)t * kD + d]), ot);
      }
      L += lt;
      O += ot;
      __syncthreads();
    }
    __half* out = reinterpret_cast<__half*>(args.out) + ((size_t)u * G + h) * kD;
    out[d] = __float2half_rn(L > 0.f ? O / L : 0.f);
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

template <int BITS, int G, int MT>
int launch_attn(const dq_attn_args& a, cudaStream_t s) {
  constexpr int CB = MT * 16 * kWarps;
  const size_t smem = sizeof(AttnSmem<G, CB>);
  static bool attr = false;
  if (!attr) {
    DQ_CUDA_TRY(cudaFuncSetAttribute(decode_attn_kernel<BITS, G, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    attr = true;
  }
  if (a.nwork > 0) {
    decode_attn_kernel<BITS, G, MT><<<a.nwork, kThreads, smem, s>>>(a);
    DQ_LAUNCH_CHECK();
  }
  const size_t csmem = sizeof(float) * (a.tail_cap > 0 ? a.tail_cap : 1);
  combine_kernel<G><<<a.units, 128, csmem, s>>>(a);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

template <int BITS, int G>
int dispatch_mt(const dq_attn_args& a, cudaStream_t s) {
  if (a.chunk_b == 256) return launch_attn<BITS, G, 2>(a, s);
  if (a.chunk_b == 512 && G <= 2) return launch_attn<BITS, G, (G <= 2 ? 4 : 2)>(a, s);
  return fail(DQ_ERR_UNSUPPORTED, "chunk_b %d not supported for g=%d (use 256%s)", a.chunk_b, G,
              G <= 2 ? " or 512" : "");
}

template <int BITS>
int dispatch_g(const dq_attn_args& a, cudaStream_t s) {
  switch (a.g) {
    case 1: return dispatch_mt<BITS, 1>(a, s);
    case 2: return dispatch_mt<BITS, 2>(a, s);
    case 4: return dispatch_mt<BITS, 4>(a, s);
  }
  return fail(DQ_ERR_UNSUPPORTED, "g must be 1, 2 or 4 in this build (got %d)", a.g);
}

}  // namespace

}  // namespace dq

using namespace dq;

extern "C" int dq_attention_plan(const dq_segment* segs, int32_t nseg, int32_t units, int32_t chunk_b, int32_t* work,
                                 int32_t* nwork, int32_t* work_part, int32_t* unit_part0, int32_t* unit_nparts,
                                 int32_t* total_parts) {
  if (nseg < 0 || units < 0 || chunk_b <= 0 || chunk_b % 64) return fail(DQ_ERR_INVALID_ARG, "bad plan arguments");
  if (!nwork || !total_parts || !unit_part0 || !unit_nparts) return fail(DQ_ERR_INVALID_ARG, "null output");
  for (int u = 0; u < units; ++u) unit_nparts[u] = 0;
  int n = 0;
  for (int s = 0; s < nseg; ++s) {
    const dq_segment& g = segs[s];
    if (g.unit < 0 || g.unit >= units) return fail(DQ_ERR_INVALID_ARG, "segment %d has unit %d", s, g.unit);
    if (g.r > kMaxR || g.r % 8 || g.i1 > 8 || g.i2p % 64) return fail(DQ_ERR_UNSUPPORTED, "segment %d plan unsupported", s);
    for (int b0 = 0; b0 < g.i2; b0 += chunk_b) {
      if (work) {
        work[2 * n] = s;
        work[2 * n + 1] = b0;
      }
      unit_nparts[g.unit]++;
      ++n;
    }
  }
  int acc = 0;
  for (int u = 0; u < units; ++u) {
    unit_part0[u] = acc;
    acc += unit_nparts[u];
  }
  if (work_part) {
    // second pass assigns slots in work-list order
    int* cursor = new int[units > 0 ? units : 1];
    for (int u = 0; u < units; ++u) cursor[u] = unit_part0[u];
    for (int i = 0; i < n; ++i) work_part[i] = cursor[segs[work[2 * i]].unit]++;
    delete[] cursor;
  }
  *nwork = n;
  *total_parts = acc;
  return DQ_OK;
}

extern "C" int dq_decode_attention(const dq_attn_args* h, void* stream) {
  if (!h) return fail(DQ_ERR_INVALID_ARG, "null args");
  const dq_attn_args& a = *h;
  if (a.units <= 0) return DQ_OK;
  if (!a.q || !a.out || (a.nwork > 0 && (!a.segs || !a.work || !a.work_part || !a.part_o || !a.part_ml)))
    return fail(DQ_ERR_INVALID_ARG, "dq_decode_attention: null pointer");
  if (!a.unit_part0 || !a.unit_nparts) return fail(DQ_ERR_INVALID_ARG, "dq_decode_attention: missing unit tables");
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

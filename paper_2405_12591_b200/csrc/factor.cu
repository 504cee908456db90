// K3 quantize-on-write: batched n=2 TT-SVD of K/V blocks in fp64, fused with the
// symmetric quantizer and packing (mpo.py:153-178 + compress.py:85-94 + quantize.py:123-151).
//
// For a block M (rows x cols) with plan i=(i1,i2), j=(j1,j2) the interleaved matrix
//   A[(a,c),(b,e)] = M[a*i2+b, c*j2+e]          (mpo.py:144-150, never materialised)
// is (m = i1*j1) x (n = i2*j2).  Its SVD is taken in Gram form on the short side
// (r = min(m,n) <= 64 because i1, j1 <= 8):
//   case A (m <= n):  G = A A^T (r x r), G = U diag(lambda) U^T,
//                     core0 = U sqrt(s), core1 = diag(s^-1/2) U^T A     (= sqrt(s) V^T)
//   case B (m >  n):  H = A^T A, H = V diag(lambda) V^T,
//                     core1 = sqrt(s) V^T, core0 = A V diag(s^-1/2)     (= U sqrt(s))
// with s = sqrt(lambda).  The eigensolver is a CTA-level parallel cyclic Jacobi
// (round-robin pairing, 32 disjoint rotations per round) in fp64 shared memory:
// the rotation angles are exactly those of one-sided (Hestenes) Jacobi on the rows
// of X, applied to the Gram form.  Everything runs in fp64 because one flipped
// int4 code moves the reconstruction by ~1e-3 relative.
//
// Sign convention: each singular vector is oriented so that its largest-magnitude
// entry of core0's column is positive (LAPACK's is implementation-defined; parity
// tests align signs per bond index).
#include "common.cuh"

namespace dq {

namespace {

constexpr int kR = 64;       // max bond dimension handled (i1, j1 <= 8)
constexpr int kTile = 64;    // contraction tile
constexpr int kThreads = 256;
constexpr int kMaxSweeps = 40;
// rotation threshold relative to sqrt(g_pp g_qq): ~20 ulp.  Rotations below it only stir the
// rounding noise of the converged matrix (a 1-ulp threshold can keep that going for dozens
// of sweeps); the eigenvectors it leaves are accurate to ~1e-14, far inside the 1e-5 factor
// tolerance
#ifndef DQ_JACOBI_TOL
#define DQ_JACOBI_TOL 2e-15
#endif
constexpr double kJacobiTol = DQ_JACOBI_TOL;

struct Dims {
  int rows, cols;
  int i1, i2, j1, j2;
  int m, n, r, kd;  // kd = contraction length of the Gram = max(m, n)
  bool caseA;       // m <= n
  int dtype;
  int64_t bstride;  // elements per block
};

Dims make_dims(const dq_plan2& p, int64_t rows, int64_t cols, int dtype) {
  Dims d;
  d.rows = (int)rows;
  d.cols = (int)cols;
  d.i1 = (int)p.i1;
  d.i2 = (int)p.i2;
  d.j1 = (int)p.j1;
  d.j2 = (int)p.j2;
  d.m = d.i1 * d.j1;
  d.n = d.i2 * d.j2;
  d.r = (int)p.r;
  d.caseA = d.m <= d.n;
  d.kd = d.caseA ? d.n : d.m;
  d.dtype = dtype;
  d.bstride = rows * cols;
  return d;
}

__device__ __forceinline__ double load_m(const void* base, int dtype, int64_t off) {
  if (dtype == DQ_F16) return (double)__half2float(((const __half*)base)[off]);
  return (double)((const float*)base)[off];
}

// A[row][col] of the interleaved matrix
__device__ __forceinline__ double load_a(const void* blk, const Dims& d, int row, int col) {
  const int a = row / d.j1, c = row - a * d.j1;
  const int b = col / d.j2, e = col - b * d.j2;
  return load_m(blk, d.dtype, (int64_t)(a * d.i2 + b) * d.cols + c * d.j2 + e);
}

// X[p][k]: the Gram operand (X = A in case A, A^T in case B), r x kd
__device__ __forceinline__ double load_x(const void* blk, const Dims& d, int p, int k) {
  return d.caseA ? load_a(blk, d, p, k) : load_a(blk, d, k, p);
}

__device__ __forceinline__ const void* block_ptr(const void* in, const Dims& d, int64_t blk) {
  const size_t es = d.dtype == DQ_F16 ? 2 : 4;
  return (const char*)in + (size_t)blk * d.bstride * es;
}

// ---- Gram: G[blk] += X[:, k0:k1] X[:, k0:k1]^T  (upper 4x4 tiles only) ------
__global__ void __launch_bounds__(kThreads) gram_kernel(const void* __restrict__ in, Dims d, int kchunk,
                                                        double* __restrict__ G, int32_t* flags) {
  __shared__ double xs[kTile][kR + 2];  // xs[k][p]
  const int64_t blk = blockIdx.x;
  const void* base = block_ptr(in, d, blk);
  const int k_begin = blockIdx.y * kchunk;
  const int k_end = min(d.kd, k_begin + kchunk);
  const int tp = threadIdx.x >> 4, tq = threadIdx.x & 15;
  const bool active = tq >= tp;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  bool nonfinite = false;
  for (int k0 = k_begin; k0 < k_end; k0 += kTile) {
    for (int idx = threadIdx.x; idx < kR * kTile; idx += kThreads) {
      const int p = idx / kTile, kk = idx - p * kTile;
      const int k = k0 + kk;
      double v = 0.0;
      if (p < d.r && k < k_end) {
        v = load_x(base, d, p, k);
        nonfinite |= !isfinite(v);
      }
      xs[kk][p] = v;
    }
    __syncthreads();
    if (active) {
#pragma unroll 4
      for (int kk = 0; kk < kTile; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a[i] = xs[kk][tp * 4 + i];
          b[i] = xs[kk][tq * 4 + i];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
    }
    __syncthreads();
  }
  if (nonfinite && flags) atomicOr(flags, (int)DQ_FLAG_NONFINITE);
  if (!active) return;
  double* g = G + blk * kR * kR;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int p = tp * 4 + i, q = tq * 4 + j;
      if (p < d.r && q < d.r && p <= q) atomicAdd(&g[p * kR + q], acc[i][j]);
    }
}

// ---- parallel cyclic Jacobi eigensolver on one r x r Gram per CTA ---------
// Round-robin (circle-method) ordering: every round rotates N/2 disjoint pairs (p, q).
// One round = (a) warp 0 computes the N/2 rotation angles, (b) every thread applies both
// sides of the rotation, G <- J^T G J, to its 2x2 blocks (pair i rows x pair j columns, i <= j,
// mirrored) and V <- V J to its column pairs: two CTA barriers per round.  The angle t is
// computed in fp32 on the fp64 entries scaled by 1/max(diag G) (an inexact angle only slows
// the annihilation, it is not an error), then c = (1 + t^2)^-1/2 by rsqrtf + two fp64 Newton
// steps and s = t c, so every rotation is orthogonal to fp64 rounding.  A pair is rotated
// while |g_pq| > max(1e-16 sqrt(|g_pp g_qq|), 1e-17 max(diag G)): the absolute floor stops
// rotations among numerically-zero eigenvalues (rank-deficient blocks: repeated or
// all-equal rows) that the relative test alone would chase forever.
struct JacobiSmem {
  double g[kR][kR + 1];
  double v[kR][kR + 1];
  double c[kR / 2], s[kR / 2];
  int pp[kR / 2], qq[kR / 2];
  double lam[kR];
  int perm[kR];
  int rotated;  // any rotation in the finished sweep
};

// 1 / sqrt(x) in fp64 from the fp32 estimate and one third-order step: with r = 1 - x y^2
// (|r| ~ 2^-22), y (1 - r)^(-1/2) = y (1 + r/2 + 3 r^2 / 8 + O(r^3)), truncation ~2^-68, so the
// result is as accurate as two Newton steps with 4 dependent fp64 operations instead of 6 (the
// plane rotations of the QL chases are a serial chain of them)
__device__ __forceinline__ double rsqrt_f64(double x) {
  const double y = (double)rsqrtf((float)x);
  const double r = fma(-x, y * y, 1.0);
  return fma(y * r, fma(r, 0.375, 0.5), y);
}

__global__ void __launch_bounds__(kThreads) jacobi_kernel(const double* __restrict__ G, Dims d,
                                                          double* __restrict__ U, double* __restrict__ lam_out,
                                                          int32_t* flags) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JacobiSmem& sm = *reinterpret_cast<JacobiSmem*>(smem_raw);
  const int64_t blk = blockIdx.x;
  const int r = d.r;
  const int N = (r + 1) & ~1;  // even number of players (a dummy index when r is odd)
  const int npairs = N / 2;
  const double* g = G + blk * kR * kR;
  for (int idx = threadIdx.x; idx < kR * kR; idx += blockDim.x) {
    const int p = idx / kR, q = idx % kR;
    double val = 0.0;
    if (p < r && q < r) val = p <= q ? g[p * kR + q] : g[q * kR + p];
    sm.g[p][q] = val;
    sm.v[p][q] = p == q ? 1.0 : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // max diagonal: the scale of the angle arithmetic
    double m = 0.0;
    for (int p = threadIdx.x; p < r; p += 32) m = fmax(m, fabs(sm.g[p][p]));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) sm.lam[0] = m;
  }
  __syncthreads();
  const double gmax = sm.lam[0];
  const double inv_gmax = gmax > 0.0 ? 1.0 / gmax : 0.0;
  const double abs_floor = 1e-17 * gmax;
  // blocks (i, j), i <= j, of the pair grid: npairs * (npairs + 1) / 2 per round
  const int nblocks = npairs * (npairs + 1) / 2;

  bool converged = gmax == 0.0;
  int sweep = 0;
  for (; sweep < kMaxSweeps && !converged; ++sweep) {
    bool rot = false;  // warp 0: any rotation this sweep
    for (int round = 0; round < N - 1; ++round) {
      if (threadIdx.x < 32) {
        for (int i = threadIdx.x; i < npairs; i += 32) {
          // circle method: slot 0 fixed, slots 1..N-1 rotate by `round`
          const int sa = i, sb = N - 1 - i;
          const int pa = sa == 0 ? 0 : ((sa - 1 + round) % (N - 1)) + 1;
          const int pb = ((sb - 1 + round) % (N - 1)) + 1;
          const int p = min(pa, pb), q = max(pa, pb);
          double cc = 1.0, ss = 0.0;
          if (q < r) {
            const double app = sm.g[p][p], aqq = sm.g[q][q], apq = sm.g[p][q];
            const double thr = fmax(kJacobiTol * sqrt(fabs(app) * fabs(aqq)), abs_floor);
            if (fabs(apq) > thr) {
              // sym.schur2 (Golub & Van Loan 8.4.2) with tau in fp32
              const float tau = (float)((aqq - app) * inv_gmax) / (2.f * (float)(apq * inv_gmax));
              const float at = fabsf(tau);
              const float t = at > 1e15f ? 0.5f / tau : copysignf(1.f, tau) / (at + sqrtf(fmaf(tau, tau, 1.f)));
              const double td = (double)t;
              cc = rsqrt_f64(fma(td, td, 1.0));
              ss = td * cc;
              rot |= ss != 0.0;
            }
          }
          sm.pp[i] = p;
          sm.qq[i] = q;
          sm.c[i] = cc;
          sm.s[i] = ss;
        }
      }
      __syncthreads();
      // G <- J^T G J on 2x2 blocks (rows of pair i, columns of pair j), mirrored below the diagonal
      for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
        // b -> (i, j) with i <= j: row-major over the upper triangle
        int i = 0, rem = b;
        while (rem >= npairs - i) {
          rem -= npairs - i;
          ++i;
        }
        const int j = i + rem;
        const double si = sm.s[i], sj = sm.s[j];
        if (si == 0.0 && sj == 0.0) continue;
        const int pi = sm.pp[i], qi = sm.qq[i], pj = sm.pp[j], qj = sm.qq[j];
        if (qi >= r || qj >= r) continue;
        const double ci = sm.c[i], cj = sm.c[j];
        const double a = sm.g[pi][pj], bq = sm.g[pi][qj], cq = sm.g[qi][pj], dd = sm.g[qi][qj];
        // left: rows (pi, qi) by pair i
        const double l0 = ci * a - si * cq, l1 = ci * bq - si * dd;
        const double l2 = si * a + ci * cq, l3 = si * bq + ci * dd;
        // right: columns (pj, qj) by pair j
        const double n00 = cj * l0 - sj * l1, n01 = sj * l0 + cj * l1;
        const double n10 = cj * l2 - sj * l3, n11 = sj * l2 + cj * l3;
        sm.g[pi][pj] = n00;
        sm.g[pi][qj] = n01;
        sm.g[qi][pj] = n10;
        sm.g[qi][qj] = n11;
        if (i != j) {
          sm.g[pj][pi] = n00;
          sm.g[qj][pi] = n01;
          sm.g[pj][qi] = n10;
          sm.g[qj][qi] = n11;
        } else {
          sm.g[qi][pi] = n01;  // diagonal block: keep it exactly symmetric
        }
      }
      // V <- V J: rows k, column pairs j
      for (int idx = threadIdx.x; idx < npairs * r; idx += blockDim.x) {
        const int j = idx / r, k = idx - j * r;
        const double sj = sm.s[j];
        if (sj == 0.0 || sm.qq[j] >= r) continue;
        const int p = sm.pp[j], q = sm.qq[j];
        const double cj = sm.c[j];
        const double vp = sm.v[k][p], vq = sm.v[k][q];
        sm.v[k][p] = cj * vp - sj * vq;
        sm.v[k][q] = sj * vp + cj * vq;
      }
      __syncthreads();
    }
    if (threadIdx.x < 32) {
      rot = __any_sync(0xffffffffu, rot);
      if (threadIdx.x == 0) sm.rotated = rot;
    }
    __syncthreads();
    converged = !sm.rotated;
  }
#ifdef DQ_JACOBI_STATS  // measurement builds: sweeps of the first blocks
  if (threadIdx.x == 0 && blk < 4) printf("jacobi block %d: converged %d after %d sweeps\n", (int)blk, (int)converged, sweep);
#endif
  if (!converged && threadIdx.x == 0 && flags) atomicOr(flags, (int)DQ_FLAG_JACOBI_NOCONV);

  // sort eigenvalues descending (ties by index), orient each vector
  if (threadIdx.x < r) {
    const int i = threadIdx.x;
    auto key = [](double x) { return x == x ? x : -INFINITY; };
    const double li = key(sm.g[i][i]);
    int rank = 0;
    for (int j = 0; j < r; ++j) {
      const double lj = key(sm.g[j][j]);
      rank += (lj > li) || (lj == li && j < i);
    }
    sm.perm[rank] = i;
  }
  __syncthreads();
  double* u = U + blk * kR * kR;
  for (int col = threadIdx.x / 32; col < r; col += blockDim.x / 32) {
    const int src = sm.perm[col];
    // largest |v| entry (first on ties) decides the sign
    double best = -1.0;
    int bidx = 0;
    for (int p = threadIdx.x & 31; p < r; p += 32) {
      const double a = fabs(sm.v[p][src]);
      if (a > best) { best = a; bidx = p; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    const double sgn = sm.v[bidx][src] < 0.0 ? -1.0 : 1.0;
    for (int p = threadIdx.x & 31; p < r; p += 32) u[p * kR + col] = sgn * sm.v[p][src];
    if ((threadIdx.x & 31) == 0) lam_out[blk * kR + col] = sm.g[src][src];
  }
}

// ---- tridiagonal eigensolver on one r x r Gram per CTA (the default) -------------------
// Householder reduction to tridiagonal form with the transformation accumulated in place
// (EISPACK tred2), then implicit QL with Wilkinson-type shifts on the tridiagonal (tqli).
// About 30x less shared-memory traffic than the cyclic Jacobi above (which moves the whole
// r x r G and V per round, ~570 rounds): the 64-thread CTA parallelises every row / column
// loop of the reduction; the QL bulge chases run on thread 0 and record their rotations,
// which every thread then applies to its own row of the eigenvector matrix.  Plane
// rotations use rsqrt (fp32 seed + two fp64 Newton steps), exactly orthogonal to fp64
// rounding.  Eigenvalues are sorted descending and the vectors oriented as in jacobi_kernel.
constexpr int kEigThreads = 64;

struct EigSmem {
  double a[kR][kR + 1];  // the matrix, then the accumulated transformation / eigenvectors
  double d[kR], e[kR];
  double rc[2][kR], rs[2][kR];  // rotations of two QL chases (double-buffered), by index i
  double red[kEigThreads / 32];
  double sh[4];          // broadcast scalars
  int ish[2][4];
  int perm[kR];
};

__device__ __forceinline__ double eig_block_sum(double v, EigSmem& sm) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();  // red[] from any previous reduction has been read
  if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < kEigThreads / 32; ++w) s += sm.red[w];
  return s;
}

// 1 / sqrt(f^2 + g^2) and the hypotenuse
__device__ __forceinline__ double hyp(double f, double g, double* rinv) {
  const double q = fma(f, f, g * g);
  if (q > 1e-30 && q < 1e30) {
    const double ri = rsqrt_f64(q);
    *rinv = ri;
    return q * ri;
  }
  const double r = sqrt(q);
  *rinv = r > 0.0 ? 1.0 / r : 0.0;
  return r;
}

__global__ void __launch_bounds__(kEigThreads) eig_tql_kernel(const double* __restrict__ G, Dims d_,
                                                              double* __restrict__ U, double* __restrict__ lam_out,
                                                              int32_t* flags) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EigSmem& sm = *reinterpret_cast<EigSmem*>(smem_raw);
  const int64_t blk = blockIdx.x;
  const int n = d_.r;
  const int t = threadIdx.x;
  const double* g = G + blk * kR * kR;
  for (int idx = t; idx < n * n; idx += kEigThreads) {
    const int p = idx / n, q = idx % n;
    sm.a[p][q] = p <= q ? g[p * kR + q] : g[q * kR + p];
  }
  __syncthreads();

  // ---- Householder reduction (tred2), rows i = n-1 .. 1 ----------------------------------
  for (int i = n - 1; i > 0; --i) {
    const int l = i - 1;
    double h = 0.0;
    if (l > 0) {
      double part = 0.0;
      for (int k = t; k <= l; k += kEigThreads) part += fabs(sm.a[i][k]);
      const double scale = eig_block_sum(part, sm);
      if (scale == 0.0) {
        if (t == 0) sm.e[i] = sm.a[i][l];
      } else {
        part = 0.0;
        for (int k = t; k <= l; k += kEigThreads) {
          const double v = sm.a[i][k] / scale;
          sm.a[i][k] = v;
          part += v * v;
        }
        h = eig_block_sum(part, sm);
        const double f = sm.a[i][l];
        const double gg = f >= 0.0 ? -sqrt(h) : sqrt(h);
        h -= f * gg;
        __syncthreads();  // every thread has read a[i][l]
        if (t == 0) {
          sm.e[i] = scale * gg;
          sm.a[i][l] = f - gg;
        }
        __syncthreads();
        const double hinv = 1.0 / h;
        part = 0.0;
        for (int j = t; j <= l; j += kEigThreads) {
          sm.a[j][i] = sm.a[i][j] * hinv;
          double acc = 0.0;
          for (int k = 0; k <= j; ++k) acc = fma(sm.a[j][k], sm.a[i][k], acc);
          for (int k = j + 1; k <= l; ++k) acc = fma(sm.a[k][j], sm.a[i][k], acc);
          const double ej = acc * hinv;
          sm.e[j] = ej;
          part = fma(ej, sm.a[i][j], part);
        }
        const double ff = eig_block_sum(part, sm);
        const double hh = ff / (h + h);
        for (int j = t; j <= l; j += kEigThreads) sm.e[j] = fma(-hh, sm.a[i][j], sm.e[j]);
        __syncthreads();
        for (int j = t; j <= l; j += kEigThreads) {
          const double fj = sm.a[i][j], gj = sm.e[j];
          for (int k = 0; k <= j; ++k) sm.a[j][k] -= fma(fj, sm.e[k], gj * sm.a[i][k]);
        }
      }
    } else {
      if (t == 0) sm.e[i] = sm.a[i][l];
    }
    if (t == 0) sm.d[i] = h;
    __syncthreads();
  }
  if (t == 0) {
    sm.d[0] = 0.0;
    sm.e[0] = 0.0;
  }
  __syncthreads();
#if defined(DQ_EIG_STOP) && DQ_EIG_STOP == 1  // measurement only: the reduction alone
  return;
#endif
  // accumulate the transformations: a <- Q
  for (int i = 0; i < n; ++i) {
    const int l = i - 1;
    if (sm.d[i] != 0.0) {
      for (int j = t; j <= l; j += kEigThreads) {
        double acc = 0.0;
        for (int k = 0; k <= l; ++k) acc = fma(sm.a[i][k], sm.a[k][j], acc);
        for (int k = 0; k <= l; ++k) sm.a[k][j] = fma(-acc, sm.a[k][i], sm.a[k][j]);
      }
    }
    __syncthreads();
    if (t == 0) {
      sm.d[i] = sm.a[i][i];
      sm.a[i][i] = 1.0;
    }
    for (int j = t; j <= l; j += kEigThreads) sm.a[j][i] = sm.a[i][j] = 0.0;
    __syncthreads();
  }

#if defined(DQ_EIG_STOP) && DQ_EIG_STOP == 2  // measurement only: reduction + accumulation
  return;
#endif
  // ---- implicit QL on (d, e) (tqli), eigenvectors in the rows of a --------------------
  // Thread 0 runs the bulge chases back to back, recording each chase's rotations into one of
  // two buffers; warp 1 applies chase c - 1 to the eigenvector rows (two per lane) while
  // thread 0 computes chase c: one barrier per chase, and the row updates leave the serial
  // path.  The chase keeps its state in registers and loads the next step's d / e one step
  // ahead (a step reads only entries the chase has not written yet).
  if (t == 0) {
    for (int i = 1; i < n; ++i) sm.e[i - 1] = sm.e[i];
    sm.e[n - 1] = 0.0;
  }
  __syncthreads();
  bool failed = false;
  int ql_l = 0, ql_iter = 0;  // thread 0: the eigenvalue being isolated, its iterations
  for (int c = 0;; ++c) {
    const int buf = c & 1;
    if (t == 0) {
      int status = 1, lo = 0, hi = 0;  // 0: a chase on rotations [lo, hi), 1: done, 2: no convergence
      while (ql_l < n) {
        const int l = ql_l;
        int m = l;
        for (; m < n - 1; ++m) {
          const double dd = fabs(sm.d[m]) + fabs(sm.d[m + 1]);
          if (fabs(sm.e[m]) <= 2.220446049250313e-16 * dd) break;
        }
        if (m == l) {
          ++ql_l;
          ql_iter = 0;
          continue;
        }
        if (ql_iter++ >= 40) {
          status = 2;
          break;
        }
        double gq = (sm.d[l + 1] - sm.d[l]) / (2.0 * sm.e[l]);
        double ri;
        double r = hyp(gq, 1.0, &ri);
        gq = sm.d[m] - sm.d[l] + sm.e[l] / (gq + copysign(r, gq));
        double s = 1.0, cc = 1.0, p = 0.0;
        int i = m - 1;
        double ei = sm.e[i], di1 = sm.d[i + 1], di = sm.d[i];
        bool deflated = false;
        for (; i >= l; --i) {
          const double ei_n = i > l ? sm.e[i - 1] : 0.0, di_n = i > l ? sm.d[i - 1] : 0.0;
          const double f = s * ei, b = cc * ei;
          r = hyp(f, gq, &ri);
          sm.e[i + 1] = r;
          if (r == 0.0) {
            sm.d[i + 1] -= p;
            sm.e[m] = 0.0;
            deflated = true;
            break;
          }
          s = f * ri;
          cc = gq * ri;
          gq = di1 - p;
          r = (di - gq) * s + 2.0 * cc * b;
          p = s * r;
          sm.d[i + 1] = gq + p;
          gq = cc * r - b;
          sm.rc[buf][i] = cc;
          sm.rs[buf][i] = s;
          ei = ei_n;
          di1 = di;
          di = di_n;
        }
        lo = deflated ? i + 1 : l;
        hi = m;
        if (!deflated) {
          sm.d[l] -= p;
          sm.e[l] = gq;
          sm.e[m] = 0.0;
        }
        status = 0;
        break;
      }
      sm.ish[buf][0] = lo;
      sm.ish[buf][1] = hi;
      sm.ish[buf][2] = status;
    }
    if (t >= 32 && c > 0 && sm.ish[buf ^ 1][2] == 0) {
      // chase c - 1 on rows t - 32 and t (i = hi - 1 .. lo, the chase's own order)
      const int lo = sm.ish[buf ^ 1][0], hi = sm.ish[buf ^ 1][1];
      const double* rcs = sm.rc[buf ^ 1];
      const double* rss = sm.rs[buf ^ 1];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row_i = t - 32 + 32 * h;
        if (row_i < n) {
          double* row = sm.a[row_i];
          double nxt = row[hi];
          for (int i = hi - 1; i >= lo; --i) {
            const double c_ = rcs[i], s_ = rss[i];
            const double cur = row[i];
            row[i + 1] = fma(s_, cur, c_ * nxt);
            nxt = fma(c_, cur, -s_ * nxt);
          }
          row[lo] = nxt;
        }
      }
    }
    __syncthreads();
    const int status = sm.ish[buf][2];
    if (status != 0) {
      failed = status == 2;
      break;
    }
  }
  if (failed && t == 0 && flags) atomicOr(flags, (int)DQ_FLAG_JACOBI_NOCONV);
#ifdef DQ_EIG_STATS  // measurement only: QL chases of the first blocks
  if (t == 0 && blk < 4) printf("eig block %d: n %d\n", (int)blk, n);
#endif

  // sort eigenvalues descending (ties by index), orient each vector (as jacobi_kernel)
  if (t < n) {  // a NaN (non-finite input, already flagged) sorts last: perm stays a permutation
    auto key = [](double x) { return x == x ? x : -INFINITY; };
    const double li = key(sm.d[t]);
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = key(sm.d[j]);
      rank += (lj > li) || (lj == li && j < t);
    }
    sm.perm[rank] = t;
  }
  __syncthreads();
  double* u = U + blk * kR * kR;
  for (int col = t / 32; col < n; col += kEigThreads / 32) {
    const int src = sm.perm[col];
    double best = -1.0;
    int bidx = 0;
    for (int p = t & 31; p < n; p += 32) {
      const double a = fabs(sm.a[p][src]);
      if (a > best) { best = a; bidx = p; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    const double sgn = sm.a[bidx][src] < 0.0 ? -1.0 : 1.0;
    for (int p = t & 31; p < n; p += 32) u[p * kR + col] = sgn * sm.a[p][src];
    if ((t & 31) == 0) lam_out[blk * kR + col] = sm.d[src];
  }
}

// singular value from an eigenvalue, with rank-deficiency cut (see file header)
__device__ __forceinline__ double sval(const double* lam, int k) {
  const double l0 = lam[0];
  const double lk = lam[k];
  if (!(lk > 0.0) || lk <= 1e-13 * l0) return 0.0;
  return sqrt(lk);
}

// ---- case A projection: core1 = diag(s^-1/2) U^T A, core0 = U sqrt(s) ---------
// grid (nblk, nsplit over the n columns); thread tile 4 (bond) x 4 (columns)
__global__ void __launch_bounds__(kThreads) project_a_kernel(const void* __restrict__ in, Dims d, int cchunk,
                                                             const double* __restrict__ U,
                                                             const double* __restrict__ lam,
                                                             float* __restrict__ core0, float* __restrict__ core1,
                                                             unsigned* __restrict__ amax) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double (*ws)[kR + 2] = reinterpret_cast<double (*)[kR + 2]>(smem_raw);  // ws[p][k] = U[p][k] / sqrt(s_k)
  double (*xs)[kTile + 2] =
      reinterpret_cast<double (*)[kTile + 2]>(smem_raw + sizeof(double) * kR * (kR + 2));  // xs[p][col]
  const int64_t blk = blockIdx.x;
  const void* base = block_ptr(in, d, blk);
  const double* u = U + blk * kR * kR;
  const double* lm = lam + blk * kR;
  const int r = d.r;
  for (int idx = threadIdx.x; idx < kR * kR; idx += kThreads) {
    const int p = idx / kR, k = idx % kR;
    double v = 0.0;
    if (p < r && k < r) {
      const double s = sval(lm, k);
      v = s > 0.0 ? u[p * kR + k] / sqrt(s) : 0.0;
    }
    ws[p][k] = v;
  }
  if (blockIdx.y == 0) {
    for (int idx = threadIdx.x; idx < r * r; idx += kThreads) {
      const int p = idx / r, k = idx % r;
      core0[blk * (int64_t)d.m * r + idx] = (float)(u[p * kR + k] * sqrt(sval(lm, k)));
    }
  }
  const int c_begin = blockIdx.y * cchunk;
  const int c_end = min(d.n, c_begin + cchunk);
  const int tk = threadIdx.x >> 4, tc = threadIdx.x & 15;
  float local_max = 0.f;
  float* out = core1 + blk * (int64_t)r * d.n;
  for (int c0 = c_begin; c0 < c_end; c0 += kTile) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kR * kTile; idx += kThreads) {
      const int p = idx / kTile, cc = idx - p * kTile;
      const int col = c0 + cc;
      xs[p][cc] = (p < r && col < c_end) ? load_a(base, d, p, col) : 0.0;
    }
    __syncthreads();
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int p = 0; p < r; ++p) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = ws[p][tk * 4 + i];
        b[i] = xs[p][tc * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = tk * 4 + i;
      if (k >= r) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = c0 + tc * 4 + j;
        if (col < c_end) {
          const float v = (float)acc[i][j];
          out[(int64_t)k * d.n + col] = v;
          local_max = fmaxf(local_max, fabsf(v));
        }
      }
    }
  }
  for (int o = 16; o; o >>= 1) local_max = fmaxf(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&amax[blk], __float_as_uint(local_max));
}

// ---- case B (n < m, tiny blocks): core1 = sqrt(s) V^T, core0 = A V diag(s^-1/2) ----
__global__ void __launch_bounds__(kThreads) project_b_kernel(const void* __restrict__ in, Dims d,
                                                             const double* __restrict__ V,
                                                             const double* __restrict__ lam,
                                                             float* __restrict__ core0, float* __restrict__ core1,
                                                             unsigned* __restrict__ amax) {
  const int64_t blk = blockIdx.x;
  const void* base = block_ptr(in, d, blk);
  const double* v = V + blk * kR * kR;
  const double* lm = lam + blk * kR;
  const int r = d.r;  // == n
  float local_max = 0.f;
  for (int idx = threadIdx.x; idx < r * d.n; idx += kThreads) {
    const int k = idx / d.n, col = idx % d.n;
    const float val = (float)(sqrt(sval(lm, k)) * v[col * kR + k]);
    core1[blk * (int64_t)r * d.n + idx] = val;
    local_max = fmaxf(local_max, fabsf(val));
  }
  for (int idx = threadIdx.x; idx < d.m * r; idx += kThreads) {
    const int row = idx / r, k = idx % r;
    const double s = sval(lm, k);
    double acc = 0.0;
    if (s > 0.0)
      for (int col = 0; col < d.n; ++col) acc = fma(load_a(base, d, row, col), v[col * kR + k], acc);
    core0[blk * (int64_t)d.m * r + idx] = s > 0.0 ? (float)(acc / sqrt(s)) : 0.f;
  }
  for (int o = 16; o; o >>= 1) local_max = fmaxf(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&amax[blk], __float_as_uint(local_max));
}

// ---- quantize + pack core1 into the requested layout (quantize.py:123-151) ----
__global__ void quantize_core_kernel(const float* __restrict__ core1, int64_t core_elems, CoreGeom geom,
                                     int64_t out_bytes, const unsigned* __restrict__ amax,
                                     uint8_t* __restrict__ payload, int64_t payload_stride,
                                     float* __restrict__ scale, int32_t* flags) {
  const int64_t blk = blockIdx.y;
  const int bits = geom.bits;
  const int per = 8 / bits;
  const int qmax = (1 << (bits - 1)) - 1;
  const float amax_f = __uint_as_float(amax[blk]);
  if (!isfinite(amax_f)) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && flags) atomicOr(flags, (int)DQ_FLAG_NONFINITE);
  }
  const double am = (double)amax_f;
  bool degenerate;
  const float sc = rtn_scale(am, qmax, &degenerate);
  if (blockIdx.x == 0 && threadIdx.x == 0) scale[blk] = sc;
  const float* src = core1 + blk * core_elems;
  uint8_t* dst = payload + blk * payload_stride;
  const double rinv = am > 0.0 ? 1.0 / am : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < out_bytes; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned v = 0;
    for (int k = 0; k < per; ++k) {
      const int64_t slot = i * per + k;
      if (slot >= geom_slots(geom)) break;
      int rr, b, e;
      int code = 0;  // padding slots and degenerate blocks hold the code 0
      if (geom_coords(geom, slot, rr, b, e) && !degenerate)
        code = rtn_code_fast(src[((int64_t)rr * geom.i2 + b) * geom.j2 + e], qmax, am, rinv);
      v |= geom_encode(code, geom) << (k * bits);
    }
    dst[i] = (uint8_t)v;
  }
}

// ---- fast path for 128-wide rows (j = (8, 16), m = 8 i1 <= n = 16 i2): X tiles ------------
// X[p = (a, c)][k = (b, e)] = M[a i2 + b][16 c + e].  A chunk of kNb b values is gathered from
// i1 * kNb whole rows of M with 16-byte coalesced loads (the interleave is the scatter into
// shared memory), converted to fp64 once, and contracted by a 16 x 16 grid of threads with
// 4 x 4 register tiles: a warp spans 4 x 8 tiles, so its fp64 operand loads are broadcasts
// (4 shared-memory wavefronts per 16 DFMA per k).  The next chunk's loads are in flight while
// the current one is contracted.
constexpr int kNb = 4;             // b values per chunk: 64 k columns
constexpr int kXk = 16 * kNb;      // k columns per chunk
constexpr int kXp = kR + 2;        // padded p pitch (doubles) of xs[k][p]
constexpr int kXpP = kR + 4;       // pitch (doubles) of the DMMA operand tiles: 136 words = 8 banks
                                   // per row, so a fragment (8 rows x 4 consecutive) hits 64 distinct
                                   // bank slots (two wavefronts, no conflict)
// 16-byte loads per thread per chunk: i1 <= 8 rows a x kNb rows b x (16 | 32) uint4 per row
template <bool F16>
constexpr int kXLoads = 8 * kNb * (F16 ? 16 : 32) / kThreads;

template <bool F16>
struct XTile {
  uint4 v[kXLoads<F16>];
};

// issue the loads of chunk [b0, b0 + kNb) (rows a*i2 + b, a < i1); rows outside read as 0
template <bool F16>
__device__ __forceinline__ void xtile_load(XTile<F16>& t, const void* blk, const Dims& d, int b0) {
  constexpr int per_row = F16 ? 16 : 32;
#pragma unroll
  for (int j = 0; j < kXLoads<F16>; ++j) {
    const int idx = threadIdx.x + j * kThreads;  // (a, b_local, q)
    const int q = idx % per_row, ab = idx / per_row;
    const int a = ab / kNb, b = b0 + ab % kNb;
    t.v[j] = make_uint4(0u, 0u, 0u, 0u);
    if (a < d.i1 && b < d.i2) {
      const uint4* row =
          reinterpret_cast<const uint4*>((const char*)blk + (size_t)(a * d.i2 + b) * d.cols * (F16 ? 2 : 4));
      t.v[j] = __ldg(row + q);
    }
  }
}

// scatter the loaded chunk into shared memory as fp64: PK = true: xs[p = (a, c)][k = (b_local, e)]
// (the Gram's operand, both fragments read along k), PK = false: xs[k][p] (the projection's B)
template <bool F16, bool PK>
__device__ __forceinline__ void xtile_store(const XTile<F16>& t, double* xs) {
  constexpr int per_row = F16 ? 16 : 32;
#pragma unroll
  for (int j = 0; j < kXLoads<F16>; ++j) {
    const int idx = threadIdx.x + j * kThreads;
    const int q = idx % per_row, ab = idx / per_row;
    const int a = ab / kNb, bl = ab % kNb;
    constexpr int NE = F16 ? 8 : 4;  // consecutive e per 16-byte load
    const int c = q / (16 / NE), e0 = (q % (16 / NE)) * NE;
    double v[NE];
    if constexpr (F16) {
      const __half2* h = reinterpret_cast<const __half2*>(&t.v[j]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 f = __half22float2(h[u]);
        v[2 * u] = (double)f.x;
        v[2 * u + 1] = (double)f.y;
      }
    } else {
      const float* f = reinterpret_cast<const float*>(&t.v[j]);
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (double)f[u];
    }
    const int p = a * 8 + c, k0 = bl * 16 + e0;
    if constexpr (PK) {
      double2* dst = reinterpret_cast<double2*>(xs + p * kXpP + k0);
#pragma unroll
      for (int u = 0; u < NE / 2; ++u) dst[u] = make_double2(v[2 * u], v[2 * u + 1]);
    } else {
#pragma unroll
      for (int u = 0; u < NE; ++u) xs[(k0 + u) * kXpP + p] = v[u];
    }
  }
}

// D(8x8) += A(8x4, row) . B(4x8, col) in fp64 on the tensor pipe.  Fragments: a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], d = D[lane/4][2 (lane%4) + {0, 1}]
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <bool F16>
__device__ __forceinline__ bool xtile_finite(const XTile<F16>& t) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < kXLoads<F16>; ++j) {
    if constexpr (F16) {
      const __half2* h = reinterpret_cast<const __half2*>(&t.v[j]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 f = __half22float2(h[u]);
        ok &= isfinite(f.x) && isfinite(f.y);
      }
    } else {
      const float* f = reinterpret_cast<const float*>(&t.v[j]);
#pragma unroll
      for (int u = 0; u < 4; ++u) ok &= isfinite(f[u]);
    }
  }
  return ok;
}

// thread (tp, tq) of the 16 x 16 tile grid: a warp spans 4 tp x 8 tq
__device__ __forceinline__ void tile_coords(int& tp, int& tq) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  tp = (w >> 1) * 4 + (l >> 3);
  tq = (w & 1) * 8 + (l & 7);
}

// G[blk] (+)= X X^T over b in [b_begin, b_end) on the fp64 tensor pipe (DMMA m8n8k4): warp w
// owns the 8 x 64 row strip w of G (8 accumulator tiles); per k-step of 4 it loads one A
// fragment and 8 B fragments (all from xs[p][k]).  grid (nblk, splits); atomics only when split
template <bool F16>
__global__ void __launch_bounds__(kThreads) gram128_kernel(const void* __restrict__ in, Dims d, int bchunk,
                                                           double* __restrict__ G, int32_t* flags) {
  __shared__ __align__(16) double xs[kR * kXpP];
  const int64_t blk = blockIdx.x;
  const void* base = block_ptr(in, d, blk);
  const int b_begin = blockIdx.y * bchunk, b_end = min(d.i2, b_begin + bchunk);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  bool finite = true;
  XTile<F16> t;
  if (b_begin < b_end) xtile_load(t, base, d, b_begin);
  const double* arow = xs + (w * 8 + g) * kXpP + t4;
  for (int b0 = b_begin; b0 < b_end; b0 += kNb) {
    __syncthreads();  // the previous chunk is consumed
    finite &= xtile_finite(t);
    xtile_store<F16, true>(t, xs);
    __syncthreads();
    if (b0 + kNb < b_end) xtile_load(t, base, d, b0 + kNb);  // in flight during the contraction
    const int kn = min(kNb, b_end - b0) * 16;
#pragma unroll 2
    for (int k = 0; k < kn; k += 4) {
      const double a = arow[k];
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], a, xs[(j * 8 + g) * kXpP + k + t4]);
    }
  }
  if (!finite && flags) atomicOr(flags, (int)DQ_FLAG_NONFINITE);
  double* gp = G + blk * kR * kR;
  const int p = w * 8 + g;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int q = j * 8 + 2 * t4 + i;
      if (p < d.r && q < d.r && p <= q) {
        if (gridDim.y > 1) atomicAdd(&gp[p * kR + q], acc[j][i]);
        else gp[p * kR + q] = acc[j][i];
      }
    }
}

// case A projection on 128-wide rows: core1[k][(b, e)] = sum_p U[p][k] / sqrt(s_k) X[p][(b, e)] on the
// fp64 tensor pipe: A = W^T from ws[k][p], B = X from xs[col][p]; warp w owns the bond rows
// 8w..8w+7 x the chunk's 64 columns.  grid (nblk, splits over b)
template <bool F16>
__global__ void __launch_bounds__(kThreads) project128_kernel(const void* __restrict__ in, Dims d, int bchunk,
                                                              const double* __restrict__ U,
                                                              const double* __restrict__ lam,
                                                              float* __restrict__ core0, float* __restrict__ core1,
                                                              unsigned* __restrict__ amax) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* ws = reinterpret_cast<double*>(smem_raw);  // ws[k][p] = U[p][k] / sqrt(s_k)
  double* xs = ws + kR * kXpP;                        // xs[col][p]
  const int64_t blk = blockIdx.x;
  const void* base = block_ptr(in, d, blk);
  const double* u = U + blk * kR * kR;
  const double* lm = lam + blk * kR;
  const int r = d.r;
  const int b_begin = blockIdx.y * bchunk, b_end = min(d.i2, b_begin + bchunk);
  XTile<F16> t;
  if (b_begin < b_end) xtile_load(t, base, d, b_begin);
  for (int idx = threadIdx.x; idx < kR * kR; idx += kThreads) {
    const int p = idx / kR, k = idx % kR;
    double v = 0.0;
    if (p < r && k < r) {
      const double sk = sval(lm, k);
      v = sk > 0.0 ? u[p * kR + k] / sqrt(sk) : 0.0;
    }
    ws[k * kXpP + p] = v;
  }
  if (blockIdx.y == 0) {
    for (int idx = threadIdx.x; idx < r * r; idx += kThreads) {
      const int p = idx / r, k = idx % r;
      core0[blk * (int64_t)d.m * r + idx] = (float)(u[p * kR + k] * sqrt(sval(lm, k)));
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const double* arow = ws + (w * 8 + g) * kXpP + t4;
  float local_max = 0.f;
  float* out = core1 + blk * (int64_t)r * d.n;
  for (int b0 = b_begin; b0 < b_end; b0 += kNb) {
    __syncthreads();
    xtile_store<F16, false>(t, xs);
    __syncthreads();
    if (b0 + kNb < b_end) xtile_load(t, base, d, b0 + kNb);
    double acc[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 2
    for (int p = 0; p < r; p += 4) {
      const double a = arow[p];
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], a, xs[(j * 8 + g) * kXpP + p + t4]);
    }
    const int k = w * 8 + g, ncol = min(kNb, b_end - b0) * 16;
    if (k < r) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = j * 8 + 2 * t4;
        if (c < ncol) {
          const float2 v = make_float2((float)acc[j][0], (float)acc[j][1]);
          *reinterpret_cast<float2*>(&out[(int64_t)k * d.n + b0 * 16 + c]) = v;
          local_max = fmaxf(local_max, fmaxf(fabsf(v.x), fabsf(v.y)));
        }
      }
    }
  }
  for (int o = 16; o; o >>= 1) local_max = fmaxf(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&amax[blk], __float_as_uint(local_max));
}

// ---- quantize + pack into the attention layouts, j2 = 16 (every 128-wide KV block) ----------
// One thread per 16-code run of the destination: KTILE rows (bt, rr, swizzled b) hold 16 e,
// VTILE runs (bt, rr, e) hold 16 consecutive b.  The coordinates come from one 32-bit
// division per run instead of three 64-bit ones per code (quantize_core_kernel, any layout).
template <int BITS, bool VT>
__global__ void __launch_bounds__(kThreads) quantize_tile16_kernel(const float* __restrict__ core1, int64_t core_elems,
                                                                   CoreGeom geom, const unsigned* __restrict__ amax,
                                                                   uint8_t* __restrict__ payload,
                                                                   int64_t payload_stride, float* __restrict__ scale,
                                                                   int32_t* flags) {
  constexpr int kQmax = (1 << (BITS - 1)) - 1, kX = 1 << (BITS - 1), kMask = (1 << BITS) - 1;
  const int64_t blk = blockIdx.y;
  const float amax_f = __uint_as_float(amax[blk]);
  if (!isfinite(amax_f) && blockIdx.x == 0 && threadIdx.x == 0 && flags) atomicOr(flags, (int)DQ_FLAG_NONFINITE);
  const double am = (double)amax_f;
  bool degenerate;
  const float sc = rtn_scale(am, kQmax, &degenerate);
  if (blockIdx.x == 0 && threadIdx.x == 0) scale[blk] = sc;
  const double rinv = am > 0.0 ? 1.0 / am : 0.0;
  const float* src = core1 + blk * core_elems;
  uint8_t* dst = payload + blk * payload_stride;
  const int r = geom.r, i2 = geom.i2;
  const int runs = r * (geom.i2p / kI2Pad) * (VT ? 16 * 4 : kI2Pad);  // 16-code runs per core
  for (int run = blockIdx.x * kThreads + threadIdx.x; run < runs; run += gridDim.x * kThreads) {
    float v[16];
    int b0, bstep, e0, estep, rr;
    if constexpr (VT) {  // run = ((bt * r + rr) * 16 + e) * 4 + quarter: 16 consecutive b at one e
      const int q = run & 3, e = (run >> 2) & 15, btr = run >> 6;
      rr = btr % r;
      b0 = (btr / r) * kI2Pad + q * 16;
      bstep = 1;
      e0 = e;
      estep = 0;
    } else {  // run = (bt * r + rr) * 64 + swizzled row: 16 e of one b
      const int bsw = run & 63, btr = run >> 6;
      rr = btr % r;
      b0 = (btr / r) * kI2Pad + (bsw ^ ktile_swizzle(rr, BITS));
      bstep = 0;
      e0 = 0;
      estep = 1;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int b = b0 + k * bstep, e = e0 + k * estep;
      v[k] = b < i2 ? src[((int64_t)rr * i2 + b) * 16 + e] : 0.f;
    }
    uint32_t w[BITS];  // 16 codes x BITS bits, low code first
#pragma unroll
    for (int i = 0; i < BITS; ++i) w[i] = 0u;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int code = (degenerate || b0 + k * bstep >= i2) ? 0 : rtn_code_fast(v[k], kQmax, am, rinv);
      const uint32_t u = (uint32_t)((code + kX) & kMask);  // excess code (DQ_LAYOUT_KTILE / VTILE)
      w[(k * BITS) / 32] |= u << ((k * BITS) % 32);
    }
    uint8_t* out = dst + (int64_t)run * 2 * BITS;  // 16 codes = 2 BITS bytes, runs in slot order
    if constexpr (BITS == 8) *reinterpret_cast<uint4*>(out) = make_uint4(w[0], w[1], w[2], w[3]);
    else if constexpr (BITS == 4) *reinterpret_cast<uint2*>(out) = make_uint2(w[0], w[1]);
    else *reinterpret_cast<uint32_t*>(out) = w[0];
  }
}

// ---- opt-in per-channel asymmetric quantisation (dq_deco_quantize_asym_batched) ----------
// channel (rr, e) of core1 [r][i2][j2] over b: scale, zero point (fp64 arithmetic, f32 scale)
__global__ void asym_channels_kernel(const float* __restrict__ core1, int64_t core_elems, int r, int i2, int j2,
                                     int bits, float* __restrict__ channels) {
  const int64_t blk = blockIdx.y;
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;  // rr * j2 + e
  if (ch >= r * j2) return;
  const int rr = ch / j2, e = ch % j2;
  const float* src = core1 + blk * core_elems + (int64_t)rr * i2 * j2 + e;
  float mn = src[0], mx = src[0];
  for (int b = 1; b < i2; ++b) {
    const float v = src[(int64_t)b * j2];
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
  }
  const int qmu = (1 << bits) - 1;
  const double range = __dadd_rn((double)mx, -(double)mn);
  const float s = range > 0.0 ? (float)__ddiv_rn(range, (double)qmu) : (mx != 0.f ? fabsf(mx) : 1.f);
  double z = floor(__dadd_rn(__ddiv_rn(-(double)mn, (double)s), 0.5));
  z = z < 0.0 ? 0.0 : (z > qmu ? (double)qmu : z);
  float* out = channels + blk * (int64_t)2 * r * j2;
  out[ch] = s;
  out[r * j2 + ch] = (float)z;
}

__global__ void quantize_core_asym_kernel(const float* __restrict__ core1, int64_t core_elems, CoreGeom geom,
                                          int64_t out_bytes, const float* __restrict__ channels,
                                          uint8_t* __restrict__ payload, int64_t payload_stride) {
  const int64_t blk = blockIdx.y;
  const int bits = geom.bits, per = 8 / bits, qmu = (1 << bits) - 1;
  const float* src = core1 + blk * core_elems;
  const float* chs = channels + blk * (int64_t)2 * geom.r * geom.j2;
  const float* chz = chs + geom.r * geom.j2;
  uint8_t* dst = payload + blk * payload_stride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < out_bytes; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned v = 0;
    for (int k = 0; k < per; ++k) {
      const int64_t slot = i * per + k;
      if (slot >= geom_slots(geom)) break;
      int rr, b, e;
      unsigned code = 0;  // padding slots hold 0
      if (geom_coords(geom, slot, rr, b, e)) {
        const int ch = rr * geom.j2 + e;
        double u = __dadd_rn(floor(__dadd_rn(__ddiv_rn((double)src[((int64_t)rr * geom.i2 + b) * geom.j2 + e],
                                                      (double)chs[ch]), 0.5)), (double)chz[ch]);
        u = u < 0.0 ? 0.0 : (u > qmu ? (double)qmu : u);
        code = (unsigned)u;
      }
      v |= (code & ((1u << bits) - 1u)) << (k * bits);
    }
    dst[i] = (uint8_t)v;
  }
}

struct Workspace {
  double* G;
  double* U;
  double* lam;
  unsigned* amax;
  float* core1;  // optional scratch
};

size_t ws_bytes(int64_t nblk, const Dims& d, bool need_core1) {
  size_t b = 0;
  b += (size_t)nblk * kR * kR * 8 * 2;  // G, U
  b += (size_t)nblk * kR * 8;           // lam
  b += round_up(nblk * 4, 256);         // amax
  if (need_core1) b += (size_t)nblk * d.r * d.n * 4;
  return b;
}

Workspace carve(void* base, int64_t nblk, const Dims& d, bool need_core1) {
  Workspace w;
  char* p = (char*)base;
  w.G = (double*)p;
  p += (size_t)nblk * kR * kR * 8;
  w.U = (double*)p;
  p += (size_t)nblk * kR * kR * 8;
  w.lam = (double*)p;
  p += (size_t)nblk * kR * 8;
  w.amax = (unsigned*)p;
  p += round_up(nblk * 4, 256);
  w.core1 = need_core1 ? (float*)p : nullptr;
  return w;
}

int check_args(const void* blocks, int32_t dtype, int64_t nblk, int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1) return fail(DQ_ERR_SHAPE_MISMATCH, "dimensions must be >= 1");
  if (nblk < 0 || (nblk && !blocks)) return fail(DQ_ERR_INVALID_ARG, "bad block arguments");
  if (dtype != DQ_F32 && dtype != DQ_F16) return fail(DQ_ERR_INVALID_ARG, "unknown input dtype %d", dtype);
  if (rows * cols > (int64_t)1 << 31) return fail(DQ_ERR_UNSUPPORTED, "block too large");
  return DQ_OK;
}

// gram -> jacobi -> projection (core0 f32 + core1 f32 + amax)
int factor_core(const void* blocks, const Dims& d, int64_t nblk, float* core0, float* core1, const Workspace& w,
                int32_t* flags, cudaStream_t s) {
  DQ_CUDA_TRY(cudaMemsetAsync(w.amax, 0, (size_t)nblk * 4, s));
  // 128-wide rows in case A (every KV block: j = (8, 16)): the X-tile kernels (coalesced row
  // loads, fp64 tiles in shared memory); anything else: the generic element-wise gathers
  const bool fast = d.cols == 128 && d.j1 == 8 && d.j2 == 16 && d.caseA;
  // split the contraction so that the batch fills ~2 waves of 148 SMs
  const int64_t target = 296;
  constexpr int kProjSmem = (int)(sizeof(double) * kR * (kR + 2) + sizeof(double) * kR * (kTile + 2));
  constexpr int kProj128Smem = (int)(sizeof(double) * 2 * kR * kXpP);
  static bool attr_set = false;
  if (!attr_set) {
    DQ_CUDA_TRY(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(JacobiSmem)));
    DQ_CUDA_TRY(cudaFuncSetAttribute(eig_tql_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(EigSmem)));
    DQ_CUDA_TRY(cudaFuncSetAttribute(project_a_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kProjSmem));
    DQ_CUDA_TRY(cudaFuncSetAttribute(project128_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kProj128Smem));
    DQ_CUDA_TRY(cudaFuncSetAttribute(project128_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kProj128Smem));
    attr_set = true;
  }
  if (fast) {
    int64_t splits = ceil_div(target, nblk);
    int64_t bchunk = round_up(ceil_div(d.i2, splits), kNb);
    if (bchunk < 4 * kNb) bchunk = 4 * kNb;
    splits = ceil_div(d.i2, bchunk);
    if (splits > 1) DQ_CUDA_TRY(cudaMemsetAsync(w.G, 0, (size_t)nblk * kR * kR * 8, s));
    if (d.dtype == DQ_F16)
      gram128_kernel<true><<<dim3((unsigned)nblk, (unsigned)splits), kThreads, 0, s>>>(blocks, d, (int)bchunk, w.G,
                                                                                      flags);
    else
      gram128_kernel<false><<<dim3((unsigned)nblk, (unsigned)splits), kThreads, 0, s>>>(blocks, d, (int)bchunk, w.G,
                                                                                       flags);
  } else {
    DQ_CUDA_TRY(cudaMemsetAsync(w.G, 0, (size_t)nblk * kR * kR * 8, s));
    int64_t splits = ceil_div(target, nblk);
    int64_t chunk = round_up(ceil_div(d.kd, splits), kTile);
    if (chunk < 4 * kTile) chunk = 4 * kTile;
    splits = ceil_div(d.kd, chunk);
    gram_kernel<<<dim3((unsigned)nblk, (unsigned)splits), kThreads, 0, s>>>(blocks, d, (int)chunk, w.G, flags);
  }
  DQ_LAUNCH_CHECK();
#ifdef DQ_EIG_JACOBI  // the cyclic Jacobi eigensolver (measurement / cross-check builds)
  jacobi_kernel<<<(unsigned)nblk, kThreads, sizeof(JacobiSmem), s>>>(w.G, d, w.U, w.lam, flags);
#else
  eig_tql_kernel<<<(unsigned)nblk, kEigThreads, sizeof(EigSmem), s>>>(w.G, d, w.U, w.lam, flags);
#endif
  DQ_LAUNCH_CHECK();
  if (fast) {
    int64_t csplits = ceil_div(target, nblk);
    int64_t bchunk = round_up(ceil_div(d.i2, csplits), kNb);
    if (bchunk < 4 * kNb) bchunk = 4 * kNb;
    csplits = ceil_div(d.i2, bchunk);
    if (d.dtype == DQ_F16)
      project128_kernel<true><<<dim3((unsigned)nblk, (unsigned)csplits), kThreads, kProj128Smem, s>>>(
          blocks, d, (int)bchunk, w.U, w.lam, core0, core1, w.amax);
    else
      project128_kernel<false><<<dim3((unsigned)nblk, (unsigned)csplits), kThreads, kProj128Smem, s>>>(
          blocks, d, (int)bchunk, w.U, w.lam, core0, core1, w.amax);
  } else if (d.caseA) {
    int64_t csplits = ceil_div(target, nblk);
    int64_t cchunk = round_up(ceil_div(d.n, csplits), kTile);
    if (cchunk < 4 * kTile) cchunk = 4 * kTile;
    csplits = ceil_div(d.n, cchunk);
    project_a_kernel<<<dim3((unsigned)nblk, (unsigned)csplits), kThreads, kProjSmem, s>>>(blocks, d, (int)cchunk, w.U,
                                                                                   w.lam, core0, core1, w.amax);
  } else {
    project_b_kernel<<<(unsigned)nblk, kThreads, 0, s>>>(blocks, d, w.U, w.lam, core0, core1, w.amax);
  }
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

}  // namespace

}  // namespace dq

using namespace dq;

extern "C" int dq_decompose_workspace_size(int64_t nblk, int64_t rows, int64_t cols, size_t* bytes) {
  if (!bytes) return fail(DQ_ERR_INVALID_ARG, "null output");
  if (rows < 1 || cols < 1) return fail(DQ_ERR_SHAPE_MISMATCH, "dimensions must be >= 1");
  Dims d = make_dims(make_plan2(rows, cols), rows, cols, DQ_F32);
  *bytes = ws_bytes(nblk, d, true);
  return DQ_OK;
}

extern "C" int dq_decompose_plan_batched(const void* blocks, int32_t dtype, int64_t nblk, const dq_plan2* hp,
                                         float* core0, float* core1, int32_t* flags, void* ws, size_t wsb,
                                         void* stream) {
  if (!hp) return fail(DQ_ERR_INVALID_ARG, "null plan");
  const int64_t rows = hp->i1 * hp->i2, cols = hp->j1 * hp->j2;
  int st = check_args(blocks, dtype, nblk, rows, cols);
  if (st) return st;
  if (hp->i1 < 1 || hp->i2 < 1 || hp->j1 < 1 || hp->j2 < 1) return fail(DQ_ERR_SHAPE_MISMATCH, "factors must be >= 1");
  const int64_t left = hp->i1 * hp->j1, right = hp->i2 * hp->j2;
  if ((left < right ? left : right) > kR) return fail(DQ_ERR_UNSUPPORTED, "bond dimension %lld > %d",
                                                      (long long)(left < right ? left : right), kR);
  if (hp->r != (left < right ? left : right)) return fail(DQ_ERR_SHAPE_MISMATCH, "plan bond does not follow the bond law");
  if (nblk == 0) return DQ_OK;
  Dims d = make_dims(*hp, rows, cols, dtype);
  if (!core0 || !core1 || !ws || wsb < ws_bytes(nblk, d, false))
    return fail(DQ_ERR_INVALID_ARG, "dq_decompose_batched: missing output or workspace too small");
  Workspace w = carve(ws, nblk, d, false);
  return factor_core(blocks, d, nblk, core0, core1, w, flags, (cudaStream_t)stream);
}

extern "C" int dq_sym_eig_batched(const double* gram, int64_t nblk, int32_t n, double* vectors, double* values,
                                  int32_t* flags, void* stream) {
  if (n < 1 || n > kR) return fail(DQ_ERR_UNSUPPORTED, "dq_sym_eig_batched: n = %d outside 1..%d", n, kR);
  if (nblk < 0 || (nblk && (!gram || !vectors || !values))) return fail(DQ_ERR_INVALID_ARG, "dq_sym_eig_batched: bad arguments");
  if (nblk == 0) return DQ_OK;
  static bool attr = false;
  if (!attr) {
    DQ_CUDA_TRY(cudaFuncSetAttribute(eig_tql_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(EigSmem)));
    attr = true;
  }
  Dims d{};
  d.r = n;
  eig_tql_kernel<<<(unsigned)nblk, kEigThreads, sizeof(EigSmem), (cudaStream_t)stream>>>(gram, d, vectors, values, flags);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_deco_quantize_batched(const void* blocks, int32_t dtype, int64_t nblk, int64_t rows, int64_t cols,
                                        int32_t bits, int32_t layout, float* core0, uint8_t* payload,
                                        int64_t payload_stride, float* scale, int32_t* flags, void* ws, size_t wsb,
                                        void* stream) {
  if (!bits_ok(bits)) return fail(DQ_ERR_UNSUPPORTED_BITS, "bits must be one of (2, 4, 8), got %d", bits);
  int st = check_args(blocks, dtype, nblk, rows, cols);
  if (st) return st;
  if (nblk == 0) return DQ_OK;
  dq_plan2 p = make_plan2(rows, cols);
  Dims d = make_dims(p, rows, cols, dtype);
  int64_t out_bytes;
  st = dq_layout_bytes(&p, bits, layout, &out_bytes);
  if (st) return st;
  if (payload_stride < out_bytes) return fail(DQ_ERR_INVALID_ARG, "payload_stride smaller than one core");
  if (!core0 || !payload || !scale || !ws || wsb < ws_bytes(nblk, d, true))
    return fail(DQ_ERR_INVALID_ARG, "dq_deco_quantize_batched: missing output or workspace too small");
  Workspace w = carve(ws, nblk, d, true);
  cudaStream_t s = (cudaStream_t)stream;
  st = factor_core(blocks, d, nblk, core0, w.core1, w, flags, s);
  if (st) return st;
  CoreGeom g = make_geom(p, bits, layout);
  if (layout != DQ_LAYOUT_REF && g.j2 == 16) {
    const int64_t runs = (int64_t)g.r * (g.i2p / kI2Pad) * 64;
    int64_t gx = ceil_div(runs, kThreads);
    if (gx > 256) gx = 256;
    const dim3 grid((unsigned)gx, (unsigned)nblk);
    const int64_t ce = (int64_t)d.r * d.n;
#define DQ_QT16(B, V) \
  quantize_tile16_kernel<B, V><<<grid, kThreads, 0, s>>>(w.core1, ce, g, w.amax, payload, payload_stride, scale, flags)
    const bool vt = layout == DQ_LAYOUT_VTILE;
    if (bits == 2) { if (vt) DQ_QT16(2, true); else DQ_QT16(2, false); }
    else if (bits == 4) { if (vt) DQ_QT16(4, true); else DQ_QT16(4, false); }
    else { if (vt) DQ_QT16(8, true); else DQ_QT16(8, false); }
#undef DQ_QT16
    DQ_LAUNCH_CHECK();
    return DQ_OK;
  }
  int64_t gx = ceil_div(out_bytes, kThreads);
  if (gx > 64) gx = 64;
  quantize_core_kernel<<<dim3((unsigned)gx, (unsigned)nblk), kThreads, 0, s>>>(
      w.core1, (int64_t)d.r * d.n, g, out_bytes, w.amax, payload, payload_stride, scale, flags);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_deco_quantize_asym_batched(const void* blocks, int32_t dtype, int64_t nblk, int64_t rows,
                                             int64_t cols, int32_t bits, int32_t layout, float* core0,
                                             uint8_t* payload, int64_t payload_stride, float* channels,
                                             int32_t* flags, void* ws, size_t wsb, void* stream) {
  if (bits != 2 && bits != 4) return fail(DQ_ERR_UNSUPPORTED_BITS, "asymmetric mode: bits must be 2 or 4, got %d", bits);
  int st = check_args(blocks, dtype, nblk, rows, cols);
  if (st) return st;
  if (nblk == 0) return DQ_OK;
  dq_plan2 p = make_plan2(rows, cols);
  Dims d = make_dims(p, rows, cols, dtype);
  int64_t out_bytes;
  st = dq_layout_bytes(&p, bits, layout, &out_bytes);
  if (st) return st;
  if (payload_stride < out_bytes) return fail(DQ_ERR_INVALID_ARG, "payload_stride smaller than one core");
  if (!core0 || !payload || !channels || !ws || wsb < ws_bytes(nblk, d, true))
    return fail(DQ_ERR_INVALID_ARG, "dq_deco_quantize_asym_batched: missing output or workspace too small");
  Workspace w = carve(ws, nblk, d, true);
  cudaStream_t s = (cudaStream_t)stream;
  st = factor_core(blocks, d, nblk, core0, w.core1, w, flags, s);
  if (st) return st;
  const int nch = (int)(p.r * p.j2);
  asym_channels_kernel<<<dim3((unsigned)ceil_div(nch, 128), (unsigned)nblk), 128, 0, s>>>(
      w.core1, (int64_t)d.r * d.n, (int)p.r, (int)p.i2, (int)p.j2, bits, channels);
  DQ_LAUNCH_CHECK();
  CoreGeom g = make_geom(p, bits, layout);
  int64_t gx = ceil_div(out_bytes, kThreads);
  if (gx > 64) gx = 64;
  quantize_core_asym_kernel<<<dim3((unsigned)gx, (unsigned)nblk), kThreads, 0, s>>>(
      w.core1, (int64_t)d.r * d.n, g, out_bytes, channels, payload, payload_stride);
  DQ_LAUNCH_CHECK();
  return DQ_OK;
}

extern "C" int dq_decompose_batched(const void* blocks, int32_t dtype, int64_t nblk, int64_t rows, int64_t cols,
                                    float* core0, float* core1, int32_t* flags, void* ws, size_t wsb, void* stream) {
  if (rows < 1 || cols < 1) return fail(DQ_ERR_SHAPE_MISMATCH, "dimensions must be >= 1");
  const dq_plan2 p = make_plan2(rows, cols);
  return dq_decompose_plan_batched(blocks, dtype, nblk, &p, core0, core1, flags, ws, wsb, stream);
}

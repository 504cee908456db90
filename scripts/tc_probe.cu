// Probe of the tcgen05 int8 path the attention kernel would use (run under gpurun):
//   D[m][n] (s32, TMEM) = sum_k A[m][k] (u8) * B[n][k] (s8),  M = 128, N = 8 or 64, K = 64
// A is written to TMEM by the 128 threads with tcgen05.st (lane = m, 4 k-bytes per column),
// or staged in shared memory (K-major, no swizzle); B is in shared memory as K-major
// no-swizzle core matrices (8 rows x 16 bytes, K chunks LBO apart, 8-row groups SBO apart).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o gpurun_out/tc_probe scripts/tc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE
  return d;
}

// instruction descriptor: kind::i8, D s32, A u8 (0) / s8 (1), B s8, both K-major
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int a_signed, int b_signed) {
  return (2u << 4) | ((uint32_t)a_signed << 7) | ((uint32_t)b_signed << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

template <int N, bool A_TMEM>
__global__ void probe(const uint8_t* A, const int8_t* B, int* D, int* flag) {
  constexpr int M = 128, K = 64;
  __shared__ __align__(1024) uint8_t sa[M * K];  // K-major core matrices
  __shared__ __align__(1024) int8_t sb[N * K];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B: core matrix (8 rows x 16 B) for rows [8g, 8g+8) and K chunk j at (g * (K/16) + j) * 128
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const int g = n / 8, r = n % 8, j = k / 16, b = k % 16;
    sb[(g * (K / 16) + j) * 128 + r * 16 + b] = B[i];
  }
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const int g = m / 8, r = m % 8, j = k / 16, b = k % 16;
    sa[(g * (K / 16) + j) * 128 + r * 16 + b] = A[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // smem operands written by threads, read by the MMA
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  const uint32_t d_col = 0, a_col = 64;  // D: N columns, A: K/4 columns
  if (A_TMEM) {
    // thread (warp w, lane l) owns row m = 32 w + l: K/4 columns of 4 bytes each
    const int m = 32 * warp + lane;
    uint32_t v[K / 4];
    for (int c = 0; c < K / 4; ++c)
      v[c] = A[m * K + 4 * c] | (A[m * K + 4 * c + 1] << 8) | (A[m * K + 4 * c + 2] << 16) |
             ((uint32_t)A[m * K + 4 * c + 3] << 24);
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + a_col;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = idesc_i8(M, N, 0, 1);
    for (int s = 0; s < K / 32; ++s) {
      const uint64_t bdesc = smem_desc(sb + s * 256, 128, (K / 16) * 128);
      const uint32_t acc = s > 0;
      if (A_TMEM) {
        const uint32_t a_t = tmem + a_col + s * 8;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem + d_col),
            "r"(a_t), "l"(bdesc), "r"(idesc), "r"(acc));
      } else {
        const uint64_t adesc = smem_desc(sa + s * 256, 128, (K / 16) * 128);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + d_col),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait for the MMA
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const int m = 32 * warp + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + d_col + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 8; ++j) D[m * N + c0 + j] = (int)r[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
  if (tid == 0) *flag = 1;
}

template <int N, bool A_TMEM>
int run() {
  constexpr int M = 128, K = 64;
  std::vector<uint8_t> a(M * K);
  std::vector<int8_t> b(N * K);
  srand(N * 7 + A_TMEM);
  for (auto& x : a) x = rand() % 16;
  for (auto& x : b) x = (int8_t)(rand() % 256 - 128);
  uint8_t* dA;
  int8_t* dB;
  int *dD, *dF;
  cudaMalloc(&dA, M * K);
  cudaMalloc(&dB, N * K);
  cudaMalloc(&dD, M * N * 4);
  cudaMalloc(&dF, 4);
  cudaMemset(dD, 0xFF, M * N * 4);
  cudaMemcpy(dA, a.data(), M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, b.data(), N * K, cudaMemcpyHostToDevice);
  probe<N, A_TMEM><<<1, 128>>>(dA, dB, dD, dF);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<int> d(M * N);
  cudaMemcpy(d.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      int ref = 0;
      for (int k = 0; k < K; ++k) ref += (int)a[m * K + k] * (int)b[n * K + k];
      if (ref != d[m * N + n]) {
        if (bad < 5) printf("  mismatch m=%d n=%d got %d want %d\n", m, n, d[m * N + n], ref);
        ++bad;
      }
    }
  printf("N=%d A_%s: %s (%s), %d mismatches\n", N, A_TMEM ? "TMEM" : "SMEM", bad ? "FAIL" : "PASS",
         cudaGetErrorString(e), bad);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  cudaFree(dF);
  return bad != 0 || e != cudaSuccess;
}

int main() {
  int f = 0;
  f |= run<8, false>();
  f |= run<8, true>();
  f |= run<64, false>();
  f |= run<64, true>();
  return f;
}

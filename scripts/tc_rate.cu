// Throughput of back-to-back tcgen05.mma.kind::i8 (M = 128, K = 32) versus N, A from TMEM or smem.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tc_rate scripts/tc_rate.cu && /tmp/tc_rate
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int bsigned = 1) { return (2u << 4) | ((uint32_t)bsigned << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24); }

template <int N, bool TS, int ND, bool BUSY = false, bool VARY = false, bool SBUSY = false, int SBO = 256, int CE = 0,
          int BS = 1>
__global__ void rate(long long* out, int iters) {
  __shared__ __align__(1024) uint8_t sa[128 * 32 * 2];
  __shared__ __align__(1024) uint8_t sb[256 * 32 * 2 + 20480];  // + room for SBO = 2048 at N = 128
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, bar2;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 32 * 2; i += blockDim.x) sa[i] = i & 7;
  for (int i = tid; i < (int)sizeof(sb); i += blockDim.x) sb[i] = i & 3;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  __shared__ volatile int stop;
  if (tid == 0) stop = 0;
  __syncthreads();
  if (BUSY && !SBUSY && warp >= 1) {  // other warps keep writing TMEM (like the consumers widening codes)
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = 0x01010101u * (i + tid);
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + 64;
    while (!stop) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
                   "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
  }
  if (SBUSY && BUSY && warp >= 1) {  // LBUSY: other warps stream tcgen05.ld (like the Y fold), columns 64..255
    const uint32_t taddr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 64 + 16 * (warp >> 2);
    uint32_t accx = 0;
    while (!stop) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      accx += r[0] ^ r[15];
    }
    if (accx == 0x1234567u) out[1] = accx;
  } else if (SBUSY && warp >= 1) {  // other warps stream 16-byte loads from shared memory (like the consumers + TMA)
    uint4 acc = make_uint4(0, 0, 0, 0);
    const uint4* p = reinterpret_cast<const uint4*>(sb);
    int i = tid;
    while (!stop) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint4 v = p[(i + k * 32) & 1023];
        acc.x ^= v.x; acc.y += v.y;
      }
      i += 7;
    }
    if (acc.x == 0x1234567u) out[1] = acc.y;
  }
  if (tid == 0) {
    const uint64_t b = sdesc(sb, 128, SBO), a = sdesc(sa, 128, (32 / 16) * 128);
    const uint32_t id = idesc(128, N, BS);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem + 256 + (i % ND) * N), "r"(tmem + (VARY ? (i % 8) * 8 : 0)), "l"(VARY ? b + (uint64_t)((i % 8) * 16) : b), "r"(id), "r"((uint32_t)(i >= ND)));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + 256 + (i % ND) * N), "l"(VARY ? a + (uint64_t)((i % 8) * 16) : a), "l"(VARY ? b + (uint64_t)((i % 8) * 16) : b), "r"(id), "r"((uint32_t)(i >= ND)));
      if (CE && i % CE == CE - 1)  // a commit every CE UMMAs (nobody waits on it)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
    out[0] = clock64() - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, bool TS, int ND = 1, bool BUSY = false, bool VARY = false, bool SBUSY = false, int SBO = 256, int CE = 0,
          int BS = 1>
void run(int grid = 1) {
  long long* d;
  cudaMalloc(&d, 8);
  long long c1 = 0, c2 = 0;
  rate<N, TS, ND, BUSY, VARY, SBUSY, SBO, CE, BS><<<grid, SBUSY ? 512 : 128>>>(d, 64);
  cudaDeviceSynchronize();
  rate<N, TS, ND, BUSY, VARY, SBUSY, SBO, CE, BS><<<grid, SBUSY ? 512 : 128>>>(d, 64);
  cudaMemcpy(&c1, d, 8, cudaMemcpyDeviceToHost);
  rate<N, TS, ND, BUSY, VARY, SBUSY, SBO, CE, BS><<<grid, SBUSY ? 512 : 128>>>(d, 1024);
  cudaMemcpy(&c2, d, 8, cudaMemcpyDeviceToHost);
  printf("BS=%d CE=%d grid=%d SBO=%d SBUSY=%d VARY=%d BUSY=%d ND=%d N=%3d A=%s: %.1f cycles per UMMA (M128 K32), first 64 took %lld cycles, %s\n", BS, CE, grid, SBO, (int)SBUSY, (int)VARY, (int)BUSY, ND, N,
         TS ? "TMEM" : "SMEM", (double)(c2 - c1) / (1024 - 64), c1, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<16, true, 4>();
  run<16, true, 4, false, true>();
  run<16, true, 1, false, true>();
  run<16, false, 4, false, true>();
  run<16, true, 4, true, true>();
  run<64, true, 2, false, true>();
  run<128, true, 1, false, true>();
  run<128, false, 1, false, true>();
  run<256, true, 1, false, true>();
  run<256, false, 1, false, true>();
  run<128, true, 1, false, true, true>();   // + 15 warps of shared-memory loads
  run<128, true, 1, true, true, false>();   // + 3 warps of TMEM stores
  run<128, true, 1, false, true, false, 1024>();  // the path-2 W slice layout (N groups 1 KB apart)
  run<128, true, 2, false, true, false, 1024>();
  run<128, true, 1, false, true, false, 1024>(148);  // every SM at once
  run<128, true, 1, false, true, true, 1024>(148);
  run<128, true, 1, false, true, false, 1024, 8>();  // + a commit every 8 UMMAs
  run<128, true, 1, false, true, false, 1024, 4>();
  run<128, true, 2, false, true, false, 1024, 2>();
  run<128, true, 1, false, true, false, 2048>();            // the path-2 P layout (groups 2 KB apart)
  run<128, true, 1, false, true, false, 2048, 8, 0>();      // + u8 x u8 + a commit every 8
  run<128, true, 1, true, true, true, 2048, 8, 0>();        // + 15 warps streaming tcgen05.ld
  return 0;
}

// Whole-GPU throughput of the legacy int8 tensor path (mma.sync.m16n8k32.s32.s8.s8.s32) on sm_100a,
// the instruction the path-0 split kernel contracts with.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mma_rate scripts/mma_rate.cu && /tmp/mma_rate
#include <cstdint>
#include <cstdio>

template <int NACC>
__global__ void rate(int* out, int iters, uint32_t seed) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  int acc[NACC][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NACC; ++k)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(acc[k][0]), "+r"(acc[k][1]), "+r"(acc[k][2]), "+r"(acc[k][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int k = 0; k < NACC; ++k) s += acc[k][0] + acc[k][1] + acc[k][2] + acc[k][3];
  if (s == 0x12345) out[0] = s;
}

template <int NACC>
void run(int sms, int warps, int ctas) {
  int* d;
  cudaMalloc(&d, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  rate<NACC><<<sms * ctas, warps * 32>>>(d, 64, 1);
  cudaEventRecord(e0);
  rate<NACC><<<sms * ctas, warps * 32>>>(d, iters, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * 16 * 8 * 32 * (double)NACC * iters * warps * sms * ctas;
  printf("mma.sync m16n8k32 s8: %d CTAs x %2d warps, %d acc chains: %.1f TOPS (%.0f MAC/clk/SM at 1.9 GHz) %s\n", sms * ctas, warps, NACC,
         ops / ms / 1e9, ops / 2 / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4>(sms, 8, 1);
  run<4>(sms, 16, 1);
  run<8>(sms, 16, 1);
  run<8>(sms, 16, 2);
  run<8>(sms, 32, 1);
  return 0;
}

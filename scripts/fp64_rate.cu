// FP64 peak on this B200: DFMA (CUDA cores) and DMMA (mma.sync.m8n8k4.f64, tensor cores).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/fp64_rate.cu -o fp64_rate && ./fp64_rate
// The write path (K3: Gram, Jacobi, projection) is fp64-bound; this is its roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, double a0, double b0) {
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    const int blocks = sms * (2048 / threads);
    dfma_kernel<<<blocks, threads>>>(out, 0.999, 1e-3);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * kIters * (double)blocks * threads;
    printf("DFMA  threads/CTA %4d: %.1f TFLOP/s\n", threads, flops / ms / 1e9);
    dmma_kernel<<<blocks, threads>>>(out, 0.999, 1e-3);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double mflops = 2.0 * 8 * 8 * 4 * 4 * kIters * (double)blocks * (threads / 32);
    printf("DMMA  threads/CTA %4d: %.1f TFLOP/s\n", threads, mflops / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

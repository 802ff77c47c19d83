// MUFU.EX2 vs FFMA issue throughput per SM (microbenchmark for the K3 softmax balance).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ex2_kernel(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void ffma_kernel(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f33800000;" : "+f"(a[i]));
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000;
  for (int threads : {128, 256, 512, 1024}) {
    for (int k = 0; k < 2; ++k) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (k == 0) ex2_kernel<<<sms, threads>>>(d, iters); else ffma_kernel<<<sms, threads>>>(d, iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = (double)sms * threads * iters * 8;
        if (rep) printf("%s threads/SM %4d: %.2f Gop/s per SM = %.2f op/clk/SM at %.0f MHz (nominal)\n", k ? "FFMA" : "EX2 ",
                        threads, ops / sms / (ms * 1e-3) / 1e9, ops / sms / (ms * 1e-3) / (clk * 1e3), clk / 1e3);
      }
    }
  }
  return 0;
}

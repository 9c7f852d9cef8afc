// MUFU sin/cos throughput on this GPU: independent sin.approx chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters, float seed) {
  float a0 = seed + threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < iters; ++i) {
    asm volatile("sin.approx.f32 %0, %0;" : "+f"(a0)); asm volatile("cos.approx.f32 %0, %0;" : "+f"(a1));
    asm volatile("sin.approx.f32 %0, %0;" : "+f"(a2)); asm volatile("cos.approx.f32 %0, %0;" : "+f"(a3));
    asm volatile("sin.approx.f32 %0, %0;" : "+f"(a4)); asm volatile("cos.approx.f32 %0, %0;" : "+f"(a5));
    asm volatile("sin.approx.f32 %0, %0;" : "+f"(a6)); asm volatile("cos.approx.f32 %0, %0;" : "+f"(a7));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void kex2(float* out, int iters, float seed) {   // ex2.approx for comparison
  float a0 = seed + threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a4)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a5));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a6)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a7));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 32 * 1024);
  const int iters = 4096, threads = 1024, blocks = sms * 2;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int which = 0; which < 2; ++which) {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0);
      if (which == 0) k<<<blocks, threads>>>(out, iters, 0.5f); else kex2<<<blocks, threads>>>(out, iters, 0.5f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double ops = double(blocks) * threads * iters * 8;
      if (r) printf("%s: %.3f ms, %.1f Gop/s, %.2f ops/clk/SM (clock %d MHz, %d SMs)\n", which ? "ex2" : "sin/cos", ms,
                    ops / ms / 1e6, ops / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000, sms);
    }
  }
  return 0;
}

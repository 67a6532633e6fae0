#include <cstdio>
__global__ void k(float* o, int n) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) o[0] = s;
}
int main() {
  float* o; cudaMalloc(&o, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int n = 4096;
  k<<<148 * 4, 512>>>(o, 16);
  cudaEventRecord(a);
  k<<<148 * 4, 512>>>(o, n);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ops = 148.0 * 4 * 512 * n * 8;
  printf("{\"ex2_per_s\": %.4g, \"ms\": %.3f}\n", ops / (ms * 1e-3), ms);
  return 0;
}

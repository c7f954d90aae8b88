#include <cstdio>
__global__ void ex2k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y - 1.0f; }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 123.f) out[0] = s;
}
__global__ void fmak(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 0.999f, 0.001f);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 123.f) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* o; cudaMalloc(&o, 4);
  for (int k = 0; k < 2; ++k) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4000, threads = 512, blocks = sms * 2;
    if (k == 0) ex2k<<<blocks, threads>>>(o, 10); else fmak<<<blocks, threads>>>(o, 10);
    cudaEventRecord(a);
    if (k == 0) ex2k<<<blocks, threads>>>(o, iters); else fmak<<<blocks, threads>>>(o, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * threads * iters * 8;
    printf("%s: %.2f Tops/s = %.1f ops/clk/SM at %d MHz\n", k == 0 ? "MUFU.EX2" : "FFMA", ops / (ms * 1e-3) / 1e12,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}

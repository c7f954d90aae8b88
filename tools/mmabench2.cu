// tcgen05 issue rate: lane-0-only issuer vs warp-uniform loop + elect.sync issuer.
#include <cstdio>
#include "../paper_2510_12747_b200/csrc/fvsr_common.cuh"
using namespace fvsr;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

template <int N, int WARPWIDE>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t done;
  if (threadIdx.x < 32) tmem_alloc(&tslot, 256);
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_barrier_init(); }
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t a = smem_u32(sm), b = smem_u32(sm + 65536);
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
  if (WARPWIDE ? threadIdx.x < 32 : threadIdx.x == 0) {
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t da = umma_desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
        const uint64_t db = umma_desc_sw128(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
        if (!WARPWIDE || elect_one()) tc_mma_f16(tmem + 128, da, db, idesc, (i | kk) > 0);
        if (WARPWIDE) __syncwarp();
      }
    }
    if (!WARPWIDE || elect_one()) tc_commit(&done);
    __syncwarp(WARPWIDE ? 0xffffffffu : 1u);
    mbar_wait(&done, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

template <int N, int W>
void run(const char* name) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out;
  cudaMalloc(&out, 4096 * 8);
  auto f = k<N, W>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
  const int iters = 16000;
  f<<<sms, 128, 98304 + 1024>>>(96, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  f<<<sms, 128, 98304 + 1024>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("%-36s %.1f cyc/mma  %.0f TFLOP/s (%s)\n", name, (double)h / iters,
         2.0 * 128 * N * 16 * (double)iters * sms / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<64, 0>("N64 lane0 issuer, unrolled");
  run<64, 1>("N64 warp-wide + elect.sync");
  run<128, 0>("N128 lane0 issuer, unrolled");
  run<128, 1>("N128 warp-wide + elect.sync");
  run<256, 1>("N256 warp-wide + elect.sync");
  return 0;
}

// Does TMA (bulk copy) smem fill or STS traffic slow tcgen05 MMAs at N=64 (smem-operand bound)?
// warp 0: MMA loop (M=128, N=64, K=16, both operands SW128 K-major from smem);
// warp 1 (LOAD): bulk global->smem copies of 16 KB into a separate region, back to back;
// warps 2-5 (STS): st.shared.v4 streams into another region.
#include <cstdio>
#include "../paper_2510_12747_b200/csrc/fvsr_common.cuh"
using namespace fvsr;

template <int LOAD, int STS>
__global__ void __launch_bounds__(192, 1) k(int iters, const uint8_t* gsrc, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t done, ld;
  __shared__ volatile int stop;
  if (threadIdx.x < 32) tmem_alloc(&tslot, 256);
  if (threadIdx.x == 0) { mbar_init(&done, 1); mbar_init(&ld, 1); stop = 0; fence_barrier_init(); }
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t a = smem_u32(sm), b = smem_u32(sm + 65536);
  constexpr uint32_t idesc = umma_idesc_bf16(128, 64, 0, 0);
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t da = umma_desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
        const uint64_t db = umma_desc_sw128(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
        if (elect_one()) tc_mma_f16(tmem + 128, da, db, idesc, (i | kk) > 0);
        __syncwarp();
      }
    }
    if (elect_one()) tc_commit(&done);
    __syncwarp();
    mbar_wait(&done, 0);
    if (threadIdx.x == 0) { out[blockIdx.x] = clock64() - t0; stop = 1; }
  } else if (warp == 1 && LOAD) {
    uint8_t* dst = sm + 98304;  // 32 KB region
    int ph = 0;
    for (int it = 0; !stop; ++it) {
      if (threadIdx.x == 32) {
        mbar_arrive_expect_tx(&ld, 32768);
        bulk_g2s(dst, gsrc + ((it * 32768) & ((1 << 22) - 1)), 16384, &ld);
        bulk_g2s(dst + 16384, gsrc + ((it * 32768 + 16384) & ((1 << 22) - 1)), 16384, &ld);
      }
      __syncwarp();
      mbar_wait(&ld, ph);
      ph ^= 1;
    }
  } else if (warp >= 2 && STS) {
    uint4* dst = reinterpret_cast<uint4*>(sm + 98304 + 32768) + (threadIdx.x - 64);
    const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    while (!stop) {
#pragma unroll
      for (int r = 0; r < 16; ++r) dst[(r * 128) & 2047] = v;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

template <int L, int S>
void run(const char* name, const uint8_t* g) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out;
  cudaMalloc(&out, 4096 * 8);
  auto f = k<L, S>;
  const int smem = 98304 + 32768 + 32768 + 1024;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 16000;
  f<<<sms, 192, smem>>>(96, g, out);
  cudaDeviceSynchronize();
  f<<<sms, 192, smem>>>(iters, g, out);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %.1f cyc/mma (%s)\n", name, (double)h / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint8_t* g;
  cudaMalloc(&g, 1 << 22);
  cudaMemset(g, 0, 1 << 22);
  run<0, 0>("MMA N64 alone", g);
  run<1, 0>("MMA N64 + bulk loads (L2-resident)", g);
  run<0, 1>("MMA N64 + STS.128 streams (4 warps)", g);
  run<1, 1>("MMA N64 + bulk loads + STS", g);
  return 0;
}

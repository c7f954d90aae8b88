// tcgen05 kind::f16 rate at M=128, N=64 by operand majorness (K-major vs MN-major SW128),
// and two interleaved accumulators (the attention kernel's QK / PV mix).
#include <cstdio>
#include "../paper_2510_12747_b200/csrc/fvsr_common.cuh"
using namespace fvsr;

template <int N, int AM, int BM, int MIX>
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
  constexpr uint32_t idesc_kk = umma_idesc_bf16(128, N, 0, 0);
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, AM, BM);
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        // A: 128 x 128 (K-major: 2 sub-tiles of 64 K; MN-major: rows = K, 2 sub-tiles of 64 M)
        const uint64_t da = AM ? umma_desc_sw128(a + kk * 2048, 16384u, 1024u)
                               : umma_desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16u, 1024u);
        const uint64_t db = BM ? umma_desc_sw128(b + kk * 2048, 16384u, 1024u)
                               : umma_desc_sw128(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16u, 1024u);
        if (elect_one()) {
          if (MIX) {
            const uint64_t ka = umma_desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16u, 1024u);
            const uint64_t kb = umma_desc_sw128(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16u, 1024u);
            tc_mma_f16(tmem, ka, kb, idesc_kk, (i | kk) > 0);
          }
          tc_mma_f16(tmem + 128, da, db, idesc, (i | kk) > 0);
        }
        __syncwarp();
      }
    }
    if (elect_one()) tc_commit(&done);
    __syncwarp();
    mbar_wait(&done, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

template <int N, int AM, int BM, int MIX>
void run(const char* name) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out;
  cudaMalloc(&out, 4096 * 8);
  auto f = k<N, AM, BM, MIX>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
  const int iters = 16000;
  f<<<sms, 128, 98304 + 1024>>>(96, out);
  cudaDeviceSynchronize();
  f<<<sms, 128, 98304 + 1024>>>(iters, out);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("%-44s %.1f cyc/mma (%s)\n", name, (double)h / (iters * (MIX ? 2 : 1)), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<64, 0, 0, 0>("N64 A K-major  B K-major");
  run<64, 1, 1, 0>("N64 A MN-major B MN-major (PV)");
  run<64, 1, 0, 0>("N64 A MN-major B K-major");
  run<64, 0, 1, 0>("N64 A K-major  B MN-major");
  run<64, 1, 1, 1>("N64 QK(KK) + PV(MN,MN) interleaved");
  run<64, 0, 0, 1>("N64 KK + KK interleaved (2 accumulators)");
  run<128, 0, 0, 0>("N128 A K-major  B K-major");
  run<128, 1, 1, 0>("N128 A MN-major B MN-major");
  return 0;
}

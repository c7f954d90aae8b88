// tcgen05 issue-rate variants: operand majors, commit cadence, concurrent TMEM loads.
#include <cstdio>
#include "../paper_2510_12747_b200/csrc/fvsr_common.cuh"
using namespace fvsr;

template <int N, int AMN, int BMN, int COMMIT, int LDWARPS>
__global__ void __launch_bounds__(160, 1) k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t done, grp;
  if (threadIdx.x < 32) tmem_alloc(&tslot, 256);
  if (threadIdx.x == 0) { mbar_init(&done, 1); mbar_init(&grp, 1); fence_barrier_init(); }
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 65536);
    const uint32_t idesc = umma_idesc_bf16(128, N, AMN, BMN);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 7;
      uint64_t da, db;
      if (AMN) da = umma_desc_sw128(a + kk * 2048, 16384, 1024);
      else da = umma_desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
      if (BMN) db = umma_desc_sw128(b + kk * 2048, 16384, 1024);
      else db = umma_desc_sw128(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
      tc_mma_f16(tmem + 128, da, db, idesc, i > 0);
      if (COMMIT && kk == 7) tc_commit(&grp);
    }
    tc_commit(&done);
    mbar_wait(&done, 0);
    out[blockIdx.x] = clock64() - t0;
  } else if (LDWARPS && warp >= 1 && warp <= 4) {
    // concurrent TMEM reader on columns [0,64)
    uint32_t r[32];
    unsigned acc = 0;
    for (int i = 0; i < iters / 8; ++i) {
      tmem_ld32(tmem + (((warp - 1) * 32) << 16), r);
      tc_wait_ld();
      acc += r[i & 31];
    }
    if (acc == 12345) out[0] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

template <int N, int AMN, int BMN, int COMMIT, int LDW>
void run(const char* name) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out;
  cudaMalloc(&out, 4096 * 8);
  auto f = k<N, AMN, BMN, COMMIT, LDW>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
  const int iters = 16000;
  f<<<sms, 160, 98304 + 1024>>>(100, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  f<<<sms, 160, 98304 + 1024>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %.1f cyc/mma  %.0f TFLOP/s  (%s)\n", name, (double)h / iters,
         2.0 * 128 * N * 16 * (double)iters * sms / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<64, 0, 0, 0, 0>("N64 Kmaj/Kmaj");
  run<64, 0, 0, 1, 0>("N64 Kmaj/Kmaj commit/8");
  run<64, 1, 1, 0, 0>("N64 MNmaj/MNmaj (PV)");
  run<64, 1, 1, 1, 0>("N64 MNmaj/MNmaj commit/8");
  run<64, 1, 0, 0, 0>("N64 MNmaj/Kmaj");
  run<64, 0, 1, 0, 0>("N64 Kmaj/MNmaj");
  run<64, 0, 0, 1, 1>("N64 Kmaj/Kmaj commit + tmem ld");
  run<128, 0, 0, 0, 0>("N128 Kmaj/Kmaj");
  run<128, 1, 1, 0, 0>("N128 MNmaj/MNmaj");
  return 0;
}

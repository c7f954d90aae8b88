// Microbenchmarks that set the sparse-attention design ceilings on B200 (sm_100a):
//   l2bw  : cp.async.bulk global->shared bandwidth from an L2-resident buffer, with
//           `share` CTAs reading the same tile sequence concurrently (dedup effect)
//   mma   : tcgen05.mma kind::f16 M=128 x N x K=16 (SS) back-to-back issue rate
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2510_12747_b200/csrc/fvsr_common.cuh"
using namespace fvsr;

__global__ void __launch_bounds__(128, 1) l2bw_kernel(const uint8_t* buf, long long ntiles, int tile_bytes, int iters,
                                                      int share, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(full + i, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long group = blockIdx.x / share;
  unsigned long long seed = 0x9E3779B97F4A7C15ull * (group + 1);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int st = it & 3;
    if (it >= 4) mbar_wait(full + st, ((it >> 2) - 1) & 1);
    seed = seed * 6364136223846793005ull + 1442695040888963407ull;
    const long long tile = (long long)((seed >> 17) % (unsigned long long)ntiles);
    mbar_arrive_expect_tx(full + st, tile_bytes);
    for (int off = 0; off < tile_bytes; off += 8192)
      bulk_g2s(sm + st * tile_bytes + off, buf + tile * tile_bytes + off, 8192, full + st);
  }
  for (int it = iters; it < iters + 4; ++it) mbar_wait(full + (it & 3), ((it >> 2) - 1) & 1);
  cycles[blockIdx.x] = clock64() - t0;
}

template <int N>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t done;
  if (threadIdx.x < 32) tmem_alloc(&tslot, 256);
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_barrier_init(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t da = umma_desc_sw128(a + (i & 3) * 32, 16, 1024);
      const uint64_t db = umma_desc_sw128(b + (i & 3) * 32, 16, 1024);
      tc_mma_f16(tmem, da, db, idesc, i > 0);
    }
    tc_commit(&done);
    mbar_wait(&done, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

int mc_main();
int main(int argc, char** argv) {
  if (argc > 1) return mc_main();
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 4096 * sizeof(unsigned long long));
  std::vector<unsigned long long> h(4096);
  // ---- L2 bulk-copy bandwidth ----
  const long long buf_bytes = 96ll << 20;  // L2-resident
  uint8_t* buf;
  cudaMalloc(&buf, buf_bytes);
  cudaMemset(buf, 1, buf_bytes);
  const int tile = 32768;
  cudaFuncSetAttribute(l2bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * tile);
  for (int share : {1, 2, 4, 8, 16}) {
    for (int ctas_per_sm : {1}) {
      const int grid = sms * ctas_per_sm;
      const int iters = 2000;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      l2bw_kernel<<<grid, 128, 4 * tile>>>(buf, buf_bytes / tile, tile, 50, share, cyc);
      cudaEventRecord(a);
      l2bw_kernel<<<grid, 128, 4 * tile>>>(buf, buf_bytes / tile, tile, iters, share, cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)grid * iters * tile;
      printf("l2bw share=%2d grid=%d: %.2f TB/s (%.1f us, %.1f B/clk/SM at %d MHz)\n", share, grid,
             bytes / (ms * 1e-3) / 1e12, ms * 1e3, bytes / grid / (ms * 1e-3 * clk_khz * 1e3), clk_khz / 1000);
    }
  }
  // ---- tcgen05 issue rate ----
  cudaFuncSetAttribute(mma_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(mma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(mma_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 20000;
  for (int n : {64, 128, 256}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto k = n == 64 ? mma_kernel<64> : (n == 128 ? mma_kernel<128> : mma_kernel<256>);
    k<<<sms, 128, 65536>>>(100, cyc);
    cudaEventRecord(a);
    k<<<sms, 128, 65536>>>(iters, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(h.data(), cyc, sms * 8, cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * n * 16 * (double)iters * sms;
    printf("mma M=128 N=%3d K=16: %.0f TFLOP/s, %.1f cyc/mma (sm0 clock64)\n", n, flops / (ms * 1e-3) / 1e12,
           (double)h[0] / iters);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

// ---- multicast: leader CTA of each cluster multicasts tiles to every CTA of the cluster ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) mc_kernel(const uint8_t* buf, long long ntiles, int tile_bytes, int iters,
                                                    unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[4], empty[4];
  const uint32_t rank = cluster_ctarank(), n = cluster_nctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, n); }
    fence_barrier_init();
  }
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x == 0) {
    const long long cl = blockIdx.x / n;
    unsigned long long seed = 0x9E3779B97F4A7C15ull * (cl + 1);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int st = it & 3;
      if (it >= 4) mbar_wait(full + st, ((it >> 2) - 1) & 1);  // my previous use of st consumed
      if (it >= 4) mbar_arrive_remote(empty + st, 0);            // tell the leader slot st is free
      mbar_arrive_expect_tx(full + st, tile_bytes);
      seed = seed * 6364136223846793005ull + 1442695040888963407ull;
      const long long tile = (long long)((seed >> 17) % (unsigned long long)ntiles);
      if (rank == 0) {
        if (it >= 4) mbar_wait(empty + st, ((it >> 2) - 1) & 1);
        for (int off = 0; off < tile_bytes; off += 8192)
          bulk_g2s_mc(sm + st * tile_bytes + off, buf + tile * tile_bytes + off, 8192, full + st, (uint16_t)((1u << n) - 1));
      }
    }
    for (int it = iters; it < iters + 4; ++it) mbar_wait(full + (it & 3), ((it >> 2) - 1) & 1);
    cycles[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  cluster_sync_all();
}

int mc_main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* buf;
  const long long buf_bytes = 96ll << 20;
  cudaMalloc(&buf, buf_bytes);
  cudaMemset(buf, 1, buf_bytes);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 4096 * 8);
  const int tile = 32768, iters = 2000;
  cudaFuncSetAttribute(mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * tile);
  cudaFuncSetAttribute(mc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8}) {
    int grid = (sms / cs) * cs;
    if (cs == 4) grid = 132;
    if (cs == 8) grid = 128;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 4 * tile;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, mc_kernel, (const uint8_t*)buf, buf_bytes / tile, tile, 50, cyc);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernelEx(&cfg, mc_kernel, (const uint8_t*)buf, buf_bytes / tile, tile, iters, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double delivered = (double)grid * iters * tile, l2 = delivered / cs;
    printf("multicast cluster=%d grid=%d: delivered %.2f TB/s, L2 reads %.2f TB/s (%s)\n", cs, grid,
           delivered / (ms * 1e-3) / 1e12, l2 / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
  }
  return 0;
}

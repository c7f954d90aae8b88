// L2 -> shared-memory gather bandwidth on B200: the roofline of the attention kernel's
// K/V tile gather (cp.async.bulk of 16 KB halves of a 32 KB frame-tile pair, the same copy
// shape as kernel_attn.cu's load_kv).
//
// One CTA per SM (or `grid`), one issuing thread, `stages` x 32 KB ring in shared memory; each
// stage is refilled as soon as its copy lands (no consumer), from pseudo-random 16 KB-aligned
// offsets of a `buf_mb` buffer (64 MB: L2-resident after the warm-up pass; 4096 MB: HBM).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/l2bench tools/l2bench.cu
//   tools/l2bench            -> one line per (buffer, grid, stages): GB/s and bytes/SM-cycle
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2510_12747_b200/csrc/fvsr_common.cuh"
using namespace fvsr;

__global__ void __launch_bounds__(32, 1) gather(const uint8_t* src, unsigned long long nchunks, int stages, int iters,
                                                unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncwarp();
  unsigned long long x = 0x9E3779B97F4A7C15ull * (blockIdx.x + 1);
  auto next = [&]() {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return (x % nchunks) * 32768ull;
  };
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      const unsigned long long o = next();
      mbar_arrive_expect_tx(&bar[s], 32768);
      bulk_g2s(sm + s * 32768, src + o, 16384, &bar[s]);
      bulk_g2s(sm + s * 32768 + 16384, src + o + 16384, 16384, &bar[s]);
    }
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      mbar_wait(&bar[s], (uint32_t)(i / stages) & 1);
      const unsigned long long o = next();
      mbar_arrive_expect_tx(&bar[s], 32768);
      bulk_g2s(sm + s * 32768, src + o, 16384, &bar[s]);
      bulk_g2s(sm + s * 32768 + 16384, src + o + 16384, 16384, &bar[s]);
    }
    for (int i = iters; i < iters + stages; ++i) mbar_wait(&bar[i % stages], (uint32_t)(i / stages) & 1);
    cycles[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = 4096ull << 20;
  uint8_t* buf = nullptr;
  if (cudaMalloc(&buf, big) != cudaSuccess) return 1;
  cudaMemset(buf, 1, big);
  unsigned long long* cyc = nullptr;
  cudaMalloc(&cyc, 1024 * sizeof(unsigned long long));
  cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  std::printf("{\"sms\": %d, \"rows\": [\n", sms);
  bool first = true;
  for (size_t mb : {64ul, 4096ul}) {
    const unsigned long long nchunks = (mb << 20) / 32768;
    for (int grid : {sms, 132, 74}) {
      for (int stages : {1, 2, 3, 4, 6}) {
        const int iters = mb == 64 ? 4000 : 2000;
        gather<<<grid, 32, stages * 32768>>>(buf, nchunks, stages, 200, cyc);  // warm-up
        cudaEventRecord(a);
        gather<<<grid, 32, stages * 32768>>>(buf, nchunks, stages, iters, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        std::vector<unsigned long long> h(grid);
        cudaMemcpy(h.data(), cyc, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (auto c : h) mx = c > mx ? c : mx;
        const double bytes = (double)grid * (iters + stages) * 32768.0;
        std::printf("%s  {\"buffer_mb\": %zu, \"grid\": %d, \"stages_32KB\": %d, \"GBps\": %.1f, "
                    "\"bytes_per_sm_cycle\": %.1f, \"bytes_per_chip_cycle\": %.1f}",
                    first ? "" : ",\n", mb, grid, stages, bytes / (ms * 1e-3) / 1e9, (iters + stages) * 32768.0 / mx,
                    bytes / (ms * 1e-3) / (clk * 1e3));
        first = false;
      }
    }
  }
  std::printf("\n], \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

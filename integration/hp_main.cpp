// hp_main.cpp — check of the C++ head-parallel layer-step (vsr_b200_parallel.hpp) on one GPU.
//
//   hp_main            world 1 with a real NCCL communicator (ncclCommInitAll on device 0)
//                      and simulated worlds 2, 4, 8 (one object per rank, null comm, shards
//                      concatenated in rank order = what ncclAllGather produces, fvsr_untile)
// Every output is compared bitwise with the unsharded fvsr_ring_step over the same frames.
// Prints one line per world, "OK" / "MISMATCH"; exit status = number of mismatches.
#include <cstdio>
#include <random>
#include <vector>

#include "vsr_b200_parallel.hpp"

using namespace vsr::b200;

#define CK(x)                                                           \
  do {                                                                  \
    if (!(x)) {                                                         \
      std::fprintf(stderr, "%s:%d: %s (%s)\n", __FILE__, __LINE__, #x, fvsr_last_error()); \
      return 100;                                                       \
    }                                                                   \
  } while (0)

int main() {
  const int heads = 12, d = 128, rows = 48, cols = 88, window = 4, frames = 6;
  const long long topk = 27;
  const long long N = (long long)rows * cols, per_frame = heads * N * d;
  std::mt19937 rng(2510);
  std::normal_distribution<float> nd;
  std::vector<uint16_t> h(3 * frames * per_frame);
  for (auto& x : h) {
    const float f = nd(rng);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    x = static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
  }
  uint16_t* dev = nullptr;
  CK(cudaMalloc(&dev, h.size() * 2) == cudaSuccess);
  CK(cudaMemcpy(dev, h.data(), h.size() * 2, cudaMemcpyHostToDevice) == cudaSuccess);
  auto q = [&](int t) { return dev + (0 * frames + t) * per_frame; };
  auto k = [&](int t) { return dev + (1 * frames + t) * per_frame; };
  auto v = [&](int t) { return dev + (2 * frames + t) * per_frame; };
  fvsr_mask mask{};
  mask.kind = FVSR_MASK_LOCALITY;
  mask.mode = FVSR_LOCALITY_TRUNCATED;
  mask.extent_h = 48;
  mask.extent_w = 72;
  const float scale = 1.0f / std::sqrt(static_cast<float>(d));
  cudaStream_t s;
  CK(cudaStreamCreate(&s) == cudaSuccess);

  // unsharded reference outputs, one per step
  std::vector<std::vector<uint16_t>> ref(frames, std::vector<uint16_t>(per_frame));
  {
    fvsr_ctx* ctx;
    fvsr_ring* ring;
    CK(fvsr_ctx_create(&ctx) == FVSR_OK);
    CK(fvsr_ring_create(ctx, 1, heads, d, rows, cols, window, &ring) == FVSR_OK);
    uint16_t* out;
    CK(cudaMalloc(&out, per_frame * 2) == cudaSuccess);
    for (int t = 0; t < frames; ++t) {
      const int32_t ids[1] = {t};
      CK(fvsr_ring_step(ctx, ring, 0, t, k(t), v(t), q(t), ids, 1, &mask, topk, scale, 0, -1, out,
                        FVSR_OUT_TOKEN_MAJOR, 0, nullptr, nullptr, reinterpret_cast<fvsr_stream_t>(s)) == FVSR_OK);
      CK(fvsr_ring_evict_sliding(ring, 0) == FVSR_OK);
      CK(cudaMemcpyAsync(ref[t].data(), out, per_frame * 2, cudaMemcpyDeviceToHost, s) == cudaSuccess);
    }
    CK(cudaStreamSynchronize(s) == cudaSuccess);
    CK(fvsr_check_errors(ctx, reinterpret_cast<fvsr_stream_t>(s)) == FVSR_OK);
    cudaFree(out);
    fvsr_ring_destroy(ring);
    fvsr_ctx_destroy(ctx);
  }
  int bad = 0;
  uint16_t* out;
  CK(cudaMalloc(&out, per_frame * 2) == cudaSuccess);
  std::vector<uint16_t> got(per_frame);
  // world 1 with NCCL
  {
    ncclComm_t comm;
    int dev0 = 0;
    CK(ncclCommInitAll(&comm, 1, &dev0) == ncclSuccess);
    HeadParallelLayerStep hp(comm, 0, 1, 1, heads, d, rows, cols, window);
    bool ok = true;
    for (int t = 0; t < frames; ++t) {
      hp.step(0, t, q(t), k(t), v(t), mask, topk, scale, out, s);
      CK(cudaMemcpyAsync(got.data(), out, per_frame * 2, cudaMemcpyDeviceToHost, s) == cudaSuccess);
      CK(cudaStreamSynchronize(s) == cudaSuccess);
      ok = ok && got == ref[t];
    }
    hp.check_errors(s);
    std::printf("world 1 (NCCL all-gather): %s\n", ok ? "OK" : "MISMATCH");
    bad += ok ? 0 : 1;
    ncclCommDestroy(comm);
  }
  // simulated worlds: ranks one after another on this GPU, shards concatenated in rank order
  for (int world : {2, 4, 8}) {
    std::vector<HeadParallelLayerStep*> ranks;
    for (int r = 0; r < world; ++r) ranks.push_back(new HeadParallelLayerStep(nullptr, r, world, 1, heads, d, rows, cols, window));
    const Shard s0 = ranks[0]->shard();
    uint16_t* gathered;
    CK(cudaMalloc(&gathered, (size_t)s0.per * world * 64 * d * 2) == cudaSuccess);
    fvsr_ctx* ctx;
    CK(fvsr_ctx_create(&ctx) == FVSR_OK);
    bool ok = true;
    for (int t = 0; t < frames; ++t) {
      for (int r = 0; r < world; ++r) {
        ranks[r]->step(0, t, q(t), k(t), v(t), mask, topk, scale, nullptr, s);
        CK(cudaMemcpyAsync(gathered + (size_t)r * s0.per * 64 * d, ranks[r]->shard_buffer(), (size_t)s0.per * 64 * d * 2,
                           cudaMemcpyDeviceToDevice, s) == cudaSuccess);
      }
      CK(fvsr_untile(ctx, gathered, s0.total_units, 1, 1, rows, cols, d, out, reinterpret_cast<fvsr_stream_t>(s)) ==
         FVSR_OK);
      CK(cudaMemcpyAsync(got.data(), out, per_frame * 2, cudaMemcpyDeviceToHost, s) == cudaSuccess);
      CK(cudaStreamSynchronize(s) == cudaSuccess);
      ok = ok && got == ref[t];
    }
    for (auto* r : ranks) {
      r->check_errors(s);
      delete r;
    }
    std::printf("world %d (simulated ranks): %s\n", world, ok ? "OK" : "MISMATCH");
    bad += ok ? 0 : 1;
    cudaFree(gathered);
    fvsr_ctx_destroy(ctx);
  }
  return bad;
}

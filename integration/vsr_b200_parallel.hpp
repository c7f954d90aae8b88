// vsr_b200_parallel.hpp — head-parallel streaming layer-step for a C++ host, one process
// (or thread) per GPU, NCCL over NVLink for the only exchange: the all-gather of the
// bf16 head outputs.  The Python path (paper_2510_12747_b200/head_parallel.py) uses the
// same unit space, shard arithmetic and tile-major layout; this is the host-stays-C++ one.
//
// The reference processes a layer-step's heads one after another (head_attention per head,
// P/src/stream.cpp:237-256, P = the reference tree).  Heads, and within a head the query
// tiles, are independent given K/V, so the (head, q-tile) units are split contiguously over
// ranks:  per = ceil(U / world), rank r owns units [r * per, min(U, (r + 1) * per)) and a
// device ring holding only the heads [h0, h1) those units touch.  Each step:
//   1. fvsr_ring_step over the rank's unit range (ring append of its heads' new K/V, mask
//      builder, attention) -> tile-major shard [per][64][d] on the compute stream;
//   2. ncclAllGather of the shards (equal counts) on the communication stream, ordered after
//      the attention by an event;
//   3. fvsr_untile -> token-major [heads][rows * cols][d] on every rank, ordered after the
//      gather; then the sliding eviction.
// Every unit is computed whole by one CTA, so the gathered output is bitwise the single-GPU
// output (tests/test_gpu_head_parallel.py checks the same on the Python side).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>
#include <nccl.h>

#include "fvsr_b200.h"

namespace vsr::b200 {

struct Shard {
  long long total_units = 0, per = 0, u0 = 0, u1 = 0;
  int h0 = 0, h1 = 0;
};
// == paper_2510_12747_b200.head_parallel.shard
Shard shard_units(long long total_units, long long units_per_head, int world, int rank);

class HeadParallelLayerStep {
 public:
  // comm: an initialised communicator of `world` ranks (this object uses the current device),
  // or null: the step then stops at the tile-major shard (shard_buffer()) and the caller
  // gathers -- how tests simulate ranks on one GPU.
  HeadParallelLayerStep(ncclComm_t comm, int rank, int world, int layers, int heads, int d, int rows, int cols,
                        int window_frames);
  ~HeadParallelLayerStep();
  HeadParallelLayerStep(const HeadParallelLayerStep&) = delete;
  HeadParallelLayerStep& operator=(const HeadParallelLayerStep&) = delete;

  // One layer-step for query frame `frame_id` (Tq = 1).  q, k, v: DEVICE bf16 [heads][rows *
  // cols][d] for ALL heads (a rank reads its heads' slice); out: DEVICE bf16 [heads][rows *
  // cols][d], complete on every rank when `stream` reaches the end of the call's work.
  void step(int layer, int frame_id, const uint16_t* q, const uint16_t* k, const uint16_t* v, const fvsr_mask& mask,
            long long topk, float scale, uint16_t* out, cudaStream_t stream);

  const Shard& shard() const { return sh_; }
  const uint16_t* shard_buffer() const { return shard_buf_; }
  // device error word of this step's context (synchronises `stream`)
  void check_errors(cudaStream_t stream);

 private:
  ncclComm_t comm_;
  int rank_, world_, heads_, d_, rows_, cols_;
  long long tiles_;
  Shard sh_;
  fvsr_ctx* ctx_ = nullptr;
  fvsr_ring* ring_ = nullptr;
  uint16_t* shard_buf_ = nullptr;
  uint16_t* gathered_ = nullptr;
  cudaStream_t comm_stream_ = nullptr;
  cudaEvent_t computed_ = nullptr, gathered_ev_ = nullptr;
};

}  // namespace vsr::b200

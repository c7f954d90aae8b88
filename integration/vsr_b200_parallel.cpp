// vsr_b200_parallel.cpp — see vsr_b200_parallel.hpp.
#include "vsr_b200_parallel.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

namespace vsr::b200 {
namespace {

void check(int st, const char* where) {
  if (st != FVSR_OK) throw std::runtime_error(std::string(where) + ": " + fvsr_last_error());
}
void cuda_check(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}
void nccl_check(ncclResult_t r, const char* where) {
  if (r != ncclSuccess) throw std::runtime_error(std::string(where) + ": " + ncclGetErrorString(r));
}

}  // namespace

Shard shard_units(long long total_units, long long units_per_head, int world, int rank) {
  Shard s;
  s.total_units = total_units;
  s.per = (total_units + world - 1) / world;
  s.u0 = std::min(total_units, rank * s.per);
  s.u1 = std::min(total_units, s.u0 + s.per);
  if (s.u1 > s.u0) {
    s.h0 = static_cast<int>(s.u0 / units_per_head);
    s.h1 = static_cast<int>((s.u1 - 1) / units_per_head + 1);
  }
  return s;
}

HeadParallelLayerStep::HeadParallelLayerStep(ncclComm_t comm, int rank, int world, int layers, int heads, int d,
                                             int rows, int cols, int window_frames)
    : comm_(comm), rank_(rank), world_(world), heads_(heads), d_(d), rows_(rows), cols_(cols) {
  tiles_ = static_cast<long long>((rows + 7) / 8) * ((cols + 7) / 8);
  sh_ = shard_units(heads * tiles_, tiles_, world, rank);
  check(fvsr_ctx_create(&ctx_), "fvsr_ctx_create");
  if (sh_.u1 > sh_.u0)
    check(fvsr_ring_create(ctx_, layers, sh_.h1 - sh_.h0, d, rows, cols, window_frames, &ring_), "fvsr_ring_create");
  const size_t shard_elems = static_cast<size_t>(sh_.per) * 64 * d;
  cuda_check(cudaMalloc(&shard_buf_, shard_elems * 2), "cudaMalloc shard");
  cuda_check(cudaMemset(shard_buf_, 0, shard_elems * 2), "cudaMemset shard");
  cuda_check(cudaMalloc(&gathered_, shard_elems * world * 2), "cudaMalloc gathered");
  cuda_check(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  (void)rank_;
  (void)world_;
  cuda_check(cudaEventCreateWithFlags(&computed_, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaEventCreateWithFlags(&gathered_ev_, cudaEventDisableTiming), "cudaEventCreate");
}

HeadParallelLayerStep::~HeadParallelLayerStep() {
  if (ring_) fvsr_ring_destroy(ring_);
  if (ctx_) fvsr_ctx_destroy(ctx_);
  cudaFree(shard_buf_);
  cudaFree(gathered_);
  if (comm_stream_) cudaStreamDestroy(comm_stream_);
  if (computed_) cudaEventDestroy(computed_);
  if (gathered_ev_) cudaEventDestroy(gathered_ev_);
}

void HeadParallelLayerStep::step(int layer, int frame_id, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                                 const fvsr_mask& mask, long long topk, float scale, uint16_t* out,
                                 cudaStream_t stream) {
  const long long N = static_cast<long long>(rows_) * cols_;
  const fvsr_stream_t s = reinterpret_cast<fvsr_stream_t>(stream);
  // the previous step's gather must be done reading shard_buf_ (and writing gathered_)
  cuda_check(cudaStreamWaitEvent(stream, gathered_ev_, 0), "cudaStreamWaitEvent");
  if (ring_) {
    const long long hoff = static_cast<long long>(sh_.h0) * N * d_;
    const int32_t qids[1] = {frame_id};
    check(fvsr_ring_step(ctx_, ring_, layer, frame_id, k + hoff, v + hoff, q + hoff, qids, 1, &mask, topk, scale,
                         sh_.u0 - static_cast<long long>(sh_.h0) * tiles_,
                         sh_.u1 - static_cast<long long>(sh_.h0) * tiles_, shard_buf_, FVSR_OUT_TILE_MAJOR, 0,
                         nullptr, nullptr, s),
          "fvsr_ring_step");
    check(fvsr_ring_evict_sliding(ring_, layer), "fvsr_ring_evict_sliding");
  }
  if (!comm_) return;  // shard only (the caller gathers; tests simulate ranks on one GPU)
  // all-gather of the equal-size shards on the communication stream, after the attention
  cuda_check(cudaEventRecord(computed_, stream), "cudaEventRecord");
  cuda_check(cudaStreamWaitEvent(comm_stream_, computed_, 0), "cudaStreamWaitEvent");
  const size_t count = static_cast<size_t>(sh_.per) * 64 * d_;
  nccl_check(ncclAllGather(shard_buf_, gathered_, count, ncclBfloat16, comm_, comm_stream_), "ncclAllGather");
  cuda_check(cudaEventRecord(gathered_ev_, comm_stream_), "cudaEventRecord");
  cuda_check(cudaStreamWaitEvent(stream, gathered_ev_, 0), "cudaStreamWaitEvent");
  check(fvsr_untile(ctx_, gathered_, sh_.total_units, 1, 1, rows_, cols_, d_, out, s), "fvsr_untile");
}

void HeadParallelLayerStep::check_errors(cudaStream_t stream) {
  check(fvsr_check_errors(ctx_, reinterpret_cast<fvsr_stream_t>(stream)), "head-parallel step");
}

}  // namespace vsr::b200

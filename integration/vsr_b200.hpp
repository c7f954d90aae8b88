// vsr_b200.hpp — C++ drop-in for the reference's hot-path operator API, on the B200.
//
// Mirrors vsr::plan_sparse / vsr::sparse_attention_exec / vsr::sparsity_report
// (P/include/vsr/sparse.hpp:45-66, P = the reference tree) with the same value types
// (TensorF32, MaskMatrix, SparsePlan, SparsityReport) and the same exception taxonomy
// (P/include/vsr/common.hpp:10-53).  Compute runs in libfvsr_b200.so through the C-ABI
// (include/fvsr_b200.h); this layer only uploads, calls and downloads.
//
// One difference in the call shape: the GPU operators take the TokenGrids the partitions
// were built from (every call site has them: head_attention, P/src/stream.cpp:178-191;
// bench_sparsity, P/src/bench.cpp:88-101), because the device kernels work on the grid
// geometry directly instead of on materialised member lists.  The returned SparsePlan is a
// complete reference object (part_q / part_k from partition_blocks), so downstream
// reference code (sparsity_report, frame_attention_mass, validate) is unchanged.
//
// Inputs are fp32 tensors as in the reference; the device computes in bf16, so values are
// rounded to bf16 on upload (round-to-nearest-even).  For bit-identical plans feed the
// reference the same rounded values (tests do).
#pragma once

#include <cstddef>
#include <cstdint>

#include "vsr/grid.hpp"
#include "vsr/mask.hpp"
#include "vsr/sparse.hpp"
#include "vsr/tensor.hpp"

namespace vsr::b200 {

// Token mask for the GPU operators: an explicit MaskMatrix (uploaded as bits), the
// analytic locality window (no bitset is ever built), or all-allowed.
struct GpuMask {
  enum class Kind { all_allowed, locality, bits };
  Kind kind = Kind::all_allowed;
  LocalityWindow window{};
  const MaskMatrix* bits = nullptr;

  static GpuMask all() { return GpuMask{}; }
  static GpuMask from(const MaskMatrix& m) {
    GpuMask g;
    g.kind = Kind::bits;
    g.bits = &m;
    return g;
  }
  static GpuMask from(const LocalityWindow& w) {
    GpuMask g;
    g.kind = Kind::locality;
    g.window = w;
    return g;
  }
};

// == vsr::plan_sparse(q, k, partition_blocks(grid_q), partition_blocks(grid_k), mask, topk)
SparsePlan plan_sparse(const TensorF32& q, const TensorF32& k, const TokenGrid& grid_q,
                       const TokenGrid& grid_k, const GpuMask& mask, std::size_t topk);

// == vsr::sparse_attention_exec(q, k, v, plan, token_mask, scale, row_begin, row_end)
TensorF32 sparse_attention_exec(const TensorF32& q, const TensorF32& k, const TensorF32& v,
                                const SparsePlan& plan, const TokenGrid& grid_q,
                                const TokenGrid& grid_k, const GpuMask& token_mask, float scale,
                                std::size_t row_begin = 0, std::size_t row_end = SIZE_MAX);

// == vsr::sparsity_report(plan, mask), counted on the device
SparsityReport sparsity_report(const SparsePlan& plan, const TokenGrid& grid_q,
                               const TokenGrid& grid_k, const GpuMask& mask);

}  // namespace vsr::b200

// vsr_b200.cpp — C++ drop-in layer over the C-ABI (see vsr_b200.hpp).
//
// Upload fp32 -> bf16 device tensors, call include/fvsr_b200.h, download the results into
// the reference's value types and translate status codes into the reference's exceptions.
#include "vsr_b200.hpp"

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "fvsr_b200.h"
#include "vsr/common.hpp"
#include "vsr/partition.hpp"

namespace vsr::b200 {
namespace {

[[noreturn]] void throw_status(int st, const char* where) {
  std::string msg = std::string(where) + ": " + fvsr_last_error();
  switch (st) {
    case FVSR_E_SHAPE: throw ShapeError(msg);
    case FVSR_E_CONFIG: throw ConfigError(msg);
    case FVSR_E_DEGENERATE: throw DegenerateRowError(msg);
    case FVSR_E_EMPTY_BLOCK: throw EmptyBlockError(msg);
    case FVSR_E_INVARIANT: throw InvariantError(msg);
    default: throw Error(msg);
  }
}

void check(int st, const char* where) {
  if (st != FVSR_OK) throw_status(st, where);
}

void cuda_check(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw Error(std::string(where) + ": " + cudaGetErrorString(e));
}

// One context per host thread: its workspace is reused across calls (the reference's
// functions are pure and thread-safe; contexts are not shared between threads).
fvsr_ctx* context() {
  thread_local std::unique_ptr<fvsr_ctx, void (*)(fvsr_ctx*)> ctx(nullptr, fvsr_ctx_destroy);
  if (!ctx) {
    fvsr_ctx* c = nullptr;
    check(fvsr_ctx_create(&c), "fvsr_ctx_create");
    ctx.reset(c);
  }
  return ctx.get();
}

// Per-thread cache of device buffers by byte size: a call's buffers go back to the cache when
// it returns, so repeated calls with the same shapes do not allocate.  Calls on one thread
// are stream-ordered on the default stream and synchronise before returning, so a cached
// buffer is idle when it is handed out again.
struct BufCache {
  std::multimap<std::size_t, void*> free_;
  ~BufCache() {
    for (auto& kv : free_) cudaFree(kv.second);
  }
  void* get(std::size_t bytes) {
    auto it = free_.find(bytes);
    if (it != free_.end()) {
      void* p = it->second;
      free_.erase(it);
      return p;
    }
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    return p;
  }
  void put(std::size_t bytes, void* p) { free_.emplace(bytes, p); }
};
BufCache& buf_cache() {
  thread_local BufCache c;
  return c;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  std::size_t bytes = 0;
  explicit DevBuf(std::size_t n) : bytes(n * sizeof(T)) {
    if (n) p = static_cast<T*>(buf_cache().get(bytes));
  }
  ~DevBuf() {
    if (p) buf_cache().put(bytes, p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

uint16_t to_bf16(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return static_cast<uint16_t>((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
  return static_cast<uint16_t>(u >> 16);
}

float from_bf16(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

// [L x d] fp32 host tensor -> bf16 device buffer
std::unique_ptr<DevBuf<uint16_t>> upload(const TensorF32& t, const char* what) {
  VSR_REQUIRE(t.rank() == 2, ShapeError, std::string(what) + ": expected a [tokens x d] tensor");
  std::vector<uint16_t> h(t.numel());
  for (std::size_t i = 0; i < h.size(); ++i) h[i] = to_bf16(t.data[i]);
  auto d = std::make_unique<DevBuf<uint16_t>>(h.size());
  cuda_check(cudaMemcpy(d->p, h.data(), h.size() * 2, cudaMemcpyHostToDevice), what);
  return d;
}

struct Grid {
  std::vector<int32_t> ids;
  fvsr_grid g{};
  explicit Grid(const TokenGrid& t) : ids(t.frame_ids().begin(), t.frame_ids().end()) {
    g.frame_ids = ids.data();
    g.n_frames = static_cast<int32_t>(ids.size());
    g.rows = static_cast<int32_t>(t.rows());
    g.cols = static_cast<int32_t>(t.cols());
  }
};

struct Mask {
  fvsr_mask m{};
  std::unique_ptr<DevBuf<uint64_t>> bits;
  Mask(const GpuMask& gm, const TokenGrid& gq, const TokenGrid& gk) {
    switch (gm.kind) {
      case GpuMask::Kind::all_allowed:
        m.kind = FVSR_MASK_ALL;
        break;
      case GpuMask::Kind::locality:
        // build_locality_mask's frame extents are the grid's (P/src/mask.cpp:114-121)
        VSR_REQUIRE(gm.window.frame_extent_h == static_cast<int>(gq.rows()) &&
                        gm.window.frame_extent_w == static_cast<int>(gq.cols()),
                    ConfigError, "GpuMask: locality frame extents must equal the grid's rows/cols");
        m.kind = FVSR_MASK_LOCALITY;
        m.mode = gm.window.mode == LocalityWindow::Mode::boundary_truncated ? FVSR_LOCALITY_TRUNCATED
                                                                            : FVSR_LOCALITY_PRESERVED;
        m.extent_h = gm.window.extent_h;
        m.extent_w = gm.window.extent_w;
        break;
      case GpuMask::Kind::bits: {
        const MaskMatrix& mm = *gm.bits;
        VSR_REQUIRE(mm.rows() == gq.token_count() && mm.cols() == gk.token_count(), ShapeError,
                    "GpuMask: mask shape does not match the grids");
        const std::size_t n = mm.rows() * mm.words_per_row();
        bits = std::make_unique<DevBuf<uint64_t>>(n);
        cuda_check(cudaMemcpy(bits->p, mm.row_words(0), n * 8, cudaMemcpyHostToDevice), "mask upload");
        m.kind = FVSR_MASK_BITMASK;
        m.bits = bits->p;
        m.words_per_row = static_cast<int64_t>(mm.words_per_row());
        break;
      }
    }
  }
};

std::size_t block_count(const TokenGrid& gq, const TokenGrid& gk, bool q) {
  Grid a(gq), b(gk);
  int32_t bnq = 0, bnk = 0;
  check(fvsr_block_counts(&a.g, &b.g, &bnq, &bnk), "fvsr_block_counts");
  return static_cast<std::size_t>(q ? bnq : bnk);
}

}  // namespace

SparsePlan plan_sparse(const TensorF32& q, const TensorF32& k, const TokenGrid& grid_q,
                       const TokenGrid& grid_k, const GpuMask& mask, std::size_t topk) {
  VSR_REQUIRE(q.rank() == 2 && k.rank() == 2 && q.shape[1] == k.shape[1], ShapeError,
              "plan_sparse: q/k must be [tokens x d] with equal d");
  VSR_REQUIRE(q.shape[0] == grid_q.token_count() && k.shape[0] == grid_k.token_count(), ShapeError,
              "plan_sparse: tensor rows must match the grids");
  VSR_REQUIRE(topk >= 1, ConfigError, "plan_sparse: topk must be >= 1");
  fvsr_ctx* ctx = context();
  const int32_t d = static_cast<int32_t>(q.shape[1]);
  Grid gq(grid_q), gk(grid_k);
  Mask m(mask, grid_q, grid_k);
  const std::size_t bnq = block_count(grid_q, grid_k, true), bnk = block_count(grid_q, grid_k, false);
  const int32_t cap = static_cast<int32_t>(std::max<std::size_t>(1, std::min(topk, bnk)));
  auto dq = upload(q, "plan_sparse q");
  auto dk = upload(k, "plan_sparse k");
  DevBuf<int32_t> sel(bnq * cap), cnt(bnq), diag(bnq);
  DevBuf<float> coarse(bnq * bnk);
  DevBuf<uint8_t> allowed(bnq * bnk);
  check(fvsr_plan_sparse(ctx, dq->p, dk->p, 1, d, &gq.g, &gk.g, &m.m, static_cast<int64_t>(topk), cap, sel.p,
                         cnt.p, diag.p, coarse.p, allowed.p, nullptr),
        "plan_sparse");
  check(fvsr_check_errors(ctx, nullptr), "plan_sparse");

  std::vector<int32_t> hsel(bnq * cap), hcnt(bnq), hdiag(bnq);
  std::vector<uint8_t> hallowed(bnq * bnk);
  SparsePlan plan;
  plan.topk = topk;
  plan.head_dim = static_cast<std::size_t>(d);
  plan.part_q = partition_blocks(grid_q);
  plan.part_k = partition_blocks(grid_k);
  plan.coarse_scores = TensorF32({bnq, bnk});
  cuda_check(cudaMemcpy(hsel.data(), sel.p, hsel.size() * 4, cudaMemcpyDeviceToHost), "download");
  cuda_check(cudaMemcpy(hcnt.data(), cnt.p, hcnt.size() * 4, cudaMemcpyDeviceToHost), "download");
  cuda_check(cudaMemcpy(hdiag.data(), diag.p, hdiag.size() * 4, cudaMemcpyDeviceToHost), "download");
  cuda_check(cudaMemcpy(plan.coarse_scores.data.data(), coarse.p, bnq * bnk * 4, cudaMemcpyDeviceToHost),
             "download");
  cuda_check(cudaMemcpy(hallowed.data(), allowed.p, hallowed.size(), cudaMemcpyDeviceToHost), "download");
  plan.coarse_allowed = MaskMatrix(bnq, bnk, false);
  for (std::size_t i = 0; i < bnq; ++i)
    for (std::size_t j = 0; j < bnk; ++j)
      if (hallowed[i * bnk + j]) plan.coarse_allowed.set(i, j, true);
  plan.selected.resize(bnq);
  plan.diagonal_block.resize(bnq);
  for (std::size_t i = 0; i < bnq; ++i) {
    plan.selected[i].assign(hsel.begin() + i * cap, hsel.begin() + i * cap + hcnt[i]);
    plan.diagonal_block[i] = hdiag[i];
  }
  return plan;
}

TensorF32 sparse_attention_exec(const TensorF32& q, const TensorF32& k, const TensorF32& v,
                                const SparsePlan& plan, const TokenGrid& grid_q,
                                const TokenGrid& grid_k, const GpuMask& token_mask, float scale,
                                std::size_t row_begin, std::size_t row_end) {
  VSR_REQUIRE(k.same_shape(v), ShapeError, "sparse_attention_exec: k/v shape mismatch");
  VSR_REQUIRE(q.shape[0] == plan.part_q.token_count && k.shape[0] == plan.part_k.token_count, ShapeError,
              "sparse_attention_exec: tensors do not match the plan's partitions");
  VSR_REQUIRE(row_begin <= row_end, ConfigError, "sparse_attention_exec: row_begin > row_end");
  fvsr_ctx* ctx = context();
  const int32_t d = static_cast<int32_t>(q.shape[1]);
  Grid gq(grid_q), gk(grid_k);
  Mask m(token_mask, grid_q, grid_k);
  const std::size_t bnq = plan.selected.size();
  std::size_t cap = 1;
  for (const auto& s : plan.selected) cap = std::max(cap, s.size());
  std::vector<int32_t> hsel(bnq * cap, -1), hcnt(bnq);
  for (std::size_t i = 0; i < bnq; ++i) {
    hcnt[i] = static_cast<int32_t>(plan.selected[i].size());
    for (std::size_t t = 0; t < plan.selected[i].size(); ++t) hsel[i * cap + t] = plan.selected[i][t];
  }
  DevBuf<int32_t> sel(hsel.size()), cnt(bnq);
  cuda_check(cudaMemcpy(sel.p, hsel.data(), hsel.size() * 4, cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(cnt.p, hcnt.data(), hcnt.size() * 4, cudaMemcpyHostToDevice), "upload");
  auto dq = upload(q, "sparse_attention_exec q");
  auto dk = upload(k, "sparse_attention_exec k");
  auto dv = upload(v, "sparse_attention_exec v");
  const std::size_t L = q.shape[0];
  DevBuf<uint16_t> out(L * d);
  const int64_t rb = static_cast<int64_t>(row_begin);
  const int64_t re = row_end >= L ? -1 : static_cast<int64_t>(row_end);
  check(fvsr_sparse_attention_exec(ctx, dq->p, dk->p, dv->p, 1, d, &gq.g, &gk.g, &m.m, static_cast<int32_t>(cap),
                                   sel.p, cnt.p, scale, rb, re, out.p, nullptr),
        "sparse_attention_exec");
  check(fvsr_check_errors(ctx, nullptr), "sparse_attention_exec");
  std::vector<uint16_t> h(L * d);
  cuda_check(cudaMemcpy(h.data(), out.p, h.size() * 2, cudaMemcpyDeviceToHost), "download");
  TensorF32 res({L, static_cast<std::size_t>(d)});
  for (std::size_t i = 0; i < h.size(); ++i) res.data[i] = from_bf16(h[i]);
  return res;
}

SparsityReport sparsity_report(const SparsePlan& plan, const TokenGrid& grid_q, const TokenGrid& grid_k,
                               const GpuMask& mask) {
  fvsr_ctx* ctx = context();
  Grid gq(grid_q), gk(grid_k);
  Mask m(mask, grid_q, grid_k);
  const std::size_t bnq = plan.selected.size();
  std::size_t cap = 1;
  for (const auto& s : plan.selected) cap = std::max(cap, s.size());
  std::vector<int32_t> hsel(bnq * cap, -1), hcnt(bnq);
  for (std::size_t i = 0; i < bnq; ++i) {
    hcnt[i] = static_cast<int32_t>(plan.selected[i].size());
    for (std::size_t t = 0; t < plan.selected[i].size(); ++t) hsel[i * cap + t] = plan.selected[i][t];
  }
  DevBuf<int32_t> sel(hsel.size()), cnt(bnq);
  DevBuf<uint64_t> out(4);
  cuda_check(cudaMemcpy(sel.p, hsel.data(), hsel.size() * 4, cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(cnt.p, hcnt.data(), hcnt.size() * 4, cudaMemcpyHostToDevice), "upload");
  check(fvsr_sparsity_report(ctx, 1, &gq.g, &gk.g, &m.m, static_cast<int32_t>(cap), sel.p, cnt.p, out.p, out.p + 1,
                             out.p + 2, out.p + 3, nullptr),
        "sparsity_report");
  uint64_t h[4];
  cuda_check(cudaMemcpy(h, out.p, sizeof(h), cudaMemcpyDeviceToHost), "download");
  // density = selected / allowed block pairs; flops = pairs * (2d + 2) (P/src/sparse.cpp:256-285)
  VSR_REQUIRE(h[3] > 0, InvariantError, "sparsity_report: no allowed block pairs");
  SparsityReport rep;
  const uint64_t per_pair = 2 * static_cast<uint64_t>(plan.head_dim) + 2;
  rep.density = static_cast<double>(h[2]) / static_cast<double>(h[3]);
  rep.executed_flops = h[0] * per_pair;
  rep.dense_flops = h[1] * per_pair;
  rep.flop_ratio = h[1] == 0 ? 0.0 : static_cast<double>(h[0]) / static_cast<double>(h[1]);
  return rep;
}

}  // namespace vsr::b200

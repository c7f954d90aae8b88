// vsr_b200_sparse.cpp — the reference's hot-path operators with their EXACT signatures
// (P/include/vsr/sparse.hpp:16-66, P = the reference tree), implemented on the B200.
//
// Link this object in place of P/src/sparse.cpp: every caller of vsr::plan_sparse,
// vsr::sparse_attention_exec, vsr::sparsity_report and the SparsePlan helpers (head_attention
// in P/src/stream.cpp, bench_sparsity, the checks, the reference's own tests/test_sparse.cpp)
// then runs on the GPU unmodified.  integration/Makefile builds the reference's
// tests/test_sparse.cpp this way (ref_test_sparse_b200).
//
//   * The token geometry the device kernels need (frame ids, rows, cols) is recovered from
//     the BlockPartition: the first TokenGrid whose partition_blocks() reproduces the given
//     partition (same token count, keys and member lists) -- any such grid yields identical
//     plans and outputs, because the reference's operators only see member lists.
//   * The plan runs on the fp32 inputs (fvsr_plan_sparse_f32): indices, coarse scores and
//     coarse-allowed are bit-exact with the CPU reference on any data.
//   * The attention runs on the tensor cores in bf16 (inputs rounded on upload, fp32
//     online softmax, bf16 output): outputs agree with the fp32 reference within the bf16
//     tolerance of tests/helpers.py, not the reference's 1e-5 fp32 budget.  Head dims below
//     64 (the reference tests use 8 and 16) are zero-padded to 64 on upload.
//   * An all-allowed MaskMatrix is detected and passed as such; any other mask goes to the
//     device as its bits.  `threads` is accepted and ignored (one stream-ordered launch).
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "fvsr_b200.h"
#include "vsr/common.hpp"
#include "vsr/partition.hpp"
#include "vsr/sparse.hpp"
#include "vsr_b200.hpp"

namespace vsr {
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

fvsr_ctx* context() {
  thread_local struct Holder {
    fvsr_ctx* c = nullptr;
    ~Holder() { fvsr_ctx_destroy(c); }
  } h;
  if (!h.c) check(fvsr_ctx_create(&h.c), "fvsr_ctx_create");
  return h.c;
}

// device buffers reused across calls (grown on demand)
struct Scratch {
  void* p = nullptr;
  std::size_t n = 0;
  void* get(std::size_t bytes) {
    if (bytes > n) {
      if (p) cudaFree(p);
      p = nullptr;
      n = 0;
      cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
      n = bytes;
    }
    return p;
  }
  ~Scratch() {
    if (p) cudaFree(p);
  }
};
thread_local Scratch s_q, s_k, s_v, s_out, s_sel, s_cnt, s_diag, s_coarse, s_allowed, s_mask, s_rep;

bool same_partition(const BlockPartition& a, const BlockPartition& b) {
  return a.token_count == b.token_count && a.block_num == b.block_num && a.block_keys == b.block_keys &&
         a.block_tokens == b.block_tokens;
}

// A TokenGrid whose partition_blocks() reproduces `part` (see the file header).
TokenGrid grid_of(const BlockPartition& part) {
  VSR_REQUIRE(part.block_num > 0 && part.token_count > 0, ShapeError, "B200 sparse: empty partition");
  int th = 0, tw = 0;
  std::vector<int> trows;
  for (const auto& key : part.block_keys) {
    th = std::max(th, key[1] + 1);
    tw = std::max(tw, key[2] + 1);
    if (trows.empty() || trows.back() != key[0]) trows.push_back(key[0]);
  }
  for (int rows = 8 * (th - 1) + 1; rows <= 8 * th; ++rows)
    for (int cols = 8 * (tw - 1) + 1; cols <= 8 * tw; ++cols) {
      const std::size_t N = static_cast<std::size_t>(rows) * cols;
      if (part.token_count % N) continue;
      // frames per temporal row from the size of its first block (tile (0, 0))
      std::vector<int> ids;
      std::size_t b = 0;
      bool ok = true;
      const std::size_t tile0 = static_cast<std::size_t>(std::min(8, rows)) * std::min(8, cols);
      for (int tr : trows) {
        while (b < part.block_num && part.block_keys[b][0] != tr) ++b;
        const std::size_t sz = part.block_tokens[b].size();
        if (sz != tile0 && sz != 2 * tile0) { ok = false; break; }
        ids.push_back(2 * tr);
        if (sz == 2 * tile0) ids.push_back(2 * tr + 1);
      }
      if (!ok || ids.size() * N != part.token_count) continue;
      TokenGrid g(ids, static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
      if (same_partition(partition_blocks(g), part)) return g;
    }
  throw ShapeError("B200 sparse: no token grid reproduces this block partition");
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

bool all_allowed(const MaskMatrix& m) {
  const std::size_t wpr = m.words_per_row(), tail = m.cols() % 64;
  const std::uint64_t last = tail ? ((1ull << tail) - 1ull) : ~0ull;
  for (std::size_t i = 0; i < m.rows(); ++i) {
    const std::uint64_t* w = m.row_words(i);
    for (std::size_t j = 0; j + 1 < wpr; ++j)
      if (w[j] != ~0ull) return false;
    if (wpr && (w[wpr - 1] & last) != last) return false;
  }
  return true;
}

fvsr_mask device_mask(const MaskMatrix& m) {
  fvsr_mask d{};
  if (all_allowed(m)) {
    d.kind = FVSR_MASK_ALL;
    return d;
  }
  const std::size_t n = m.rows() * m.words_per_row();
  void* p = s_mask.get(std::max<std::size_t>(8, n * 8));
  cuda_check(cudaMemcpy(p, m.row_words(0), n * 8, cudaMemcpyHostToDevice), "mask upload");
  d.kind = FVSR_MASK_BITMASK;
  d.bits = static_cast<const uint64_t*>(p);
  d.words_per_row = static_cast<int64_t>(m.words_per_row());
  return d;
}

uint16_t to_bf16(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return static_cast<uint16_t>((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

void* upload_f32(Scratch& s, const TensorF32& t) {
  void* p = s.get(std::max<std::size_t>(4, t.numel() * 4));
  cuda_check(cudaMemcpy(p, t.data.data(), t.numel() * 4, cudaMemcpyHostToDevice), "upload");
  return p;
}
// [L x d] fp32 -> bf16 [L x dp], channels d..dp-1 zero (zero channels add nothing to q.k and
// their output columns are dropped: the tensor-core kernel's head dims are 64 and 128)
void* upload_bf16(Scratch& s, const TensorF32& t, std::size_t dp) {
  const std::size_t L = t.shape[0], d = t.shape[1];
  std::vector<uint16_t> h(L * dp, 0);
  for (std::size_t i = 0; i < L; ++i)
    for (std::size_t c = 0; c < d; ++c) h[i * dp + c] = to_bf16(t.data[i * d + c]);
  void* p = s.get(std::max<std::size_t>(2, h.size() * 2));
  cuda_check(cudaMemcpy(p, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "upload");
  return p;
}

// plan.selected -> device [bnq][cap] (-1 padded) + counts
int32_t upload_selection(const SparsePlan& plan, int32_t** sel, int32_t** cnt) {
  const std::size_t bnq = plan.selected.size();
  std::size_t cap = 1;
  for (const auto& s : plan.selected) cap = std::max(cap, s.size());
  std::vector<int32_t> hsel(bnq * cap, -1), hcnt(bnq);
  for (std::size_t i = 0; i < bnq; ++i) {
    hcnt[i] = static_cast<int32_t>(plan.selected[i].size());
    for (std::size_t t = 0; t < plan.selected[i].size(); ++t) hsel[i * cap + t] = plan.selected[i][t];
  }
  *sel = static_cast<int32_t*>(s_sel.get(std::max<std::size_t>(4, hsel.size() * 4)));
  *cnt = static_cast<int32_t*>(s_cnt.get(std::max<std::size_t>(4, hcnt.size() * 4)));
  cuda_check(cudaMemcpy(*sel, hsel.data(), hsel.size() * 4, cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(*cnt, hcnt.data(), hcnt.size() * 4, cudaMemcpyHostToDevice), "upload");
  return static_cast<int32_t>(cap);
}

}  // namespace

std::size_t SparsePlan::selected_pairs() const {
  std::size_t n = 0;
  for (const auto& s : selected) n += s.size();
  return n;
}

std::size_t SparsePlan::allowed_pairs() const { return coarse_allowed.count_allowed(); }

// SparsePlan invariants (the reference's contract, P/src/sparse.cpp:20-45)
void SparsePlan::validate() const {
  const std::size_t bnq = part_q.block_num, bnk = part_k.block_num;
  VSR_REQUIRE(topk >= 1, InvariantError, "SparsePlan: topk must be >= 1");
  VSR_REQUIRE(selected.size() == bnq && diagonal_block.size() == bnq, InvariantError,
              "SparsePlan: per-query-block table sizes disagree");
  VSR_REQUIRE(coarse_scores.rank() == 2 && coarse_scores.shape[0] == bnq && coarse_scores.shape[1] == bnk,
              InvariantError, "SparsePlan: coarse score shape mismatch");
  for (std::size_t qb = 0; qb < bnq; ++qb) {
    const std::vector<int>& s = selected[qb];
    VSR_REQUIRE(s.size() <= topk, InvariantError, "SparsePlan: selection exceeds k");
    for (std::size_t t = 0; t < s.size(); ++t) {
      VSR_REQUIRE(t == 0 || s[t - 1] < s[t], InvariantError, "SparsePlan: selection not sorted unique");
      VSR_REQUIRE(s[t] >= 0 && static_cast<std::size_t>(s[t]) < bnk, InvariantError,
                  "SparsePlan: key block id out of range");
      VSR_REQUIRE(coarse_allowed.allowed(qb, static_cast<std::size_t>(s[t])), InvariantError,
                  "SparsePlan: selection not mask-allowed");
    }
    const int dg = diagonal_block[qb];
    if (dg >= 0 && coarse_allowed.allowed(qb, static_cast<std::size_t>(dg)))
      VSR_REQUIRE(std::find(s.begin(), s.end(), dg) != s.end(), InvariantError,
                  "SparsePlan: diagonal block missing from selection");
  }
}

SparsePlan plan_sparse(const TensorF32& q, const TensorF32& k, const BlockPartition& part_q,
                       const BlockPartition& part_k, const MaskMatrix& mask, std::size_t topk) {
  VSR_REQUIRE(q.rank() == 2 && k.rank() == 2 && q.shape[1] == k.shape[1], ShapeError,
              "plan_sparse: q/k dim mismatch");
  VSR_REQUIRE(q.shape[0] == part_q.token_count && k.shape[0] == part_k.token_count, ShapeError,
              "plan_sparse: partitions do not cover the inputs");
  VSR_REQUIRE(mask.rows() == part_q.token_count && mask.cols() == part_k.token_count, ShapeError,
              "plan_sparse: mask shape mismatch");
  VSR_REQUIRE(topk >= 1, ConfigError, "plan_sparse: topk must be >= 1");
  fvsr_ctx* ctx = context();
  const TokenGrid tq = grid_of(part_q), tk = grid_of(part_k);
  Grid gq(tq), gk(tk);
  const fvsr_mask dm = device_mask(mask);
  const std::size_t bnq = part_q.block_num, bnk = part_k.block_num;
  const int32_t cap = static_cast<int32_t>(std::max<std::size_t>(1, std::min(topk, bnk)));
  const int32_t d = static_cast<int32_t>(q.shape[1]);
  auto* dq = static_cast<const float*>(upload_f32(s_q, q));
  auto* dk = static_cast<const float*>(upload_f32(s_k, k));
  auto* sel = static_cast<int32_t*>(s_sel.get(bnq * cap * 4));
  auto* cnt = static_cast<int32_t*>(s_cnt.get(bnq * 4));
  auto* dg = static_cast<int32_t*>(s_diag.get(bnq * 4));
  auto* coarse = static_cast<float*>(s_coarse.get(std::max<std::size_t>(4, bnq * bnk * 4)));
  auto* allowed = static_cast<uint8_t*>(s_allowed.get(std::max<std::size_t>(1, bnq * bnk)));
  check(fvsr_plan_sparse_f32(ctx, dq, dk, 1, d, &gq.g, &gk.g, &dm, static_cast<int64_t>(topk), cap, sel, cnt, dg,
                             coarse, allowed, nullptr),
        "plan_sparse");
  check(fvsr_check_errors(ctx, nullptr), "plan_sparse");
  std::vector<int32_t> hsel(bnq * cap), hcnt(bnq), hdg(bnq);
  std::vector<uint8_t> hal(bnq * bnk);
  SparsePlan plan;
  plan.topk = topk;
  plan.head_dim = static_cast<std::size_t>(d);
  plan.part_q = part_q;
  plan.part_k = part_k;
  plan.coarse_scores = TensorF32({bnq, bnk});
  cuda_check(cudaMemcpy(hsel.data(), sel, hsel.size() * 4, cudaMemcpyDeviceToHost), "download");
  cuda_check(cudaMemcpy(hcnt.data(), cnt, hcnt.size() * 4, cudaMemcpyDeviceToHost), "download");
  cuda_check(cudaMemcpy(hdg.data(), dg, hdg.size() * 4, cudaMemcpyDeviceToHost), "download");
  cuda_check(cudaMemcpy(plan.coarse_scores.data.data(), coarse, bnq * bnk * 4, cudaMemcpyDeviceToHost), "download");
  cuda_check(cudaMemcpy(hal.data(), allowed, hal.size(), cudaMemcpyDeviceToHost), "download");
  plan.coarse_allowed = MaskMatrix(bnq, bnk, false);
  for (std::size_t i = 0; i < bnq; ++i)
    for (std::size_t j = 0; j < bnk; ++j)
      if (hal[i * bnk + j]) plan.coarse_allowed.set(i, j, true);
  plan.selected.resize(bnq);
  plan.diagonal_block.resize(bnq);
  for (std::size_t i = 0; i < bnq; ++i) {
    plan.selected[i].assign(hsel.begin() + i * cap, hsel.begin() + i * cap + hcnt[i]);
    plan.diagonal_block[i] = hdg[i];
  }
  return plan;
}

SparsePlan plan_sparse(const TensorF32& q, const TensorF32& k, const BlockPartition& part, const MaskMatrix& mask,
                       std::size_t topk) {
  return plan_sparse(q, k, part, part, mask, topk);
}

TensorF32 sparse_attention_exec(const TensorF32& q, const TensorF32& k, const TensorF32& v, const SparsePlan& plan,
                                const MaskMatrix& token_mask, float scale, std::size_t row_begin,
                                std::size_t row_end, unsigned /*threads*/) {
  VSR_REQUIRE(k.same_shape(v), ShapeError, "sparse_attention_exec: k/v shape mismatch");
  VSR_REQUIRE(q.rank() == 2 && q.shape[0] == plan.part_q.token_count && k.shape[0] == plan.part_k.token_count,
              ShapeError, "sparse_attention_exec: plan does not match inputs");
  VSR_REQUIRE(token_mask.rows() == q.shape[0] && token_mask.cols() == k.shape[0], ShapeError,
              "sparse_attention_exec: mask shape mismatch");
  const std::size_t L = q.shape[0];
  const std::size_t re = std::min(row_end, L);
  VSR_REQUIRE(row_begin <= re, ConfigError, "sparse_attention_exec: empty or inverted row range");
  fvsr_ctx* ctx = context();
  const TokenGrid tq = grid_of(plan.part_q), tk = grid_of(plan.part_k);
  Grid gq(tq), gk(tk);
  const fvsr_mask dm = device_mask(token_mask);
  int32_t *sel, *cnt;
  const int32_t cap = upload_selection(plan, &sel, &cnt);
  const std::size_t d = q.shape[1];
  VSR_REQUIRE(d >= 1 && d <= 128 && v.shape[1] == d, ShapeError, "sparse_attention_exec: head dim must be <= 128");
  const std::size_t dp = d <= 64 ? 64 : 128;  // zero-padded to the kernel's head dim
  auto* dq = static_cast<const uint16_t*>(upload_bf16(s_q, q, dp));
  auto* dk = static_cast<const uint16_t*>(upload_bf16(s_k, k, dp));
  auto* dv = static_cast<const uint16_t*>(upload_bf16(s_v, v, dp));
  auto* out = static_cast<uint16_t*>(s_out.get(L * dp * 2));
  check(fvsr_sparse_attention_exec(ctx, dq, dk, dv, 1, static_cast<int32_t>(dp), &gq.g, &gk.g, &dm, cap, sel, cnt, scale,
                                   static_cast<int64_t>(row_begin), re >= L ? -1 : static_cast<int64_t>(re), out,
                                   nullptr),
        "sparse_attention_exec");
  check(fvsr_check_errors(ctx, nullptr), "sparse_attention_exec");
  std::vector<uint16_t> h(L * dp);
  cuda_check(cudaMemcpy(h.data(), out, h.size() * 2, cudaMemcpyDeviceToHost), "download");
  TensorF32 res({L, d});
  for (std::size_t i = 0; i < L; ++i)
    for (std::size_t c = 0; c < d; ++c) {
      const uint32_t u = static_cast<uint32_t>(h[i * dp + c]) << 16;
      std::memcpy(&res.data[i * d + c], &u, 4);
    }
  return res;
}

SparsityReport sparsity_report(const SparsePlan& plan, const MaskMatrix& mask) {
  fvsr_ctx* ctx = context();
  const TokenGrid tq = grid_of(plan.part_q), tk = grid_of(plan.part_k);
  Grid gq(tq), gk(tk);
  const fvsr_mask dm = device_mask(mask);
  int32_t *sel, *cnt;
  const int32_t cap = upload_selection(plan, &sel, &cnt);
  auto* o = static_cast<uint64_t*>(s_rep.get(4 * 8));
  check(fvsr_sparsity_report(ctx, 1, &gq.g, &gk.g, &dm, cap, sel, cnt, o, o + 1, o + 2, o + 3, nullptr),
        "sparsity_report");
  uint64_t h[4];
  cuda_check(cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost), "download");
  // density = selected / allowed block pairs; flops = pairs x (2d + 2) (P/src/sparse.cpp:256-285)
  VSR_REQUIRE(h[3] > 0, InvariantError, "sparsity_report: no allowed block pairs");
  SparsityReport rep;
  const uint64_t per_pair = 2 * static_cast<uint64_t>(plan.head_dim) + 2;
  rep.density = static_cast<double>(h[2]) / static_cast<double>(h[3]);
  rep.executed_flops = h[0] * per_pair;
  rep.dense_flops = h[1] * per_pair;
  rep.flop_ratio = h[1] == 0 ? 0.0 : static_cast<double>(h[0]) / static_cast<double>(h[1]);
  return rep;
}

}  // namespace vsr

// parity_main.cpp — the reference's own operators vs the B200 drop-in, in one process.
//
// Test infrastructure (run by tests/test_gpu_facade.py on a B200): every case calls the
// UNMODIFIED reference (vsr::plan_sparse / sparse_attention_exec / sparsity_report, linked
// from oracle/_ref) and vsr::b200 (libfvsr_b200.so) on identical bf16-representable inputs
// and checks:
//   plan   — selected ids, diagonal, coarse-allowed and coarse-score bits identical
//   exec   — rel L2 <= 5e-3 and max |diff| <= 2e-2 against the reference's fp32 output
//   report — density / executed / dense flops identical
//   errors — DegenerateRowError surfaces as the same exception type
// Cases follow P/tests/test_sparse.cpp and the streaming shapes of BASELINE.json.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "vsr/common.hpp"
#include "vsr/mask.hpp"
#include "vsr/partition.hpp"
#include "vsr/rng.hpp"
#include "vsr/sparse.hpp"
#include "vsr_b200.hpp"

using namespace vsr;

namespace {

float bf16_round(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  float y;
  std::memcpy(&y, &u, 4);
  return y;
}

TensorF32 gaussian_bf16(std::size_t rows, std::size_t d, Rng& rng) {
  TensorF32 t = TensorF32::gaussian({rows, d}, rng);
  for (float& x : t.data) x = bf16_round(x);
  return t;
}

int failures = 0;
#define EXPECT(cond, ...)                  \
  do {                                     \
    if (!(cond)) {                         \
      std::printf("  FAIL: " __VA_ARGS__); \
      std::printf("\n");                   \
      ++failures;                          \
    }                                      \
  } while (0)

struct Case {
  const char* name;
  uint64_t seed;
  std::size_t d;
  std::vector<int> qf, kf;
  std::size_t rows, cols;
  int mask;  // 0 all, 1 locality truncated, 2 locality preserved (analytic), 3 locality as MaskMatrix bits
  int eh, ew;
  std::size_t topk;
};

void run_case(const Case& c) {
  std::printf("case %s\n", c.name);
  const TokenGrid gq(c.qf, c.rows, c.cols), gk(c.kf, c.rows, c.cols);
  Rng rng(c.seed);
  const TensorF32 q = gaussian_bf16(gq.token_count(), c.d, rng);
  const TensorF32 k = gaussian_bf16(gk.token_count(), c.d, rng);
  const TensorF32 v = gaussian_bf16(gk.token_count(), c.d, rng);
  LocalityWindow win;
  win.mode = c.mask == 2 ? LocalityWindow::Mode::boundary_preserved : LocalityWindow::Mode::boundary_truncated;
  win.extent_h = c.eh;
  win.extent_w = c.ew;
  win.frame_extent_h = static_cast<int>(c.rows);
  win.frame_extent_w = static_cast<int>(c.cols);
  const MaskMatrix mask = c.mask == 0 ? MaskMatrix::all_allowed(gq.token_count(), gk.token_count())
                                      : build_locality_mask(win, gq.positions(), gk.positions());
  const b200::GpuMask gmask =
      c.mask == 0 ? b200::GpuMask::all() : (c.mask == 3 ? b200::GpuMask::from(mask) : b200::GpuMask::from(win));

  // ---- plan ----
  const SparsePlan ref = plan_sparse(q, k, partition_blocks(gq), partition_blocks(gk), mask, c.topk);
  const SparsePlan gpu = b200::plan_sparse(q, k, gq, gk, gmask, c.topk);
  gpu.validate();
  EXPECT(gpu.selected == ref.selected, "selected ids differ");
  EXPECT(gpu.diagonal_block == ref.diagonal_block, "diagonal blocks differ");
  EXPECT(gpu.coarse_allowed == ref.coarse_allowed, "coarse_allowed differs");
  EXPECT(gpu.coarse_scores.shape == ref.coarse_scores.shape &&
             std::memcmp(gpu.coarse_scores.data.data(), ref.coarse_scores.data.data(),
                         ref.coarse_scores.data.size() * 4) == 0,
         "coarse scores differ bitwise");

  // ---- exec ----
  const float scale = 1.0f / std::sqrt(static_cast<float>(c.d));
  const TensorF32 ro = sparse_attention_exec(q, k, v, ref, mask, scale);
  const TensorF32 go = b200::sparse_attention_exec(q, k, v, gpu, gq, gk, gmask, scale);
  double num = 0, den = 0, mx = 0;
  for (std::size_t i = 0; i < ro.data.size(); ++i) {
    const double e = static_cast<double>(go.data[i]) - ro.data[i];
    num += e * e;
    den += static_cast<double>(ro.data[i]) * ro.data[i];
    mx = std::fmax(mx, std::fabs(e));
  }
  const double rel = std::sqrt(num / std::fmax(den, 1e-30));
  std::printf("  exec rel_l2 %.3e max_abs %.3e\n", rel, mx);
  EXPECT(rel <= 5e-3 && mx <= 2e-2, "exec outside tolerance (rel %.3e, max %.3e)", rel, mx);

  // row range: rows outside [row_begin, row_end) are zero (P/tests/test_sparse.cpp:310-325)
  const std::size_t rb = gq.token_count() / 4, re = gq.token_count() / 2;
  const TensorF32 gpart = b200::sparse_attention_exec(q, k, v, gpu, gq, gk, gmask, scale, rb, re);
  bool zeros = true, same = true;
  for (std::size_t i = 0; i < gq.token_count(); ++i)
    for (std::size_t j = 0; j < c.d; ++j) {
      const float x = gpart.data[i * c.d + j];
      if (i < rb || i >= re) zeros = zeros && x == 0.0f;
      else same = same && x == go.data[i * c.d + j];
    }
  EXPECT(zeros && same, "row range contract violated");

  // ---- report ----
  const SparsityReport rr = sparsity_report(ref, mask);
  const SparsityReport gr = b200::sparsity_report(gpu, gq, gk, gmask);
  EXPECT(rr.executed_flops == gr.executed_flops && rr.dense_flops == gr.dense_flops && rr.density == gr.density,
         "sparsity report differs (%llu/%llu vs %llu/%llu)", (unsigned long long)gr.executed_flops,
         (unsigned long long)gr.dense_flops, (unsigned long long)rr.executed_flops,
         (unsigned long long)rr.dense_flops);
}

void degenerate_case() {
  std::printf("case degenerate_row\n");
  const TokenGrid g(std::vector<int>{0, 1}, 8, 8);
  Rng rng(7);
  const TensorF32 q = gaussian_bf16(g.token_count(), 64, rng);
  const TensorF32 k = gaussian_bf16(g.token_count(), 64, rng);
  MaskMatrix mask = MaskMatrix::all_allowed(g.token_count(), g.token_count());
  for (std::size_t j = 0; j < g.token_count(); ++j) mask.set(5, j, false);  // row 5 sees nothing
  const b200::GpuMask gm = b200::GpuMask::from(mask);
  const SparsePlan plan = b200::plan_sparse(q, k, g, g, gm, 1);
  bool ref_threw = false, gpu_threw = false;
  try {
    sparse_attention_exec(q, k, k, plan_sparse(q, k, partition_blocks(g), partition_blocks(g), mask, 1), mask,
                          0.125f);
  } catch (const DegenerateRowError&) {
    ref_threw = true;
  }
  try {
    b200::sparse_attention_exec(q, k, k, plan, g, g, gm, 0.125f);
  } catch (const DegenerateRowError&) {
    gpu_threw = true;
  }
  EXPECT(ref_threw && gpu_threw, "DegenerateRowError not raised by both (ref %d gpu %d)", ref_threw, gpu_threw);
  bool cfg = false;
  try {
    b200::plan_sparse(q, k, g, g, gm, 0);
  } catch (const ConfigError&) {
    cfg = true;
  }
  EXPECT(cfg, "topk = 0 must raise ConfigError");
}

}  // namespace

int main() {
  const std::vector<Case> cases = {
      {"tiny_stream_step_d64", 2510, 64, {1}, {0, 1}, 16, 16, 0, 0, 0, 2},
      {"self_2x16x16_d64", 2510, 64, {0, 1}, {0, 1}, 16, 16, 0, 0, 0, 2},
      {"stream_w4_d128", 401, 128, {9}, {5, 6, 7, 8, 9}, 24, 40, 0, 0, 0, 5},
      {"odd_oldest_d128", 402, 128, {10}, {7, 8, 9, 10}, 16, 24, 0, 0, 0, 3},
      {"two_frame_q_d64", 403, 64, {4, 5}, {2, 3, 4, 5}, 16, 32, 0, 0, 0, 4},
      {"ragged_locality_trunc", 404, 64, {3}, {1, 2, 3}, 20, 28, 1, 9, 11, 3},
      {"ragged_locality_pres", 405, 128, {3}, {1, 2, 3}, 20, 28, 2, 9, 11, 3},
      {"locality_bits", 406, 64, {6}, {4, 5, 6}, 24, 32, 3, 12, 16, 4},
      {"saturated", 407, 64, {3}, {1, 2, 3}, 16, 24, 0, 0, 0, 1000},
  };
  for (const Case& c : cases) {
    try {
      run_case(c);
    } catch (const std::exception& e) {
      std::printf("  FAIL: exception %s\n", e.what());
      ++failures;
    }
  }
  try {
    degenerate_case();
  } catch (const std::exception& e) {
    std::printf("  FAIL: exception %s\n", e.what());
    ++failures;
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}

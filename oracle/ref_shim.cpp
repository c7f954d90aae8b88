// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference sources (compiled read-only
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It
// lets tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg drive
// the reference hot path through ctypes:
//   vsr::partition_blocks        P/src/partition.cpp:38-62
//   vsr::build_locality_mask     P/src/mask.cpp:109-147
//   vsr::plan_sparse             P/src/sparse.cpp:72-133
//   vsr::sparse_attention_exec   P/src/sparse.cpp:208-254
//   vsr::sparsity_report         P/src/sparse.cpp:256-285
//   vsr::dense_attention_oracle  P/src/attention.cpp:40-56
//   vsr::Rng::gaussian           P/include/vsr/rng.hpp:34-48
//   vsr::build_segment_mask      P/src/mask.cpp:67-84
//   vsr::build_causal_mask       P/src/mask.cpp:86-101
//   vsr::apply_rope              P/src/rope.cpp:30-62
//   vsr::frame_attention_mass    P/src/kv_cache.cpp:170-206
//   vsr::KVCache::evict          P/src/kv_cache.cpp:97-137
// (P = /root/reference/proj).  The shim only marshals arrays and maps the
// reference exception taxonomy (P/include/vsr/common.hpp:10-48) to ints.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "vsr/attention.hpp"
#include "vsr/kv_cache.hpp"
#include "vsr/rope.hpp"
#include "vsr/grid.hpp"
#include "vsr/mask.hpp"
#include "vsr/partition.hpp"
#include "vsr/rng.hpp"
#include "vsr/sparse.hpp"
#include "vsr/tensor.hpp"

namespace {

enum : int {
  kOk = 0,
  kShape = 1,
  kConfig = 2,
  kDegenerate = 3,
  kEmptyBlock = 4,
  kInvariant = 5,
  kOther = 9,
};

void put_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg, static_cast<std::size_t>(errlen - 1));
    err[errlen - 1] = 0;
  }
}

template <typename F>
int guarded(char* err, int errlen, F&& fn) {
  try {
    fn();
    return kOk;
  } catch (const vsr::ShapeError& e) {
    put_err(err, errlen, e.what());
    return kShape;
  } catch (const vsr::ConfigError& e) {
    put_err(err, errlen, e.what());
    return kConfig;
  } catch (const vsr::DegenerateRowError& e) {
    put_err(err, errlen, e.what());
    return kDegenerate;
  } catch (const vsr::EmptyBlockError& e) {
    put_err(err, errlen, e.what());
    return kEmptyBlock;
  } catch (const vsr::InvariantError& e) {
    put_err(err, errlen, e.what());
    return kInvariant;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return kOther;
  }
}

}  // namespace

struct vsrref_case {
  std::unique_ptr<vsr::TokenGrid> grid_q, grid_k;
  vsr::BlockPartition part_q, part_k;
  vsr::TensorF32 q, k, v;
  vsr::MaskMatrix mask;
  vsr::SparsePlan plan;
  bool have_plan = false;
};

extern "C" {

// Fresh vsr::Rng(seed) gaussian stream, n draws, in the order
// TensorF32::gaussian consumes them (P/src/tensor.cpp:39-43).
void vsrref_gaussian(std::uint64_t seed, float* out, std::size_t n) {
  vsr::Rng rng(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = rng.gaussian_f(1.0f);
}

// mask_kind: 0 all-allowed, 1 locality window, 2 caller bitmask
// ([Lq][(Lk+63)/64] uint64 words, MaskMatrix layout P/include/vsr/mask.hpp:16-59).
// mode: 0 boundary_preserved, 1 boundary_truncated (LocalityWindow::Mode).
vsrref_case* vsrref_case_new(const int* qf, int nqf, const int* kf, int nkf, int rows,
                             int cols, int d, const float* q, const float* k,
                             const float* v, int mask_kind, int mode, int eh, int ew,
                             const std::uint64_t* bits, int* status, char* err,
                             int errlen) {
  auto c = std::make_unique<vsrref_case>();
  *status = guarded(err, errlen, [&] {
    c->grid_q = std::make_unique<vsr::TokenGrid>(std::vector<int>(qf, qf + nqf),
                                                 static_cast<std::size_t>(rows),
                                                 static_cast<std::size_t>(cols));
    c->grid_k = std::make_unique<vsr::TokenGrid>(std::vector<int>(kf, kf + nkf),
                                                 static_cast<std::size_t>(rows),
                                                 static_cast<std::size_t>(cols));
    const std::size_t Lq = c->grid_q->token_count(), Lk = c->grid_k->token_count();
    const std::size_t dd = static_cast<std::size_t>(d);
    c->q = vsr::TensorF32({Lq, dd}, std::vector<float>(q, q + Lq * dd));
    c->k = vsr::TensorF32({Lk, dd}, std::vector<float>(k, k + Lk * dd));
    c->v = vsr::TensorF32({Lk, dd}, std::vector<float>(v, v + Lk * dd));
    c->part_q = vsr::partition_blocks(*c->grid_q);
    c->part_k = vsr::partition_blocks(*c->grid_k);
    if (mask_kind == 0) {
      c->mask = vsr::MaskMatrix::all_allowed(Lq, Lk);
    } else if (mask_kind == 1) {
      vsr::LocalityWindow win;
      win.mode = mode == 0 ? vsr::LocalityWindow::Mode::boundary_preserved
                           : vsr::LocalityWindow::Mode::boundary_truncated;
      win.extent_h = eh;
      win.extent_w = ew;
      win.frame_extent_h = rows;
      win.frame_extent_w = cols;
      c->mask = vsr::build_locality_mask(win, c->grid_q->positions(),
                                         c->grid_k->positions());
    } else {
      c->mask = vsr::MaskMatrix(Lq, Lk, false);
      const std::size_t wpr = c->mask.words_per_row();
      for (std::size_t i = 0; i < Lq; ++i)
        std::memcpy(c->mask.row_words(i), bits + i * wpr, wpr * sizeof(std::uint64_t));
    }
  });
  if (*status != kOk) return nullptr;
  return c.release();
}

void vsrref_case_free(vsrref_case* c) { delete c; }

void vsrref_case_dims(const vsrref_case* c, int* lq, int* lk, int* bnq, int* bnk,
                      int* words_per_row) {
  *lq = static_cast<int>(c->grid_q->token_count());
  *lk = static_cast<int>(c->grid_k->token_count());
  *bnq = static_cast<int>(c->part_q.block_num);
  *bnk = static_cast<int>(c->part_k.block_num);
  *words_per_row = static_cast<int>(c->mask.words_per_row());
}

// Token-mask bits as the reference materialized them (for the GPU bitmask path).
void vsrref_mask_bits(const vsrref_case* c, std::uint64_t* out) {
  const std::size_t wpr = c->mask.words_per_row();
  for (std::size_t i = 0; i < c->mask.rows(); ++i)
    std::memcpy(out + i * wpr, c->mask.row_words(i), wpr * sizeof(std::uint64_t));
}

int vsrref_plan(vsrref_case* c, long topk, char* err, int errlen) {
  c->have_plan = false;
  const int st = guarded(err, errlen, [&] {
    c->plan = vsr::plan_sparse(c->q, c->k, c->part_q, c->part_k, c->mask,
                               static_cast<std::size_t>(topk));
  });
  c->have_plan = st == kOk;
  return st;
}

// sel: [bnq][cap] ascending ids, -1 padded; coarse: [bnq][bnk]; allowed: [bnq][bnk].
int vsrref_plan_get(const vsrref_case* c, int cap, int* sel, int* sel_count, int* diag,
                    float* coarse, std::uint8_t* allowed) {
  if (!c->have_plan) return kInvariant;
  const std::size_t bnq = c->part_q.block_num, bnk = c->part_k.block_num;
  for (std::size_t qb = 0; qb < bnq; ++qb) {
    const auto& s = c->plan.selected[qb];
    if (static_cast<int>(s.size()) > cap) return kShape;
    sel_count[qb] = static_cast<int>(s.size());
    diag[qb] = c->plan.diagonal_block[qb];
    for (int i = 0; i < cap; ++i)
      sel[qb * static_cast<std::size_t>(cap) + i] =
          i < static_cast<int>(s.size()) ? s[static_cast<std::size_t>(i)] : -1;
    for (std::size_t kb = 0; kb < bnk; ++kb) {
      if (coarse) coarse[qb * bnk + kb] = c->plan.coarse_scores.at(qb, kb);
      if (allowed) allowed[qb * bnk + kb] = c->plan.coarse_allowed.allowed(qb, kb) ? 1 : 0;
    }
  }
  return kOk;
}

// Overwrite the selection lists (negative controls such as the degenerate-row
// case of P/tests/test_sparse.cpp:327-342 edit plan.selected directly).
int vsrref_plan_set_selection(vsrref_case* c, int cap, const int* sel,
                              const int* sel_count) {
  if (!c->have_plan) return kInvariant;
  for (std::size_t qb = 0; qb < c->part_q.block_num; ++qb) {
    auto& s = c->plan.selected[qb];
    s.assign(sel + qb * static_cast<std::size_t>(cap),
             sel + qb * static_cast<std::size_t>(cap) + sel_count[qb]);
  }
  return kOk;
}

int vsrref_exec(const vsrref_case* c, float scale, long row_begin, long row_end,
                unsigned threads, float* out, char* err, int errlen) {
  if (!c->have_plan) return kInvariant;
  return guarded(err, errlen, [&] {
    const std::size_t rb = static_cast<std::size_t>(row_begin);
    const std::size_t re = row_end < 0 ? SIZE_MAX : static_cast<std::size_t>(row_end);
    vsr::TensorF32 o =
        vsr::sparse_attention_exec(c->q, c->k, c->v, c->plan, c->mask, scale, rb, re, threads);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

int vsrref_report(const vsrref_case* c, double* density, std::uint64_t* executed_flops,
                  std::uint64_t* dense_flops, char* err, int errlen) {
  if (!c->have_plan) return kInvariant;
  return guarded(err, errlen, [&] {
    const vsr::SparsityReport r = vsr::sparsity_report(c->plan, c->mask);
    *density = r.density;
    *executed_flops = r.executed_flops;
    *dense_flops = r.dense_flops;
  });
}

int vsrref_dense(const vsrref_case* c, float scale, float* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    vsr::TensorF32 o = vsr::dense_attention_oracle(c->q, c->k, c->v, c->mask, scale);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

// dense_attention_stream (P/src/attention.cpp:58-99), the reference's dense baseline, on the
// first `rows` query rows of the case (timed CPU sample for the dense-causal comparison).
int vsrref_dense_stream(const vsrref_case* c, float scale, long rows, float* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const std::size_t m = std::min<std::size_t>(static_cast<std::size_t>(rows), c->q.shape[0]);
    const std::size_t d = c->q.shape[1];
    vsr::TensorF32 qs({m, d}, std::vector<float>(c->q.data.begin(), c->q.data.begin() + m * d));
    vsr::MaskMatrix ms(m, c->mask.cols(), false);
    for (std::size_t i = 0; i < m; ++i)
      std::memcpy(ms.row_words(i), c->mask.row_words(i), ms.words_per_row() * sizeof(std::uint64_t));
    vsr::TensorF32 o = vsr::dense_attention_stream(qs, c->k, c->v, ms, scale);
    if (out) std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

// One head of the reference streaming hot path as head_attention runs it
// (P/src/stream.cpp:175-194): partitions, mask, plan_sparse, sparse_attention_exec.
// Used only as the timed CPU baseline.  Returns the executed plan's density.
int vsrref_head_attention(vsrref_case* c, long topk, float scale, unsigned threads,
                          int mask_kind, int mode, int eh, int ew, float* out, char* err,
                          int errlen) {
  return guarded(err, errlen, [&] {
    const vsr::BlockPartition pq = vsr::partition_blocks(*c->grid_q);
    const vsr::BlockPartition pk = vsr::partition_blocks(*c->grid_k);
    vsr::MaskMatrix mask;
    if (mask_kind == 1) {
      vsr::LocalityWindow win;
      win.mode = mode == 0 ? vsr::LocalityWindow::Mode::boundary_preserved
                           : vsr::LocalityWindow::Mode::boundary_truncated;
      win.extent_h = eh;
      win.extent_w = ew;
      win.frame_extent_h = static_cast<int>(c->grid_q->rows());
      win.frame_extent_w = static_cast<int>(c->grid_q->cols());
      mask = vsr::build_locality_mask(win, c->grid_q->positions(), c->grid_k->positions());
    } else {
      mask = vsr::MaskMatrix::all_allowed(c->grid_q->token_count(), c->grid_k->token_count());
    }
    vsr::SparsePlan plan =
        vsr::plan_sparse(c->q, c->k, pq, pk, mask, static_cast<std::size_t>(topk));
    vsr::TensorF32 o =
        vsr::sparse_attention_exec(c->q, c->k, c->v, plan, mask, scale, 0, SIZE_MAX, threads);
    if (out) std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

// apply_rope over a TokenGrid's positions (x: [frames*rows*cols][d] fp32, in place).
// axis_split NULL -> RopeConfig::split_default(d).
int vsrref_apply_rope(const int* fids, int nf, int rows, int cols, int d, double theta0,
                      const int* axis_split, float* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const vsr::TokenGrid g(std::vector<int>(fids, fids + nf), static_cast<std::size_t>(rows),
                           static_cast<std::size_t>(cols));
    vsr::RopeConfig rc = vsr::RopeConfig::split_default(d);
    if (axis_split) rc.axis_split = {axis_split[0], axis_split[1], axis_split[2]};
    rc.theta0 = theta0;
    const std::size_t L = g.token_count();
    vsr::TensorF32 t({L, static_cast<std::size_t>(d)},
                     std::vector<float>(x, x + L * static_cast<std::size_t>(d)));
    const vsr::TensorF32 o = vsr::apply_rope(t, g.positions(), rc);
    std::memcpy(x, o.data.data(), o.data.size() * sizeof(float));
  });
}

// Token masks from the reference builders, as MaskMatrix words [L][(L+63)/64].
int vsrref_segment_mask(const int* seg, long L, std::uint64_t* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    vsr::SegmentLabels lab;
    lab.seg.assign(seg, seg + L);
    const vsr::MaskMatrix m = vsr::build_segment_mask(lab);
    const std::size_t wpr = m.words_per_row();
    for (std::size_t i = 0; i < m.rows(); ++i) std::memcpy(out + i * wpr, m.row_words(i), wpr * 8);
  });
}

int vsrref_causal_mask(const int* frame, long L, int lookahead, std::uint64_t* out, char* err,
                       int errlen) {
  return guarded(err, errlen, [&] {
    vsr::CausalSpec spec;
    spec.frame.assign(frame, frame + L);
    spec.lookahead = lookahead;
    const vsr::MaskMatrix m = vsr::build_causal_mask(spec, static_cast<std::size_t>(L));
    const std::size_t wpr = m.words_per_row();
    for (std::size_t i = 0; i < m.rows(); ++i) std::memcpy(out + i * wpr, m.row_words(i), wpr * 8);
  });
}

// Per-frame attention mass of the current plan over the key grid (ascending frame ids).
int vsrref_frame_mass(const vsrref_case* c, double* out, char* err, int errlen) {
  if (!c->have_plan) return kInvariant;
  return guarded(err, errlen, [&] {
    const std::vector<double> m = vsr::frame_attention_mass(c->plan, *c->grid_k);
    std::memcpy(out, m.data(), m.size() * sizeof(double));
  });
}

// One KVCache layer: every head holds frames ids[0..n), then evict(layer, scores) with
// strategy 0 sliding / 1 uniform / 2 head_wise.  scores: [heads][n] (NULL -> {}).
// out_ids: [heads][n] retained ids, out_n: [heads] retained counts.
int vsrref_kv_evict(int strategy, int heads, int window, int n, const int* ids,
                    const double* scores, int* out_ids, int* out_n, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const vsr::EvictStrategy st = strategy == 0 ? vsr::EvictStrategy::sliding_window
                                  : strategy == 1 ? vsr::EvictStrategy::uniform
                                                  : vsr::EvictStrategy::head_wise;
    vsr::KVCache cache(1, static_cast<std::size_t>(heads), static_cast<std::size_t>(window), st);
    for (int h = 0; h < heads; ++h)
      for (int i = 0; i < n; ++i)
        cache.append(0, static_cast<std::size_t>(h), ids[i], vsr::TensorF32({1, 1}),
                     vsr::TensorF32({1, 1}));
    std::vector<std::vector<double>> sc;
    if (scores)
      for (int h = 0; h < heads; ++h)
        sc.emplace_back(scores + static_cast<std::size_t>(h) * n,
                        scores + static_cast<std::size_t>(h + 1) * n);
    cache.evict(0, sc);
    for (int h = 0; h < heads; ++h) {
      const std::vector<int> r = cache.frame_ids(0, static_cast<std::size_t>(h));
      out_n[h] = static_cast<int>(r.size());
      std::memcpy(out_ids + static_cast<std::size_t>(h) * n, r.data(), r.size() * sizeof(int));
    }
  });
}

}  // extern "C"

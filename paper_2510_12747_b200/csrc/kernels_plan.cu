// kernels_plan.cu — mask builder (plan_sparse) and data-movement kernels for sm_100a.
//
//   pack_frames_kernel   flat [heads][L][d] bf16  ->  swizzled frame-tiles (fvsr_common.cuh)
//   pool_partials_kernel exact sequential fp32 block sums per frame-tile      (HBM-bound)
//   score_select_kernel  coarse scores, coarse-allowed, top-k with forced diagonal
//   sparsity_count_kernel executed / dense token pairs, selected / allowed block pairs
//
// Bit-exactness of the plan (P = /root/reference/proj):
//   * avg_pool_blocks (P/src/tensor.cpp:161-186) sums member rows into a zeroed row in
//     ascending token order, then multiplies by (1.0f / count).  A block's members in
//     token order are frame 2m's tile (row-major) then frame 2m+1's tile, so we keep per
//     frame-tile partial sums S0 (from 0) and, for the second frame of a t_row, S1 (the
//     same sequence continued from the first frame's S0).  Every add is __fadd_rn in
//     that exact order; the scale is __fmul_rn by __fdiv_rn(1, count).
//   * matmul (P/src/tensor.cpp:121-151) accumulates each coarse score over channels in
//     ascending order from 0.0f with separate multiply and add: __fmul_rn / __fadd_rn,
//     one thread per (q-block, k-block) pair, then __fmul_rn by 1/sqrt(d) (sparse.cpp:97-99).
//   * selection (sparse.cpp:103-130): candidates ordered by (score desc, id asc) — we
//     bitonic-sort 64-bit keys (orderable(score) << 32 | ~id) with -0.0 canonicalised to
//     +0.0 (they compare equal in the reference), force the diagonal block first, fill to
//     k, emit ascending ids.
#include "fvsr_common.cuh"

namespace fvsr {

struct SlotList {
  int s[kMaxFrames];
};

// ---------------------------------------------------------------------------------------
// pack: one CTA per (tile, frame, head).  Source row for tile row r is spatial
// (8*th + r/8, 8*tw + r%8); rows outside the frame are zero.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) pack_frames_kernel(const uint16_t* __restrict__ src,
                                                          long long src_head_stride,  // elements
                                                          int rows, int cols, int tiles_w, int n_tiles,
                                                          int d, uint8_t* __restrict__ dst,
                                                          long long dst_head_stride,  // bytes
                                                          SlotList slots) {
  const int tile = blockIdx.x, f = blockIdx.y, head = blockIdx.z;
  const int th = tile / tiles_w, tw = tile % tiles_w;
  const int chunks_per_row = d >> 3;  // 16-byte chunks
  const long long N = (long long)rows * cols;
  const uint16_t* s = src + head * src_head_stride + (long long)f * N * d;
  const uint32_t tile_bytes = (uint32_t)d * 128u;
  uint8_t* t = dst + head * dst_head_stride + ((long long)slots.s[f] * n_tiles + tile) * tile_bytes;
  for (int idx = threadIdx.x; idx < 64 * chunks_per_row; idx += blockDim.x) {
    const int r = idx / chunks_per_row, ch = idx % chunks_per_row;
    const int h = 8 * th + (r >> 3), w = 8 * tw + (r & 7);
    uint4 val = make_uint4(0, 0, 0, 0);
    if (h < rows && w < cols) val = *reinterpret_cast<const uint4*>(s + ((long long)h * cols + w) * d + ch * 8);
    *reinterpret_cast<uint4*>(t + tile_byte_offset(r, ch * 8)) = val;
  }
}

// ---------------------------------------------------------------------------------------
// pooled partial sums.  One CTA per (tile, t_row group, head); thread c owns channel c.
// Group g covers source frames [first, first+count) (count 1 or 2, consecutive frames of
// one temporal row).  Outputs are indexed by the frames' storage slots:
//   s0[slot][tile][c] = sum from 0.0f over the frame's tile rows (ascending)
//   s1[slot][tile][c] = the first frame's S0 continued over the second frame's rows
//                       (count 2), or ext_s0 continued (count 1 with a partner)
// ---------------------------------------------------------------------------------------
struct PoolGroups {
  int first[kMaxFrames];
  int count[kMaxFrames];
  int ext_slot[kMaxFrames];  // count==1: slot of the partner frame's S0 in ext_s0, or -1
};

__global__ void __launch_bounds__(256) pool_partials_kernel(const uint16_t* __restrict__ src,
                                                            long long src_head_stride, int rows, int cols,
                                                            int tiles_w, int n_tiles, int d, PoolGroups groups,
                                                            SlotList slots, float* __restrict__ s0,
                                                            float* __restrict__ s1,
                                                            long long part_head_stride,  // elements
                                                            const float* __restrict__ ext_s0) {
  const int tile = blockIdx.x, grp = blockIdx.y, head = blockIdx.z;
  const int th = tile / tiles_w, tw = tile % tiles_w;
  const int hc = min(8, rows - 8 * th), wc = min(8, cols - 8 * tw);
  const long long N = (long long)rows * cols;
  float* S0 = s0 + head * part_head_stride;
  float* S1 = s1 + head * part_head_stride;
  const int f0 = groups.first[grp], cnt = groups.count[grp];
  const int es = groups.ext_slot[grp];

  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const uint16_t* base = src + head * src_head_stride + c;
    // Sequential fp32 sum over one frame's tile rows in ascending token order, carried
    // in two accumulators: a0 (from 0.0f) and a1 (continued from `start`).
    auto frame_sum2 = [&](int f, float& a0, float& a1, bool two) {
      const uint16_t* fb = base + (long long)f * N * d;
#pragma unroll 1
      for (int rh = 0; rh < hc; ++rh) {
        const uint16_t* rowp = fb + ((long long)(8 * th + rh) * cols + 8 * tw) * d;
        float v[8];
#pragma unroll
        for (int rw = 0; rw < 8; ++rw)
          v[rw] = rw < wc ? __uint_as_float((uint32_t)rowp[(long long)rw * d] << 16) : 0.0f;
#pragma unroll
        for (int rw = 0; rw < 8; ++rw)
          if (rw < wc) {
            a0 = __fadd_rn(a0, v[rw]);
            if (two) a1 = __fadd_rn(a1, v[rw]);
          }
      }
    };
    const long long o = (long long)tile * d + c;
    if (cnt == 2) {
      float a = 0.0f, unused = 0.0f;
      frame_sum2(f0, a, unused, false);
      S0[(long long)slots.s[f0] * n_tiles * d + o] = a;
      float b0 = 0.0f, b1 = a;
      frame_sum2(f0 + 1, b0, b1, true);
      S0[(long long)slots.s[f0 + 1] * n_tiles * d + o] = b0;
      S1[(long long)slots.s[f0 + 1] * n_tiles * d + o] = b1;
    } else {
      const bool ext = es >= 0 && ext_s0 != nullptr;
      float a0 = 0.0f;
      float a1 = ext ? ext_s0[head * part_head_stride + (long long)es * n_tiles * d + o] : 0.0f;
      frame_sum2(f0, a0, a1, ext);
      S0[(long long)slots.s[f0] * n_tiles * d + o] = a0;
      if (ext) S1[(long long)slots.s[f0] * n_tiles * d + o] = a1;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Coarse-allowed predicate for a (q-block, k-block) pair: "some token pair is allowed"
// (coarse_allowed_mask, P/src/sparse.cpp:47-70).
// ---------------------------------------------------------------------------------------
__device__ inline bool bitmask_pair_any(const DevGeom& g, const DevMask& m, int qtr, int qtile, int ktr,
                                        int ktile, bool count_mode, unsigned long long* count) {
  const int qh0 = 8 * (qtile / g.tiles_w), qw0 = 8 * (qtile % g.tiles_w);
  const int kh0 = 8 * (ktile / g.tiles_w), kw0 = 8 * (ktile % g.tiles_w);
  const int qhc = tile_h_count(g, qtile), qwc = tile_w_count(g, qtile);
  const int khc = tile_h_count(g, ktile), kwc = tile_w_count(g, ktile);
  unsigned long long n = 0;
  for (int a = 0; a < g.q_tr_count[qtr]; ++a) {
    const int fq = g.q_tr_first[qtr] + a;
    for (int r = 0; r < qhc * qwc; ++r) {
      const long long tq = g.q_frame_tok0[fq] + (long long)(qh0 + r / qwc) * g.cols + qw0 + r % qwc;
      const uint64_t* row = m.bits + tq * m.words_per_row;
      for (int b = 0; b < g.k_tr_count[ktr]; ++b) {
        const int fk = g.k_tr_first[ktr] + b;
        for (int kr = 0; kr < khc; ++kr) {
          const long long tk0 = g.k_frame_tok0[fk] + (long long)(kh0 + kr) * g.cols + kw0;
          for (int kc = 0; kc < kwc; ++kc) {
            const long long tk = tk0 + kc;
            if ((row[tk >> 6] >> (tk & 63)) & 1ull) {
              if (!count_mode) return true;
              ++n;
            }
          }
        }
      }
    }
  }
  if (count) *count = n;
  return n > 0;
}

__device__ inline bool range_overlap(int mode, int q0, int qc, int k0, int kc, int e, int F) {
  int lo0, hi0, lo1, hi1;
  locality_range(mode, q0, e, F, lo0, hi0);
  locality_range(mode, q0 + qc - 1, e, F, lo1, hi1);
  // windows slide monotonically with the query coordinate, so their union is [lo0, hi1)
  return lo0 < k0 + kc && k0 < hi1;
}

__device__ inline bool coarse_allowed(const DevGeom& g, const DevMask& m, int qtr, int qtile, int ktr, int ktile) {
  if (m.kind == 0) return true;
  if (m.kind == 1) {
    const int qh0 = 8 * (qtile / g.tiles_w), qw0 = 8 * (qtile % g.tiles_w);
    const int kh0 = 8 * (ktile / g.tiles_w), kw0 = 8 * (ktile % g.tiles_w);
    return range_overlap(m.mode, qh0, tile_h_count(g, qtile), kh0, tile_h_count(g, ktile), m.extent_h, g.rows) &&
           range_overlap(m.mode, qw0, tile_w_count(g, qtile), kw0, tile_w_count(g, ktile), m.extent_w, g.cols);
  }
  return bitmask_pair_any(g, m, qtr, qtile, ktr, ktile, false, nullptr);
}

// number of allowed (q, k) coordinate pairs along one axis for locality
__device__ inline long long axis_pairs(int mode, int q0, int qc, int k0, int kc, int e, int F) {
  long long n = 0;
  for (int a = 0; a < qc; ++a) {
    int lo, hi;
    locality_range(mode, q0 + a, e, F, lo, hi);
    const int l = max(lo, k0), h = min(hi, k0 + kc);
    if (h > l) n += h - l;
  }
  return n;
}

__device__ inline unsigned long long pair_count(const DevGeom& g, const DevMask& m, int qtr, int qtile, int ktr,
                                                int ktile) {
  const unsigned long long fq = g.q_tr_count[qtr], fk = g.k_tr_count[ktr];
  if (m.kind == 0)
    return fq * fk * (unsigned long long)(tile_h_count(g, qtile) * tile_w_count(g, qtile)) *
           (unsigned long long)(tile_h_count(g, ktile) * tile_w_count(g, ktile));
  if (m.kind == 1) {
    const int qh0 = 8 * (qtile / g.tiles_w), qw0 = 8 * (qtile % g.tiles_w);
    const int kh0 = 8 * (ktile / g.tiles_w), kw0 = 8 * (ktile % g.tiles_w);
    return fq * fk *
           (unsigned long long)axis_pairs(m.mode, qh0, tile_h_count(g, qtile), kh0, tile_h_count(g, ktile),
                                          m.extent_h, g.rows) *
           (unsigned long long)axis_pairs(m.mode, qw0, tile_w_count(g, qtile), kw0, tile_w_count(g, ktile),
                                          m.extent_w, g.cols);
  }
  unsigned long long n = 0;
  bitmask_pair_any(g, m, qtr, qtile, ktr, ktile, true, &n);
  return n;
}

// ---------------------------------------------------------------------------------------
// score + select.  One CTA (256 threads) per (q-block, head).
// ---------------------------------------------------------------------------------------
__device__ inline uint64_t order_key(float s, int kb) {
  uint32_t u = __float_as_uint(s == 0.0f ? 0.0f : s);  // -0.0 ties with +0.0
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((uint64_t)u << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)kb);
}

struct SelectParams {
  const float* q_s0;
  const float* q_s1;
  long long q_head_stride;  // elements, indexed [nqf][n_tiles][d]
  const float* k_s0;
  const float* k_s1;
  long long k_head_stride;  // elements, indexed [slot][n_tiles][d]
  float scale;
  long long topk;
  int cap;
  int npow2;
  int* sel;
  int* sel_count;
  int* diag;
  float* coarse;
  uint8_t* allowed;
  unsigned* err;
};

__global__ void __launch_bounds__(256) score_select_kernel(DevGeom g, DevMask m, SelectParams p) {
  extern __shared__ __align__(16) uint8_t sm_raw[];
  const int qb = blockIdx.x, head = blockIdx.y;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int d = g.d;
  uint64_t* keys = reinterpret_cast<uint64_t*>(sm_raw);              // [npow2]
  float* pq = reinterpret_cast<float*>(keys + p.npow2);              // [d]
  uint8_t* allow_f = reinterpret_cast<uint8_t*>(pq + d);             // [bnk]
  uint8_t* sel_f = allow_f + g.bnk;                                  // [bnk]
  __shared__ int s_nallowed;
  __shared__ int s_warp[8];
  __shared__ int s_running;
  __shared__ unsigned s_err;
  if (tid == 0) { s_nallowed = 0; s_running = 0; s_err = 0; }

  const int qtr = qb / g.n_tiles, qtile = qb % g.n_tiles;
  const int qcnt = g.q_tr_count[qtr];
  const int qf = g.q_tr_first[qtr] + qcnt - 1;
  const float* qsrc = (qcnt == 2 ? p.q_s1 : p.q_s0) + head * p.q_head_stride + ((long long)qf * g.n_tiles + qtile) * d;
  const float inv_q = __fdiv_rn(1.0f, (float)(qcnt * tile_h_count(g, qtile) * tile_w_count(g, qtile)));
  for (int c = tid; c < d; c += nthr) {
    const float v = __fmul_rn(qsrc[c], inv_q);
    if (!isfinite(v)) s_err = kErrShape;
    pq[c] = v;
  }
  __syncthreads();

  int local_allowed = 0;
  for (int kb = tid; kb < p.npow2; kb += nthr) {
    if (kb >= g.bnk) { keys[kb] = 0; continue; }
    const int ktr = kb / g.n_tiles, ktile = kb % g.n_tiles;
    const int kcnt = g.k_tr_count[ktr];
    const int kf = g.k_tr_first[ktr] + kcnt - 1;
    const float* ksrc = (kcnt == 2 ? p.k_s1 : p.k_s0) + head * p.k_head_stride +
                        ((long long)g.k_slot[kf] * g.n_tiles + ktile) * d;
    const float inv_k = __fdiv_rn(1.0f, (float)(kcnt * tile_h_count(g, ktile) * tile_w_count(g, ktile)));
    float dot = 0.0f;
    bool fin = true;
    for (int c = 0; c < d; ++c) {
      const float pk = __fmul_rn(ksrc[c], inv_k);
      fin = fin && isfinite(pk);
      dot = __fadd_rn(dot, __fmul_rn(pq[c], pk));
    }
    if (!fin) s_err = kErrShape;
    const float s = __fmul_rn(dot, p.scale);
    const bool al = coarse_allowed(g, m, qtr, qtile, ktr, ktile);
    const long long o = ((long long)head * g.bnq + qb) * g.bnk + kb;
    if (p.coarse) p.coarse[o] = s;
    if (p.allowed) p.allowed[o] = al ? 1 : 0;
    allow_f[kb] = al ? 1 : 0;
    sel_f[kb] = 0;
    keys[kb] = al ? order_key(s, kb) : 0ull;
    local_allowed += al ? 1 : 0;
  }
  if (local_allowed) atomicAdd(&s_nallowed, local_allowed);
  __syncthreads();

  // bitonic sort, descending
  for (int k = 2; k <= p.npow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < p.npow2; i += nthr) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = keys[i], b = keys[ixj];
          const bool desc = (i & k) == 0;
          if (desc ? (a < b) : (a > b)) { keys[i] = b; keys[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }

  // selection: diagonal first (if coarse-allowed), then best-first skipping it
  int dg = -1;
  if (g.q_tr_diag[qtr] >= 0) dg = g.q_tr_diag[qtr] * g.n_tiles + qtile;
  if (dg >= 0 && !allow_f[dg]) dg = -1;
  if (tid == 0) {
    long long cnt = 0;
    if (dg >= 0) { sel_f[dg] = 1; cnt = 1; }
    for (int i = 0; i < s_nallowed && cnt < p.topk; ++i) {
      const int id = (int)(0xFFFFFFFFu - (uint32_t)(keys[i] & 0xFFFFFFFFull));
      if (id != dg) { sel_f[id] = 1; ++cnt; }
    }
  }
  __syncthreads();

  // ordered compaction of sel_f -> ascending ids
  int* out = p.sel + ((long long)head * g.bnq + qb) * p.cap;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  for (int base = 0; base < g.bnk; base += nthr) {
    const int kb = base + tid;
    const bool f = kb < g.bnk && sel_f[kb];
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    int before = s_running;
    for (int w = 0; w < warp; ++w) before += s_warp[w];
    if (f) {
      const int pos = before + __popc(bal & ((1u << lane) - 1u));
      if (pos < p.cap) out[pos] = kb;
    }
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < nwarps; ++w) tot += s_warp[w];
      s_running += tot;
    }
    __syncthreads();
  }
  const int total = s_running;
  for (int i = total + tid; i < p.cap; i += nthr) out[i] = -1;
  if (tid == 0) {
    p.sel_count[(long long)head * g.bnq + qb] = total;
    if (p.diag) p.diag[(long long)head * g.bnq + qb] = dg;
    if (total > p.cap) atomicOr(p.err, kErrInvariant);
    if (s_err) atomicOr(p.err, s_err);
  }
}

// ---------------------------------------------------------------------------------------
// sparsity accounting (sparsity_report, P/src/sparse.cpp:256-285): one CTA per (q-block, head)
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) sparsity_count_kernel(DevGeom g, DevMask m, const int* __restrict__ sel,
                                                             const int* __restrict__ sel_count, int cap,
                                                             unsigned long long* executed,
                                                             unsigned long long* dense,
                                                             unsigned long long* nselected,
                                                             unsigned long long* nallowed) {
  const int qb = blockIdx.x, head = blockIdx.y;
  const int qtr = qb / g.n_tiles, qtile = qb % g.n_tiles;
  unsigned long long ex = 0, dn = 0, na = 0;
  for (int kb = threadIdx.x; kb < g.bnk; kb += blockDim.x) {
    const int ktr = kb / g.n_tiles, ktile = kb % g.n_tiles;
    const unsigned long long pc = pair_count(g, m, qtr, qtile, ktr, ktile);
    dn += pc;
    na += pc > 0 ? 1 : 0;
  }
  const int n = sel_count[(long long)head * g.bnq + qb];
  const int* s = sel + ((long long)head * g.bnq + qb) * cap;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int kb = s[i];
    ex += pair_count(g, m, qtr, qtile, kb / g.n_tiles, kb % g.n_tiles);
  }
  for (int o = 16; o > 0; o >>= 1) {
    ex += __shfl_xor_sync(0xffffffffu, ex, o);
    dn += __shfl_xor_sync(0xffffffffu, dn, o);
    na += __shfl_xor_sync(0xffffffffu, na, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(executed + head, ex);
    atomicAdd(dense + head, dn);
    atomicAdd(nallowed + head, na);
  }
  if (threadIdx.x == 0) atomicAdd(nselected + head, (unsigned long long)n);
}

}  // namespace fvsr

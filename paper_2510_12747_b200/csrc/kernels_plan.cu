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
// Fused pack + pool: one pass over a frame list writes the swizzled frame-tiles and the
// exact-order partial sums (S0 / S1 as in pool_partials_kernel).  An optional second tensor
// (V) is packed alongside without pooling.  One CTA per (tile, t_row group, head); thread t
// owns channels 2t, 2t+1 (bf16x2 loads, 128 B per warp per token row).
// ---------------------------------------------------------------------------------------
struct PackPoolArgs {
  const uint16_t* src;   // pooled + packed, [heads][frames * rows * cols][d]
  const uint16_t* src2;  // packed only (may be null)
  long long src_head_stride;  // elements (both sources)
  uint8_t* dst;
  uint8_t* dst2;
  long long dst_head_stride;  // bytes
  float* s0;
  float* s1;
  long long part_head_stride;  // elements
  const float* ext_s0;         // partner S0 for single-frame groups (ring appends), may be null
  int rows, cols, tiles_w, n_tiles, d;
};

__global__ void __launch_bounds__(64) pack_pool_kernel(PackPoolArgs a, PoolGroups groups, SlotList slots) {
  const int tile = blockIdx.x, grp = blockIdx.y, head = blockIdx.z;
  const int c = 2 * threadIdx.x;
  if (c >= a.d) return;
  const int th = tile / a.tiles_w, tw = tile % a.tiles_w;
  const int hc = min(8, a.rows - 8 * th), wc = min(8, a.cols - 8 * tw);
  const long long N = (long long)a.rows * a.cols;
  const uint32_t tile_bytes = (uint32_t)a.d * 128u;
  const int f0 = groups.first[grp], cnt = groups.count[grp], es = groups.ext_slot[grp];
  const bool ext = cnt == 1 && es >= 0 && a.ext_s0 != nullptr;
  const long long po = (long long)tile * a.d + c;
  float s1x = 0.0f, s1y = 0.0f;
  if (ext) {
    const float* e = a.ext_s0 + head * a.part_head_stride + (long long)es * a.n_tiles * a.d + po;
    s1x = e[0];
    s1y = e[1];
  }
  for (int fi = 0; fi < cnt; ++fi) {
    const int f = f0 + fi, slot = slots.s[f];
    const bool cont = fi == 1 || ext;  // S1 accumulates this frame too
    const long long so = head * a.src_head_stride + (long long)f * N * a.d + c;
    const long long to = head * a.dst_head_stride + ((long long)slot * a.n_tiles + tile) * tile_bytes;
    float s0x = 0.0f, s0y = 0.0f;
    const uint16_t* __restrict__ src = a.src + so;
    const uint16_t* __restrict__ src2 = a.src2 ? a.src2 + so : nullptr;
    uint8_t* __restrict__ dst = a.dst + to;
    uint8_t* __restrict__ dst2 = a.dst2 ? a.dst2 + to : nullptr;
    constexpr int kBatch = 16;  // token rows in flight per thread
    for (int r0 = 0; r0 < 64; r0 += kBatch) {
      uint32_t v[kBatch], v2[kBatch];
#pragma unroll
      for (int i = 0; i < kBatch; ++i) {
        const int r = r0 + i;
        const bool valid = (r >> 3) < hc && (r & 7) < wc;
        const long long tok = (long long)(8 * th + (r >> 3)) * a.cols + 8 * tw + (r & 7);
        v[i] = valid ? __ldg(reinterpret_cast<const unsigned int*>(src + tok * a.d)) : 0u;
        v2[i] = (valid && src2) ? __ldg(reinterpret_cast<const unsigned int*>(src2 + tok * a.d)) : 0u;
      }
#pragma unroll
      for (int i = 0; i < kBatch; ++i) {
        const int r = r0 + i;
        const uint32_t off = tile_byte_offset(r, c);
        *reinterpret_cast<uint32_t*>(dst + off) = v[i];
        if (dst2) *reinterpret_cast<uint32_t*>(dst2 + off) = v2[i];
        if ((r >> 3) < hc && (r & 7) < wc) {
          const float x = __uint_as_float(v[i] << 16), y = __uint_as_float(v[i] & 0xffff0000u);
          s0x = __fadd_rn(s0x, x);
          s0y = __fadd_rn(s0y, y);
          if (cont) {
            s1x = __fadd_rn(s1x, x);
            s1y = __fadd_rn(s1y, y);
          }
        }
      }
    }
    float* S0 = a.s0 + head * a.part_head_stride + (long long)slot * a.n_tiles * a.d + po;
    S0[0] = s0x;
    S0[1] = s0y;
    if (cont) {
      float* S1 = a.s1 + head * a.part_head_stride + (long long)slot * a.n_tiles * a.d + po;
      S1[0] = s1x;
      S1[1] = s1y;
    }
    if (fi == 0 && cnt == 2) {  // frame B continues frame A's sequence
      s1x = s0x;
      s1y = s0y;
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

// One CTA per (head, kSelQG consecutive q-blocks), kSelThreads threads.  Pooled key rows
// are staged once per CTA in chunks of kSelChunk blocks (warp-coalesced float4 loads, row
// stride d+1 floats so column walks are conflict-free).  Each thread owns one key row of
// the chunk and kSelQG/2... interleaved q-blocks, accumulating their dot products as
// independent sequential chains (exact reference order per score, ILP across scores).
// Selection: warp w handles q-block w; top-k by exact rank counting — rank(i) =
// #{j : key_j > key_i} over 64-bit (orderable score, ~id) keys, i.e. the position in the
// reference's stable_sort(score desc, id asc) — then a ballot compaction in id order.
constexpr int kSelThreads = 256;
constexpr int kSelQG = 8;        // q-blocks per CTA (one selection warp each)
constexpr int kSelChunk = 128;   // key blocks staged per pass
constexpr int kSelQPerThr = kSelQG * kSelChunk / kSelThreads;  // 4 scores per thread per chunk

__global__ void __launch_bounds__(kSelThreads) score_select_kernel(DevGeom g, DevMask m, SelectParams p) {
  extern __shared__ __align__(16) uint8_t sm_raw[];
  const int qb0 = blockIdx.x * kSelQG, head = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = g.d, bnk = g.bnk, ld = d + 1;
  const int nq = min(kSelQG, g.bnq - qb0);
  uint64_t* keys = reinterpret_cast<uint64_t*>(sm_raw);              // [kSelQG][bnk]
  float* pq = reinterpret_cast<float*>(keys + kSelQG * bnk);         // [kSelQG][d]
  float* pk = pq + kSelQG * d;                                       // [kSelChunk][d+1]
  uint8_t* sel_f = reinterpret_cast<uint8_t*>(pk + kSelChunk * ld);  // [kSelQG][bnk]
  __shared__ unsigned s_err;
  if (tid == 0) s_err = 0;

  for (int idx = tid; idx < nq * d; idx += kSelThreads) {
    const int qq = idx / d, c = idx - qq * d;
    const int qb = qb0 + qq;
    const int qtr = qb / g.n_tiles, qtile = qb % g.n_tiles;
    const int qcnt = g.q_tr_count[qtr];
    const int qf = g.q_tr_first[qtr] + qcnt - 1;
    const float* qsrc = (qcnt == 2 ? p.q_s1 : p.q_s0) + head * p.q_head_stride + ((long long)qf * g.n_tiles + qtile) * d;
    const float inv_q = __fdiv_rn(1.0f, (float)(qcnt * tile_h_count(g, qtile) * tile_w_count(g, qtile)));
    const float v = __fmul_rn(qsrc[c], inv_q);
    if (!isfinite(v)) s_err = kErrShape;
    pq[qq * d + c] = v;
  }

  // ---- coarse scores, chunk by chunk ----------------------------------------------------
  for (int kb0 = 0; kb0 < bnk; kb0 += kSelChunk) {
    const int nk = min(kSelChunk, bnk - kb0);
    __syncthreads();  // previous chunk consumed; pq visible on the first pass
    bool fin = true;
#pragma unroll 4
    for (int r = warp; r < nk; r += kSelThreads / 32) {  // warp per pooled row
      const int kb = kb0 + r;
      const int ktr = kb / g.n_tiles, ktile = kb - ktr * g.n_tiles;
      const int kcnt = g.k_tr_count[ktr];
      const int kf = g.k_tr_first[ktr] + kcnt - 1;
      const float* row = (kcnt == 2 ? p.k_s1 : p.k_s0) + head * p.k_head_stride +
                         ((long long)g.k_slot[kf] * g.n_tiles + ktile) * d;
      const float inv_k = __fdiv_rn(1.0f, (float)(kcnt * tile_h_count(g, ktile) * tile_w_count(g, ktile)));
      for (int c4 = lane; c4 < d / 4; c4 += 32) {
        const float4 v = *reinterpret_cast<const float4*>(row + 4 * c4);
        const float a = __fmul_rn(v.x, inv_k), b = __fmul_rn(v.y, inv_k);
        const float e = __fmul_rn(v.z, inv_k), f = __fmul_rn(v.w, inv_k);
        fin = fin && isfinite(a) && isfinite(b) && isfinite(e) && isfinite(f);
        float* dst = pk + r * ld + 4 * c4;
        dst[0] = a; dst[1] = b; dst[2] = e; dst[3] = f;
      }
    }
    if (!fin) s_err = kErrShape;
    __syncthreads();
    // thread -> key row r = tid % kSelChunk, q-blocks qq = tid / kSelChunk + 2i
    const int r = tid % kSelChunk, qbase = tid / kSelChunk;
    if (r < nk) {
      const float* row = pk + r * ld;
      float acc[kSelQPerThr];
#pragma unroll
      for (int i = 0; i < kSelQPerThr; ++i) acc[i] = 0.0f;
#pragma unroll 4
      for (int c = 0; c < d; ++c) {
        const float kv = row[c];
#pragma unroll
        for (int i = 0; i < kSelQPerThr; ++i)
          acc[i] = __fadd_rn(acc[i], __fmul_rn(pq[(qbase + 2 * i) * d + c], kv));
      }
      const int kb = kb0 + r;
      const int ktr = kb / g.n_tiles, ktile = kb - ktr * g.n_tiles;
#pragma unroll
      for (int i = 0; i < kSelQPerThr; ++i) {
        const int qq = qbase + 2 * i;
        if (qq >= nq) continue;
        const int qb = qb0 + qq;
        const int qtr = qb / g.n_tiles, qtile = qb % g.n_tiles;
        const float sc = __fmul_rn(acc[i], p.scale);
        const bool al = coarse_allowed(g, m, qtr, qtile, ktr, ktile);
        const long long o = ((long long)head * g.bnq + qb) * bnk + kb;
        if (p.coarse) p.coarse[o] = sc;
        if (p.allowed) p.allowed[o] = al ? 1 : 0;
        keys[qq * bnk + kb] = al ? order_key(sc, kb) : 0ull;
      }
    }
  }
  __syncthreads();

  // ---- selection by rank, one warp per q-block: diagonal first, then the best k' others ---
  if (warp < nq) {
    const int qq = warp, qb = qb0 + qq;
    const int qtr = qb / g.n_tiles, qtile = qb % g.n_tiles;
    const uint64_t* kq = keys + qq * bnk;
    uint8_t* sf = sel_f + qq * bnk;
    int dg = -1;
    if (g.q_tr_diag[qtr] >= 0) dg = g.q_tr_diag[qtr] * g.n_tiles + qtile;
    if (dg >= 0 && kq[dg] == 0ull) dg = -1;
    const uint64_t kdg = dg >= 0 ? kq[dg] : ~0ull;
    const long long kprime = p.topk - (dg >= 0 ? 1 : 0);
    // 8 register-held candidates per lane per pass: each shared key read feeds 8 compares
    for (int i0 = 0; i0 < bnk; i0 += 32 * 8) {
      uint64_t kc[8];
      int rank[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int i = i0 + v * 32 + lane;
        kc[v] = i < bnk ? kq[i] : 0ull;
        rank[v] = 0;
      }
#pragma unroll 2
      for (int jj = 0; jj < bnk; ++jj) {
        const uint64_t kj = kq[jj];
#pragma unroll
        for (int v = 0; v < 8; ++v) rank[v] += kj > kc[v] ? 1 : 0;
      }
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int i = i0 + v * 32 + lane;
        if (i >= bnk) continue;
        bool s = false;
        if (kc[v] != 0ull) {
          if (i == dg) {
            s = true;
          } else {
            const int r = rank[v] - ((dg >= 0 && kdg > kc[v]) ? 1 : 0);  // among non-diagonal candidates
            s = r < kprime;
          }
        }
        sf[i] = s ? 1 : 0;
      }
    }
    __syncwarp();
    int* out = p.sel + ((long long)head * g.bnq + qb) * p.cap;
    int total = 0;
    for (int base = 0; base < bnk; base += 32) {
      const int kb = base + lane;
      const bool f = kb < bnk && sf[kb];
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (f) {
        const int pos = total + __popc(bal & ((1u << lane) - 1u));
        if (pos < p.cap) out[pos] = kb;
      }
      total += __popc(bal);
    }
    for (int i = total + lane; i < p.cap; i += 32) out[i] = -1;
    if (lane == 0) {
      p.sel_count[(long long)head * g.bnq + qb] = total;
      if (p.diag) p.diag[(long long)head * g.bnq + qb] = dg;
      if (total > p.cap) atomicOr(p.err, kErrInvariant);
    }
  }
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(p.err, s_err);
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

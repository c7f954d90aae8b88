// kernel_attn.cu — block-sparse streaming attention on tcgen05 / TMEM (sm_100a).
//
// Replaces exec_block_range / sparse_attention_exec (P/src/sparse.cpp:141-254,
// P = /root/reference/proj): for each query row, exact softmax attention over the keys of
// its q-block's selected key blocks, filtered by the token mask, merged across blocks
// with a running max.  Rows outside [row_begin, row_end) are zero; a row whose selected
// blocks hold no allowed key latches DegenerateRowError (sparse.cpp:198-200).
//
// Work unit: one 64-row query frame-tile (the reference's streaming q-block is one
// frame's 8x8 tile, 64 rows).  tcgen05 issues M in {64,128} and M=64 runs at half rate,
// so the kernel is TRANSPOSED: keys sit on the M=128 axis.
//     S^T[128 keys x 64 q]  = K_tile[128 x d]   . Q_tile[64 x d]^T       (K-major A, K-major B)
//     O^T[d x 64 q]        += V_tile^T[d x 128] . P^T[128 keys x 64 q]   (MN-major A, MN-major B)
// Both MMAs are M=128, N=64 — full tensor-core rate — and a key block is exactly one
// 128-row tile (frames 2m and 2m+1 of one spatial 8x8 tile; 64 rows when only one frame
// of the pair is in context, in which case PV issues only the 4 valid K=16 steps).
//
// Softmax in the transposed layout: TMEM lane j holds key j's scores for all 64 queries,
// so thread j (4 warps = 128 lanes) owns one key row.  Per-query max/sum are column
// reductions across threads; we avoid one per tile:
//   * the running reference c_q only moves when some score exceeds it by > 8 (log2
//     units, FA4-style lazy rescale); detecting that is one CTA-wide OR per tile;
//   * on the (rare) exceed path — always on the first tile — the exact column max is a
//     warp butterfly + smem across warps, followed by a rescale of O^T in TMEM and of the
//     per-thread partial sums;
//   * the denominators are per-thread partial sums (thread j sums its own key's p over
//     tiles) reduced once at the end.
//
// Roles (192 threads): warps 0-3 softmax + epilogue (TMEM lanes 0-127), warp 4 producer
// (cp.async.bulk of pre-swizzled frame-tiles), warp 5 TMEM allocator + MMA issuer.
#include "fvsr_common.cuh"

namespace fvsr {

constexpr int kNK = 3;  // K stages
constexpr int kNV = 2;  // V stages
constexpr int kNP = 2;  // P^T buffers (== S buffers)
constexpr uint32_t kTmemCols = 256;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct AttnParams {
  const uint8_t* q;         // packed q frame-tiles [heads][nqf][n_tiles]
  long long q_head_stride;  // bytes
  const uint8_t* k;         // packed k frame-tiles [heads][slots][n_tiles]
  const uint8_t* v;
  long long kv_head_stride; // bytes
  const int* sel;           // [heads][bnq][cap]
  const int* sel_count;     // [heads][bnq]
  int cap;
  uint16_t* out;            // bf16 [heads][Lq][d]
  long long out_head_stride;// elements
  long long row_begin, row_end;
  float scale_log2;         // scale * log2(e)
  long long unit_begin;
  int out_tile_major;       // 1: out is [unit - unit_begin][64][d] (head-parallel gather layout)
  unsigned* err;
  unsigned long long* pairs;// += executed (mask-allowed) token pairs, reference definition
};

template <int D>
struct AttnCfg {
  static constexpr uint32_t kTileBytes = D * 128;        // one packed frame-tile
  static constexpr uint32_t kQBytes = kTileBytes;        // 64 rows
  static constexpr uint32_t kKVBytes = 2 * kTileBytes;   // 128 rows
  static constexpr uint32_t kPBytes = 128 * 128;         // 128 keys x 64 q bf16
  static constexpr uint32_t kOffQ = 0;
  static constexpr uint32_t kOffK = kOffQ + kQBytes;
  static constexpr uint32_t kOffV = kOffK + kNK * kKVBytes;
  static constexpr uint32_t kOffP = kOffV + kNV * kKVBytes;
  static constexpr uint32_t kOffBar = kOffP + kNP * kPBytes;
  static constexpr uint32_t kScratch = 2048;                 // barriers, softmax scratch
  static constexpr uint32_t kBytes = kOffBar + kScratch + 1024;  // + alignment slack
};

// Butterfly reduce-scatter of 64 per-thread column values across a warp: step s keeps
// the half selected by lane bit (4-s), so on return v[0], v[1] hold the warp-wide
// reduction for columns 2*lane and 2*lane+1.
template <bool kMax>
__device__ __forceinline__ void warp_colreduce64(float (&v)[64], int lane) {
#pragma unroll
  for (int step = 0; step < 5; ++step) {
    const int half = 32 >> step;  // live values before this step: 2*half
    const int off = 16 >> step;
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float keep = upper ? v[half + i] : v[i];
      const float send = upper ? v[i] : v[half + i];
      const float recv = __shfl_xor_sync(0xffffffffu, send, off);
      v[i] = kMax ? fmaxf(keep, recv) : keep + recv;
    }
  }
}
__device__ __forceinline__ int colreduce_col(int lane, int i) { return (lane << 1) | i; }

template <int D>
__global__ void __launch_bounds__(192, 1) sparse_attn_kernel(DevGeom g, DevMask m, AttnParams p) {
  using Cfg = AttnCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + Cfg::kOffQ;
  uint8_t* sK = smem + Cfg::kOffK;
  uint8_t* sV = smem + Cfg::kOffV;
  uint8_t* sP = smem + Cfg::kOffP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kOffBar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + kNK;
  uint64_t* v_full = k_empty + kNK;
  uint64_t* v_empty = v_full + kNV;
  uint64_t* s_full = v_empty + kNV;
  uint64_t* s_empty = s_full + kNP;
  uint64_t* p_full = s_empty + kNP;
  uint64_t* p_empty = p_full + kNP;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_empty + kNP);
  float* c_ref = reinterpret_cast<float*>(smem + Cfg::kOffBar + 256);  // [64]
  float* alpha = c_ref + 64;                                           // [64]
  float* red = alpha + 64;                                             // [4][64]
  int* flags = reinterpret_cast<int*>(red + 256);                      // [2][4]
  int* win = flags + 8;                                                // [4][8] hlo,hhi,wlo,whi

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- unit decode --------------------------------------------------------------------
  const long long unit = p.unit_begin + blockIdx.x;
  const int tiles_per_head = g.nqf * g.n_tiles;
  const int head = (int)(unit / tiles_per_head);
  const int rem = (int)(unit % tiles_per_head);
  const int qf = rem / g.n_tiles, qtile = rem % g.n_tiles;
  const int qtr = g.q_frame_tr[qf];
  const int qb = qtr * g.n_tiles + qtile;
  const int n = min(max(p.sel_count[(long long)head * g.bnq + qb], 0), p.cap);
  const int* sel = p.sel + ((long long)head * g.bnq + qb) * p.cap;
  // Selection ids come from the caller; every role reads them through this clamp so the
  // barrier protocol stays consistent, and the producer latches InvariantError.
  auto sel_at = [&](int t) {
    const int kb = sel[t];
    return kb < 0 ? 0 : (kb >= g.bnk ? g.bnk - 1 : kb);
  };
  const int qh0 = 8 * (qtile / g.tiles_w), qw0 = 8 * (qtile % g.tiles_w);

  // ---- setup ----------------------------------------------------------------------------
  if (warp == 5) tmem_alloc(tmem_slot, kTmemCols);
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < kNK; ++i) { mbar_init(k_full + i, 1); mbar_init(k_empty + i, 1); }
    for (int i = 0; i < kNV; ++i) { mbar_init(v_full + i, 1); mbar_init(v_empty + i, 1); }
    for (int i = 0; i < kNP; ++i) {
      mbar_init(s_full + i, 1); mbar_init(s_empty + i, 4);
      mbar_init(p_full + i, 4); mbar_init(p_empty + i, 1);
    }
    fence_barrier_init();
  }
  if (threadIdx.x < 64) c_ref[threadIdx.x] = -INFINITY;
  if (threadIdx.x < 8) {
    int lo, hi;
    locality_range(m.mode, qh0 + threadIdx.x, m.extent_h, g.rows, lo, hi);
    win[threadIdx.x] = lo; win[8 + threadIdx.x] = hi;
    locality_range(m.mode, qw0 + threadIdx.x, m.extent_w, g.cols, lo, hi);
    win[16 + threadIdx.x] = lo; win[24 + threadIdx.x] = hi;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem + 0u, tmem + 64u};
  const uint32_t tO = tmem + 128u;

  if (warp == 4) {
    // ===================================== producer =====================================
    if (lane == 0 && n > 0) {
      mbar_arrive_expect_tx(q_full, Cfg::kQBytes);
      bulk_g2s(sQ, p.q + head * p.q_head_stride + ((long long)qf * g.n_tiles + qtile) * Cfg::kTileBytes,
               Cfg::kQBytes, q_full);
      for (int t = 0; t < n; ++t) {
        if (sel[t] < 0 || sel[t] >= g.bnk) atomicOr(p.err, kErrInvariant);
        const int kb = sel_at(t);
        const int ktr = kb / g.n_tiles, ktile = kb % g.n_tiles;
        const int kcnt = g.k_tr_count[ktr], f0 = g.k_tr_first[ktr];
        const uint8_t* srcA_k = p.k + head * p.kv_head_stride + ((long long)g.k_slot[f0] * g.n_tiles + ktile) * Cfg::kTileBytes;
        const uint8_t* srcA_v = p.v + head * p.kv_head_stride + ((long long)g.k_slot[f0] * g.n_tiles + ktile) * Cfg::kTileBytes;
        const uint8_t* srcB_k = nullptr;
        const uint8_t* srcB_v = nullptr;
        if (kcnt == 2) {
          srcB_k = p.k + head * p.kv_head_stride + ((long long)g.k_slot[f0 + 1] * g.n_tiles + ktile) * Cfg::kTileBytes;
          srcB_v = p.v + head * p.kv_head_stride + ((long long)g.k_slot[f0 + 1] * g.n_tiles + ktile) * Cfg::kTileBytes;
        }
        const int ks = t % kNK;
        if (t >= kNK) mbar_wait(k_empty + ks, ((t / kNK) - 1) & 1);
        mbar_arrive_expect_tx(k_full + ks, kcnt * Cfg::kTileBytes);
        uint8_t* dk = sK + ks * Cfg::kKVBytes;
#pragma unroll
        for (int s = 0; s < D / 64; ++s) {
          bulk_g2s(dk + s * 16384, srcA_k + s * kSubBytes, kSubBytes, k_full + ks);
          if (kcnt == 2) bulk_g2s(dk + s * 16384 + kSubBytes, srcB_k + s * kSubBytes, kSubBytes, k_full + ks);
        }
        const int vs = t % kNV;
        if (t >= kNV) mbar_wait(v_empty + vs, ((t / kNV) - 1) & 1);
        mbar_arrive_expect_tx(v_full + vs, kcnt * Cfg::kTileBytes);
        uint8_t* dv = sV + vs * Cfg::kKVBytes;
#pragma unroll
        for (int s = 0; s < D / 64; ++s) {
          bulk_g2s(dv + s * 16384, srcA_v + s * kSubBytes, kSubBytes, v_full + vs);
          if (kcnt == 2) bulk_g2s(dv + s * 16384 + kSubBytes, srcB_v + s * kSubBytes, kSubBytes, v_full + vs);
        }
      }
    }
  } else if (warp == 5) {
    // ===================================== MMA issuer ===================================
    if (lane == 0 && n > 0) {
      constexpr uint32_t idesc_qk = umma_idesc_bf16(128, 64, 0, 0);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(128, 64, 1, 1);
      const uint32_t aQ = smem_u32(sQ);
      auto issue_pv = [&](int u) {
        const int vs = u % kNV, pb = u & 1;
        mbar_wait(v_full + vs, (u / kNV) & 1);
        mbar_wait(p_full + pb, (u >> 1) & 1);
        tc_fence_after();
        const int kb = sel_at(u);
        const int steps = g.k_tr_count[kb / g.n_tiles] == 2 ? 8 : 4;
        const uint32_t aV = smem_u32(sV + vs * Cfg::kKVBytes);
        const uint32_t aP = smem_u32(sP + pb * Cfg::kPBytes);
        for (int kk = 0; kk < steps; ++kk) {
          const uint64_t da = umma_desc_sw128(aV + kk * 2048, D == 128 ? 16384u : 0u, 1024u);
          const uint64_t db = umma_desc_sw128(aP + kk * 2048, 0u, 1024u);
          tc_mma_f16(tO, da, db, idesc_pv, (u > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(v_empty + vs);
        tc_commit(p_empty + pb);
      };
      mbar_wait(q_full, 0);
      for (int t = 0; t < n; ++t) {
        const int ks = t % kNK, sb = t & 1;
        mbar_wait(k_full + ks, (t / kNK) & 1);
        if (t >= 2) mbar_wait(s_empty + sb, ((t >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t aK = smem_u32(sK + ks * Cfg::kKVBytes);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t da = umma_desc_sw128(aK + (kk >> 2) * 16384 + (kk & 3) * 32, 16u, 1024u);
          const uint64_t db = umma_desc_sw128(aQ + (kk >> 2) * kSubBytes + (kk & 3) * 32, 16u, 1024u);
          tc_mma_f16(tS[sb], da, db, idesc_qk, kk > 0 ? 1u : 0u);
        }
        tc_commit(k_empty + ks);
        tc_commit(s_full + sb);
        if (t >= 1) issue_pv(t - 1);
      }
      issue_pv(n - 1);
    }
  } else {
    // ===================================== softmax (warps 0-3) ==========================
    const int j = threadIdx.x;  // key row == TMEM lane
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    float lpart[64];
#pragma unroll
    for (int q = 0; q < 64; ++q) lpart[q] = 0.0f;
    const int r_in_tile = j & 63;
    // query columns that are real tokens (ragged tiles have padding rows)
    uint32_t qv_lo = 0, qv_hi = 0;
#pragma unroll
    for (int q = 0; q < 64; ++q) {
      const bool ok = (qh0 + (q >> 3)) < g.rows && (qw0 + (q & 7)) < g.cols;
      if (ok) { if (q < 32) qv_lo |= 1u << q; else qv_hi |= 1u << (q - 32); }
    }
    unsigned long long my_pairs = 0;

    for (int t = 0; t < n; ++t) {
      const int sb = t & 1;
      // ---- key row j of this block: validity and allowed-query mask --------------------
      const int kb = sel_at(t);
      const int ktr = kb / g.n_tiles, ktile = kb % g.n_tiles;
      const int kcnt = g.k_tr_count[ktr];
      const int kframe = g.k_tr_first[ktr] + (j >> 6);
      const int kh = 8 * (ktile / g.tiles_w) + (r_in_tile >> 3);
      const int kw = 8 * (ktile % g.tiles_w) + (r_in_tile & 7);
      const bool kvalid = (j < 64 || kcnt == 2) && kh < g.rows && kw < g.cols;
      uint32_t mlo = 0, mhi = 0;  // bit q: query column q may attend key j
      if (kvalid) {
        if (m.kind == 0) {
          mlo = mhi = 0xffffffffu;
        } else if (m.kind == 1) {
          uint32_t wb = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) wb |= (kw >= win[16 + i] && kw < win[24 + i]) ? (1u << i) : 0u;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const bool hb = kh >= win[i] && kh < win[8 + i];
            if (hb) {
              if (i < 4) mlo |= wb << (8 * i);
              else mhi |= wb << (8 * (i - 4));
            }
          }
        } else {
          const long long tk = g.k_frame_tok0[kframe] + (long long)kh * g.cols + kw;
#pragma unroll 4
          for (int q = 0; q < 64; ++q) {
            const int qh = qh0 + (q >> 3), qw = qw0 + (q & 7);
            if (qh < g.rows && qw < g.cols) {
              const long long tq = g.q_frame_tok0[qf] + (long long)qh * g.cols + qw;
              if ((m.bits[tq * m.words_per_row + (tk >> 6)] >> (tk & 63)) & 1ull) {
                if (q < 32) mlo |= 1u << q; else mhi |= 1u << (q - 32);
              }
            }
          }
        }
      }

      my_pairs += __popc(mlo & qv_lo) + __popc(mhi & qv_hi);

      // ---- S^T row j -> registers ----------------------------------------------------
      mbar_wait(s_full + sb, (t >> 1) & 1);
      tc_fence_after();
      uint32_t sr[64];
      tmem_ld32(tS[sb] + lane_off, sr);
      tmem_ld32(tS[sb] + lane_off + 32u, sr + 32);
      tc_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_empty + sb);

      float x[64];
      bool exceed = false;
#pragma unroll
      for (int q = 0; q < 64; ++q) {
        const bool ok = ((q < 32 ? mlo >> q : mhi >> (q - 32)) & 1u) != 0u;
        x[q] = ok ? __uint_as_float(sr[q]) * p.scale_log2 : -INFINITY;
        exceed |= x[q] > c_ref[q] + kRescaleThreshold;
      }
      const bool wneed = __any_sync(0xffffffffu, exceed);
      if (lane == 0) flags[sb * 4 + warp] = wneed ? 1 : 0;
      named_bar_sync(1, 128);
      const bool need = (flags[sb * 4 + 0] | flags[sb * 4 + 1] | flags[sb * 4 + 2] | flags[sb * 4 + 3]) != 0;

      if (need) {
        float v[64];
#pragma unroll
        for (int q = 0; q < 64; ++q) v[q] = x[q];
        warp_colreduce64<true>(v, lane);
        red[warp * 64 + colreduce_col(lane, 0)] = v[0];
        red[warp * 64 + colreduce_col(lane, 1)] = v[1];
        named_bar_sync(1, 128);
        if (j < 64) {
          const float old = c_ref[j];
          const float mx = fmaxf(fmaxf(red[j], red[64 + j]), fmaxf(red[128 + j], red[192 + j]));
          const float nw = fmaxf(old, mx);
          c_ref[j] = nw;
          alpha[j] = (nw == -INFINITY) ? 1.0f : exp2f(old - nw);
        }
        named_bar_sync(1, 128);
#pragma unroll
        for (int q = 0; q < 64; ++q) lpart[q] *= alpha[q];
        if (t > 0) {
          // O^T holds PV(0..t-1): wait for PV(t-1), rescale column q by alpha[q].
          mbar_wait(p_empty + ((t - 1) & 1), ((t - 1) >> 1) & 1);
          tc_fence_after();
          if (j < D) {
            uint32_t o[64];
            tmem_ld32(tO + lane_off, o);
            tmem_ld32(tO + lane_off + 32u, o + 32);
            tc_wait_ld();
#pragma unroll
            for (int q = 0; q < 64; ++q) o[q] = __float_as_uint(__uint_as_float(o[q]) * alpha[q]);
            tmem_st32(tO + lane_off, o);
            tmem_st32(tO + lane_off + 32u, o + 32);
            tc_wait_st();
          }
        }
      }

      // ---- P^T row j (bf16), partial denominators -------------------------------------
      uint32_t pk[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float c0 = c_ref[2 * i], c1 = c_ref[2 * i + 1];
        const float p0 = x[2 * i] == -INFINITY ? 0.0f : exp2f(x[2 * i] - c0);
        const float p1 = x[2 * i + 1] == -INFINITY ? 0.0f : exp2f(x[2 * i + 1] - c1);
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
        lpart[2 * i] += __low2float(h2);
        lpart[2 * i + 1] += __high2float(h2);
        pk[i] = *reinterpret_cast<const uint32_t*>(&h2);
      }
      if (t >= 2) mbar_wait(p_empty + sb, ((t >> 1) - 1) & 1);
      uint8_t* prow = sP + sb * Cfg::kPBytes + j * 128;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        *reinterpret_cast<uint4*>(prow + ((ch ^ (j & 7)) << 4)) =
            make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full + sb);
    }

    // ---- epilogue ------------------------------------------------------------------------
    if (p.pairs) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) my_pairs += __shfl_xor_sync(0xffffffffu, my_pairs, o);
      if (lane == 0 && my_pairs) atomicAdd(p.pairs, my_pairs);
    }
    warp_colreduce64<false>(lpart, lane);
    red[warp * 64 + colreduce_col(lane, 0)] = lpart[0];
    red[warp * 64 + colreduce_col(lane, 1)] = lpart[1];
    named_bar_sync(1, 128);
    float* lsum = alpha;  // reuse
    if (j < 64) {
      const float l = (red[j] + red[64 + j]) + (red[128 + j] + red[192 + j]);
      lsum[j] = l;
      const int qh = qh0 + (j >> 3), qw = qw0 + (j & 7);
      if (qh < g.rows && qw < g.cols) {
        const long long tq = g.q_frame_tok0[qf] + (long long)qh * g.cols + qw;
        if (tq >= p.row_begin && tq < p.row_end && !(l > 0.0f)) atomicOr(p.err, kErrDegenerate);
      }
    }
    named_bar_sync(1, 128);
    // stage O (row-major [64 q][D] bf16) in P buffer 0, then write rows out
    uint16_t* so = reinterpret_cast<uint16_t*>(sP);
    if (n > 0) {
      mbar_wait(p_empty + ((n - 1) & 1), ((n - 1) >> 1) & 1);
      tc_fence_after();
      if (j < D) {
        uint32_t o[64];
        tmem_ld32(tO + lane_off, o);
        tmem_ld32(tO + lane_off + 32u, o + 32);
        tc_wait_ld();
#pragma unroll
        for (int q = 0; q < 64; ++q) {
          const float l = lsum[q];
          const float val = l > 0.0f ? __uint_as_float(o[q]) / l : 0.0f;
          so[q * D + j] = __bfloat16_as_ushort(__float2bfloat16_rn(val));
        }
      }
    } else if (j < D) {
#pragma unroll 8
      for (int q = 0; q < 64; ++q) so[q * D + j] = 0;
    }
    named_bar_sync(1, 128);
    constexpr int kChunks = D / 8;
    if (p.out_tile_major) {
      // unit-contiguous rows (padding rows included) for the head-parallel all-gather
      uint16_t* outu = p.out + (long long)blockIdx.x * 64 * D;
      for (int idx = j; idx < 64 * kChunks; idx += 128)
        *reinterpret_cast<uint4*>(outu + idx * 8) = *reinterpret_cast<const uint4*>(so + idx * 8);
    }
    uint16_t* outh = p.out + head * p.out_head_stride;
    for (int idx = j; idx < 64 * kChunks && !p.out_tile_major; idx += 128) {
      const int q = idx / kChunks, ch = idx % kChunks;
      const int qh = qh0 + (q >> 3), qw = qw0 + (q & 7);
      if (qh < g.rows && qw < g.cols) {
        const long long tq = g.q_frame_tok0[qf] + (long long)qh * g.cols + qw;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (tq >= p.row_begin && tq < p.row_end) val = *reinterpret_cast<const uint4*>(so + q * D + ch * 8);
        *reinterpret_cast<uint4*>(outh + tq * D + ch * 8) = val;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem, kTmemCols);
}

template __global__ void sparse_attn_kernel<64>(DevGeom, DevMask, AttnParams);
template __global__ void sparse_attn_kernel<128>(DevGeom, DevMask, AttnParams);

}  // namespace fvsr

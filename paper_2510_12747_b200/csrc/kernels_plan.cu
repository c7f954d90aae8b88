// kernels_plan.cu — mask builder (plan_sparse) and data-movement kernels for sm_100a.
//
//   pack_frames_kernel   flat [heads][L][d] bf16  ->  swizzled frame-tiles (fvsr_common.cuh)
//   pool_partials_kernel exact sequential fp32 block sums per frame-tile      (HBM-bound)
//   pack_pool_kernel     fused pack + pooled partial sums (ring append / query pooling)
//   coarse_score_kernel  coarse block scores, one thread per (q-block, k-block)
//   topk_select_kernel   coarse-allowed, top-k with forced diagonal, one warp per q-block
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
//   * selection (sparse.cpp:103-130): candidates ordered by (score desc, id asc) — we rank
//     64-bit keys (orderable(score) << 32 | ~id) with -0.0 canonicalised to +0.0 (they
//     compare equal in the reference), force the diagonal block first, take the k-1 best
//     others by a threshold search over the unique keys, emit ascending ids.
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
  pdl_wait();
  pdl_trigger();
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

// element loads of the pooling pass: bf16 bit patterns or fp32 (the reference's own inputs)
__device__ __forceinline__ float load_elem(const uint16_t* p) { return __uint_as_float((uint32_t)*p << 16); }
__device__ __forceinline__ float load_elem(const float* p) { return *p; }

template <typename T>
__global__ void __launch_bounds__(256) pool_partials_kernel(const T* __restrict__ src,
                                                            long long src_head_stride, int rows, int cols,
                                                            int tiles_w, int n_tiles, int d, PoolGroups groups,
                                                            SlotList slots, float* __restrict__ s0,
                                                            float* __restrict__ s1,
                                                            long long part_head_stride,  // elements
                                                            const float* __restrict__ ext_s0) {
  pdl_wait();
  pdl_trigger();
  const int tile = blockIdx.x, grp = blockIdx.y, head = blockIdx.z;
  const int th = tile / tiles_w, tw = tile % tiles_w;
  const int hc = min(8, rows - 8 * th), wc = min(8, cols - 8 * tw);
  const long long N = (long long)rows * cols;
  float* S0 = s0 + head * part_head_stride;
  float* S1 = s1 + head * part_head_stride;
  const int f0 = groups.first[grp], cnt = groups.count[grp];
  const int es = groups.ext_slot[grp];

  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const T* base = src + head * src_head_stride + c;
    // Sequential fp32 sum over one frame's tile rows in ascending token order, carried
    // in two accumulators: a0 (from 0.0f) and a1 (continued from `start`).
    auto frame_sum2 = [&](int f, float& a0, float& a1, bool two) {
      const T* fb = base + (long long)f * N * d;
#pragma unroll 1
      for (int rh = 0; rh < hc; ++rh) {
        const T* rowp = fb + ((long long)(8 * th + rh) * cols + 8 * tw) * d;
        float v[8];
#pragma unroll
        for (int rw = 0; rw < 8; ++rw) v[rw] = rw < wc ? load_elem(rowp + (long long)rw * d) : 0.0f;
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
// (V) is packed alongside without pooling.  One CTA (kPPThreads) per (tile, t_row group,
// head).  A tile row of 8 tokens is 8*d*2 contiguous bytes in the token-major source, so
// one elected thread stages the group's tiles into shared memory with one cp.async.bulk per
// tile row (all loads of the CTA in flight at once, no registers held); then threads
// < d/2 pool channels 2t, 2t+1 in token order from shared memory while every thread writes
// the swizzled tiles with coalesced 16-byte stores (thread i writes destination chunk i;
// the source chunk is the inverse swizzle).  Requires d % 8 == 0 (16-byte rows).
// ---------------------------------------------------------------------------------------
struct alignas(64) PackPoolArgs {
  // TMA path (use_tma): tensor maps of src / src2 as 5-D (channel, col, row, frame, head) with a
  // (64, 8, 8, 1, 1) box and 128-byte swizzle, i.e. one box = one 64-channel panel of a frame-tile
  // in exactly the ring's swizzled layout (fvsr_common.cuh); built on the host per call
  CUtensorMap tm;
  CUtensorMap tm2;
  int use_tma;
  const uint16_t* src;   // pooled + packed, [heads][frames * rows * cols][d]
  const uint16_t* src2;  // packed only (may be null)
  long long src_head_stride;  // elements (both sources)
  long long src_token_stride; // elements between consecutive tokens (0: d, i.e. [heads][L][d]);
                              // D = heads * d reads a projection GEMM's [L][D] output in place
  uint8_t* dst;
  uint8_t* dst2;
  long long dst_head_stride;  // bytes
  float* s0;
  float* s1;
  long long part_head_stride;  // elements
  const float* ext_s0;         // partner S0 for single-frame groups (ring appends), may be null
  float* norm2;                // optional: max squared row norm of src per frame-tile [slot][tile]
  long long norm2_head_stride; // elements
  // optional: the pooled block means themselves (avg_pool_blocks' final 1/count scale applied):
  // p0 = S0 / (rows x cols of the tile), p1 = S1 / (2 x that), channel-quad interleaved
  // [slot][d/4][tile][4] (head stride as s0 / s1); pflag
  // [slot][tile] (stride norm2_head_stride) gets bit 0 / bit 1 when p0 / p1 has a non-finite
  // value (matmul's check_finite, P/src/tensor.cpp:126-127, without re-reading the rows)
  float* p0;
  float* p1;
  unsigned* pflag;
  int rows, cols, tiles_w, n_tiles, d;
  // optional fused RoPE of src (apply_rope, P/src/rope.cpp:30-62) before pooling / packing:
  // (cos, sin) tables per axis position, float-rounded from the reference's double math
  const float2* rope_t;  // [frame id][dt/2]
  const float2* rope_h;  // [row][dh/2]
  const float2* rope_w;  // [col][dw/2]
  int rope_dt, rope_dh, rope_dw;
  int rope_fid[4];       // absolute frame id of source frame index 0..3
};

constexpr int kPPThreads = 128;

// shared bytes: [cnt frames][1 or 2 tensors][64 rows][d] bf16 + barrier
inline size_t pack_pool_smem(int d, int max_cnt, bool two) {
  return (size_t)max_cnt * (two ? 2 : 1) * 64 * d * 2 + 16 + 1024;  // + 1 KB: 128-byte-swizzle alignment
}


// Packed fp32 pair add (FADD2): {a0, a1} += {b0, b1}, each lane rounded exactly as add.rn.f32.
// (A packed multiply feeding it gets contracted into FFMA2 by ptxas, so the products stay
// scalar __fmul_rn.)
__device__ __forceinline__ void padd_rn(float& a0, float& a1, float b0, float b1) {
  unsigned long long x;
  asm("{\n\t.reg .b64 b2;\n\tmov.b64 b2, {%3, %4};\n\tmov.b64 %0, {%1, %2};\n\t"
      "add.rn.f32x2 %0, %0, b2;\n\t}"
      : "=l"(x)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(x));
}

// one bf16 channel pair (x0 | x1 << 16) rotated by (cos, sin): x0*c - x1*s, x0*s + x1*c in
// fp32 with separate multiply and add (apply_rope, P/src/rope.cpp:50-55), then bf16 RNE
__device__ __forceinline__ uint32_t rope_word(uint32_t v, float2 cs) {
  const float x0 = __uint_as_float(v << 16), x1 = __uint_as_float(v & 0xffff0000u);
  const float y0 = __fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y));
  const float y1 = __fadd_rn(__fmul_rn(x0, cs.y), __fmul_rn(x1, cs.x));
  const __nv_bfloat162 b = __floats2bfloat162_rn(y0, y1);
  return *reinterpret_cast<const uint32_t*>(&b);
}

// One (tile, t_row group, head) of the fused pack + pool pass by the whole CTA (kPPThreads
// threads), staging through `sm_pp` (pack_pool_smem bytes + RoPE tables).  A CTA that runs
// several passes calls it with use = 0, 1, 2, ...: the staging barrier is initialised once
// (use 0) and waited on with parity use & 1 (an mbarrier is not re-initialised while live),
// with a __syncthreads between passes.  `aux` (if given) holds the staging barrier and the
// RoPE tables apart from the tile staging area, which the caller may then reuse.
template <bool ROPE>
__device__ __forceinline__ void pack_pool_body(const PackPoolArgs& a, const PoolGroups& groups,
                                               const SlotList& slots, int tile, int grp, int head,
                                               uint8_t* sm_pp, int use = 0, uint8_t* aux = nullptr) {
  const int tid = threadIdx.x;
  const int d = a.d;
  const int th = tile / a.tiles_w, tw = tile - th * a.tiles_w;
  const int hc = min(8, a.rows - 8 * th), wc = min(8, a.cols - 8 * tw);
  const long long N = (long long)a.rows * a.cols;
  const uint32_t tile_bytes = (uint32_t)d * 128u;
  const int f0 = groups.first[grp], cnt = groups.count[grp], es = groups.ext_slot[grp];
  const int nt = a.src2 ? 2 : 1;
  uint8_t* aux_p = aux ? aux : sm_pp + (size_t)cnt * nt * tile_bytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(aux_p);
  auto stage = [&](int fi, int t) -> uint8_t* { return sm_pp + (size_t)(fi * nt + t) * tile_bytes; };
  const bool full = hc == 8 && wc == 8;
  if (!full) {  // edge tile: rows / columns past the frame are zero
    for (int i = tid; i < cnt * nt * (int)tile_bytes / 16; i += kPPThreads)
      reinterpret_cast<uint4*>(sm_pp)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
  }
  if (tid == 0) {
    if (use == 0) {
      mbar_init(bar, 1);
      fence_barrier_init();
    }
    fence_proxy_async_smem();
    const uint32_t row_bytes = (uint32_t)wc * d * 2;
    mbar_arrive_expect_tx(bar, row_bytes * hc * cnt * nt);
    const long long ts = a.src_token_stride ? a.src_token_stride : d;
    for (int fi = 0; fi < cnt; ++fi)
      for (int t = 0; t < nt; ++t) {
        const uint16_t* src = (t == 0 ? a.src : a.src2) + head * a.src_head_stride + (long long)(f0 + fi) * N * ts;
        for (int rh = 0; rh < hc; ++rh) {
          const long long tok = (long long)(8 * th + rh) * a.cols + 8 * tw;
          if (ts == d) {  // a tile row is contiguous
            bulk_g2s(stage(fi, t) + rh * 8 * d * 2, src + tok * d, row_bytes, bar);
          } else {        // one copy per token (its d channels are contiguous)
            for (int rw = 0; rw < wc; ++rw)
              bulk_g2s(stage(fi, t) + (rh * 8 + rw) * d * 2, src + (tok + rw) * ts, (uint32_t)d * 2, bar);
          }
        }
      }
  }
  // RoPE tables of this tile -> shared memory while the bulk copies are in flight:
  // t: [cnt][dt/2], h: [8 tile rows][dh/2], w: [8 tile cols][dw/2]
  float2* rtab = reinterpret_cast<float2*>(aux_p + 16);
  if constexpr (ROPE) {
    const int ht = a.rope_dt >> 1, hh = a.rope_dh >> 1, hw = a.rope_dw >> 1;
    for (int i = tid; i < cnt * ht; i += kPPThreads) {
      const int fi = i / ht, p = i - fi * ht;
      rtab[i] = a.rope_t[(long long)a.rope_fid[f0 + fi] * ht + p];
    }
    float2* rh_t = rtab + cnt * ht;
    for (int i = tid; i < 8 * hh; i += kPPThreads) {
      const int k = i / hh, p = i - k * hh;
      if (8 * th + k < a.rows) rh_t[i] = a.rope_h[(8 * th + k) * hh + p];
    }
    float2* rw_t = rh_t + 8 * hh;
    for (int i = tid; i < 8 * hw; i += kPPThreads) {
      const int k = i / hw, p = i - k * hw;
      if (8 * tw + k < a.cols) rw_t[i] = a.rope_w[(8 * tw + k) * hw + p];
    }
  }
  if (a.pflag && tid < cnt) a.pflag[head * a.norm2_head_stride + (long long)slots.s[f0 + tid] * a.n_tiles + tile] = 0u;
  __syncthreads();
  mbar_wait(bar, (uint32_t)use & 1u);
  // RoPE (ROPE): applied on the fly where the pooling and packing phases read the staged
  // src rows (both round the rotated pair to bf16 the same way, so the pooled sums, the |k|
  // bound and the stored tile agree); no serial rotate phase, no write-back
  const int r_ht = a.rope_dt >> 1, r_hh = a.rope_dh >> 1, r_hw = a.rope_dw >> 1;
  auto rope_cs = [&](int fi, int pi, int rh, int rw) -> float2 {
    if (pi < r_ht) return rtab[fi * r_ht + pi];
    if (pi < r_ht + r_hh) return rtab[cnt * r_ht + rh * r_hh + (pi - r_ht)];
    return rtab[cnt * r_ht + 8 * r_hh + rw * r_hw + (pi - r_ht - r_hh)];
  };
  // pooling (exact token order; rows past the frame are skipped, not added as zeros); a pass
  // with no partials (s0 null: the ring append's V) only packs
  if (a.s0 && 2 * tid < d) {
    const int c = 2 * tid;
    const long long po = (long long)tile * d + c;
    const bool ext = cnt == 1 && es >= 0 && a.ext_s0 != nullptr;
    float s1x = 0.0f, s1y = 0.0f;
    if (ext) {
      const float* e = a.ext_s0 + head * a.part_head_stride + (long long)es * a.n_tiles * d + po;
      s1x = e[0];
      s1y = e[1];
    }
    for (int fi = 0; fi < cnt; ++fi) {
      const int slot = slots.s[f0 + fi];
      const bool cont = fi == 1 || ext;
      const uint8_t* st = stage(fi, 0);
      float s0x = 0.0f, s0y = 0.0f;
      // ROPE: this thread's pair is fixed, so its (cos, sin) depends on at most the row (h axis)
      // or the column (w axis): the 8 column values live in registers, the row value is
      // reloaded once per tile row
      float2 cs_w[8];
      if constexpr (ROPE) {
#pragma unroll
        for (int rw = 0; rw < 8; ++rw) cs_w[rw] = rope_cs(fi, c >> 1, 0, rw < wc ? rw : 0);
      }
      for (int rh = 0; rh < hc; ++rh) {
        float2 cs_h = make_float2(1.0f, 0.0f);
        if constexpr (ROPE) cs_h = rope_cs(fi, c >> 1, rh, 0);
        const bool by_row = (c >> 1) < r_ht + r_hh;  // t or h axis: constant along the tile row
#pragma unroll
        for (int rw = 0; rw < 8; ++rw) {
          if (rw < wc) {
            uint32_t v = *reinterpret_cast<const uint32_t*>(st + ((rh * 8 + rw) * d + c) * 2);
            if constexpr (ROPE) v = rope_word(v, by_row ? cs_h : cs_w[rw]);
            const float x = __uint_as_float(v << 16), y = __uint_as_float(v & 0xffff0000u);
            s0x = __fadd_rn(s0x, x);
            s0y = __fadd_rn(s0y, y);
            if (cont) {
              s1x = __fadd_rn(s1x, x);
              s1y = __fadd_rn(s1y, y);
            }
          }
        }
      }
      float* S0 = a.s0 + head * a.part_head_stride + (long long)slot * a.n_tiles * d + po;
      S0[0] = s0x;
      S0[1] = s0y;
      if (cont) {
        float* S1 = a.s1 + head * a.part_head_stride + (long long)slot * a.n_tiles * d + po;
        S1[0] = s1x;
        S1[1] = s1y;
      }
      if (a.p0) {  // block means: single-frame block of this frame; pair block ending here
        const long long pofs = head * a.part_head_stride + (long long)slot * a.n_tiles * d + po;
        const float inv0 = __fdiv_rn(1.0f, (float)(hc * wc));
        const float m0x = __fmul_rn(s0x, inv0), m0y = __fmul_rn(s0y, inv0);
        // quad-interleaved [slot][c/4][tile][4]: a warp of the selector reading 32 consecutive
        // tiles' channel quad is one contiguous 512-byte run
        const long long qofs = head * a.part_head_stride + (((long long)slot * (d >> 2) + (c >> 2)) * a.n_tiles + tile) * 4 +
                               (c & 3);
        a.p0[qofs] = m0x;
        a.p0[qofs + 1] = m0y;
        unsigned bad = (isfinite(m0x) && isfinite(m0y)) ? 0u : 1u;
        if (cont) {
          const float inv1 = __fdiv_rn(1.0f, (float)(2 * hc * wc));
          const float m1x = __fmul_rn(s1x, inv1), m1y = __fmul_rn(s1y, inv1);
          a.p1[qofs] = m1x;
          a.p1[qofs + 1] = m1y;
          if (!(isfinite(m1x) && isfinite(m1y))) bad |= 2u;
        }
        if (bad && a.pflag) atomicOr(a.pflag + head * a.norm2_head_stride + (long long)slot * a.n_tiles + tile, bad);
      }
      if (fi == 0 && cnt == 2) {  // frame B continues frame A's sequence
        s1x = s0x;
        s1y = s0y;
      }
    }
  }
  // packing: destination chunk i (16 B) of a tile <- source (row r, channel chunk)
  const int chunks = (int)tile_bytes / 16;
  for (int fi = 0; fi < cnt; ++fi) {
    const int slot = slots.s[f0 + fi];
    const long long to = head * a.dst_head_stride + ((long long)slot * a.n_tiles + tile) * tile_bytes;
    for (int t = 0; t < nt; ++t) {
      const uint8_t* st = stage(fi, t);
      uint8_t* dst = (t == 0 ? a.dst : a.dst2) + to;
      // Thread tid touches rows tid/8 + 16*(k%4) (8 channels per chunk); with norm2 it also
      // accumulates those rows' sums of squares (bounds every score |q.k| <= |q||k| for the
      // attention kernel's rescale-vote skip).
      float rowacc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int i = tid, k = 0; i < chunks; i += kPPThreads, ++k) {
        const int panel = i >> 9, r = (i >> 3) & 63, j = i & 7;
        const int c = panel * 64 + ((j ^ (r & 7)) << 3);
        uint4 v = *reinterpret_cast<const uint4*>(st + (r * d + c) * 2);
        if constexpr (ROPE) {
          if (t == 0 && (r >> 3) < hc && (r & 7) < wc) {  // rows past the frame stay zero
            const int p0 = c >> 1, rh = r >> 3, rw = r & 7;
            v.x = rope_word(v.x, rope_cs(fi, p0, rh, rw));
            v.y = rope_word(v.y, rope_cs(fi, p0 + 1, rh, rw));
            v.z = rope_word(v.z, rope_cs(fi, p0 + 2, rh, rw));
            v.w = rope_word(v.w, rope_cs(fi, p0 + 3, rh, rw));
          }
        }
        *reinterpret_cast<uint4*>(dst + (size_t)i * 16) = v;
        if (t == 0 && a.norm2) {
          const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
          float acc = rowacc[k & 3];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x = __uint_as_float(w4[e] << 16), y = __uint_as_float(w4[e] & 0xffff0000u);
            acc = fmaf(x, x, fmaf(y, y, acc));
          }
          rowacc[k & 3] = acc;
        }
      }
      if (t == 0 && a.norm2) {
        __shared__ float wmax[kPPThreads / 32];
        float mx = 0.0f;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          float rs = rowacc[kk];  // full row sum over the 8 lanes sharing tid / 8
          rs += __shfl_xor_sync(0xffffffffu, rs, 1);
          rs += __shfl_xor_sync(0xffffffffu, rs, 2);
          rs += __shfl_xor_sync(0xffffffffu, rs, 4);
          mx = fmaxf(mx, rs);
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        if ((tid & 31) == 0) wmax[tid >> 5] = mx;
        __syncthreads();
        if (tid == 0) {
#pragma unroll
          for (int w = 1; w < kPPThreads / 32; ++w) mx = fmaxf(mx, wmax[w]);
          a.norm2[head * a.norm2_head_stride + (long long)slot * a.n_tiles + tile] = mx;
        }
        __syncthreads();
      }
    }
  }
}

// The same pass with the tiles brought in by the tensor cores' copy engine already in the
// ring's layout: one TMA box per 64-channel panel per (frame, tensor) lands swizzled (and
// zero-filled past the frame edge) in shared memory, the threads pool (and with ROPE first
// rotate in place) and take the |row| bounds from it, and one bulk copy per frame-tile
// writes it to the ring slot / query workspace.  No per-chunk register traffic: an append of
// V is three instructions of one thread.
template <bool ROPE>
__device__ __forceinline__ void pack_pool_tma(const PackPoolArgs& a, const PoolGroups& groups, const SlotList& slots,
                                              int tile, int grp, int head, uint8_t* sm_raw) {
  const int tid = threadIdx.x;
  const int d = a.d;
  const int th = tile / a.tiles_w, tw = tile - th * a.tiles_w;
  const int hc = min(8, a.rows - 8 * th), wc = min(8, a.cols - 8 * tw);
  const uint32_t tile_bytes = (uint32_t)d * 128u;
  const int f0 = groups.first[grp], cnt = groups.count[grp], es = groups.ext_slot[grp];
  const int nt = a.src2 ? 2 : 1;
  uint8_t* base = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  auto stage = [&](int fi, int t) -> uint8_t* { return base + (size_t)(fi * nt + t) * tile_bytes; };
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + (size_t)cnt * nt * tile_bytes);
  float2* rtab = reinterpret_cast<float2*>(base + (size_t)cnt * nt * tile_bytes + 16);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(bar, tile_bytes * cnt * nt);
    for (int fi = 0; fi < cnt; ++fi)
      for (int t = 0; t < nt; ++t)
        for (int pnl = 0; pnl < d / 64; ++pnl)
          tma_load_5d(stage(fi, t) + pnl * 8192, t == 0 ? &a.tm : &a.tm2, 64 * pnl, 8 * tw, 8 * th, f0 + fi, head, bar);
  }
  if (a.pflag && tid < cnt) a.pflag[head * a.norm2_head_stride + (long long)slots.s[f0 + tid] * a.n_tiles + tile] = 0u;
  const int r_ht = a.rope_dt >> 1, r_hh = a.rope_dh >> 1, r_hw = a.rope_dw >> 1;
  if constexpr (ROPE) {  // this tile's (cos, sin): t: [cnt][dt/2], h: [8][dh/2], w: [8][dw/2]
    for (int i = tid; i < cnt * r_ht; i += kPPThreads) {
      const int fi = i / r_ht, q = i - fi * r_ht;
      rtab[i] = a.rope_t[(long long)a.rope_fid[f0 + fi] * r_ht + q];
    }
    float2* rh_t = rtab + cnt * r_ht;
    for (int i = tid; i < 8 * r_hh; i += kPPThreads) {
      const int k = i / r_hh, q = i - k * r_hh;
      if (8 * th + k < a.rows) rh_t[i] = a.rope_h[(8 * th + k) * r_hh + q];
    }
    float2* rw_t = rh_t + 8 * r_hh;
    for (int i = tid; i < 8 * r_hw; i += kPPThreads) {
      const int k = i / r_hw, q = i - k * r_hw;
      if (8 * tw + k < a.cols) rw_t[i] = a.rope_w[(8 * tw + k) * r_hw + q];
    }
  }
  __syncthreads();  // barrier initialised, flags reset, RoPE tables staged
  mbar_wait(bar, 0);
  // byte offset of (row r, channel c) in a swizzled frame-tile
  auto at = [](int r, int c) -> uint32_t {
    return (uint32_t)((c >> 6) * 8192 + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) + (c & 7) * 2);
  };
  if constexpr (ROPE) {  // rotate src in place (rows past the frame stay zero)
    const int chunks = (int)tile_bytes / 16;
    for (int fi = 0; fi < cnt; ++fi) {
      uint8_t* st = stage(fi, 0);
      for (int i = tid; i < chunks; i += kPPThreads) {
        const int pnl = i >> 9, r = (i >> 3) & 63, j = i & 7;
        const int rh = r >> 3, rw = r & 7;
        if (rh >= hc || rw >= wc) continue;
        const int p0 = (pnl * 64 + ((j ^ (r & 7)) << 3)) >> 1;  // first channel pair of the chunk
        uint4 v = *reinterpret_cast<uint4*>(st + (size_t)i * 16);
        auto cs = [&](int pi) -> float2 {
          if (pi < r_ht) return rtab[fi * r_ht + pi];
          if (pi < r_ht + r_hh) return rtab[cnt * r_ht + rh * r_hh + (pi - r_ht)];
          return rtab[cnt * r_ht + 8 * r_hh + rw * r_hw + (pi - r_ht - r_hh)];
        };
        v.x = rope_word(v.x, cs(p0));
        v.y = rope_word(v.y, cs(p0 + 1));
        v.z = rope_word(v.z, cs(p0 + 2));
        v.w = rope_word(v.w, cs(p0 + 3));
        *reinterpret_cast<uint4*>(st + (size_t)i * 16) = v;
      }
    }
    __syncthreads();
  }
  // pooling: channels 2t, 2t+1 in exact token order (rows past the frame skipped)
  if (a.s0 && 2 * tid < d) {
    const int c = 2 * tid;
    const long long po = (long long)tile * d + c;
    const bool ext = cnt == 1 && es >= 0 && a.ext_s0 != nullptr;
    float s1x = 0.0f, s1y = 0.0f;
    if (ext) {
      const float* e = a.ext_s0 + head * a.part_head_stride + (long long)es * a.n_tiles * d + po;
      s1x = e[0];
      s1y = e[1];
    }
    for (int fi = 0; fi < cnt; ++fi) {
      const int slot = slots.s[f0 + fi];
      const bool cont = fi == 1 || ext;
      const uint8_t* st = stage(fi, 0);
      float s0x = 0.0f, s0y = 0.0f;
      // x and y advance together as one packed add
      for (int rh = 0; rh < hc; ++rh) {
        uint32_t w[8];
#pragma unroll
        for (int rw = 0; rw < 8; ++rw) w[rw] = *reinterpret_cast<const uint32_t*>(st + at(rh * 8 + rw, c));
#pragma unroll
        for (int rw = 0; rw < 8; ++rw) {
          if (rw < wc) {
            const float x = __uint_as_float(w[rw] << 16), y = __uint_as_float(w[rw] & 0xffff0000u);
            padd_rn(s0x, s0y, x, y);
            if (cont) padd_rn(s1x, s1y, x, y);
          }
        }
      }
      const long long pofs = head * a.part_head_stride + (long long)slot * a.n_tiles * d + po;
      a.s0[pofs] = s0x;
      a.s0[pofs + 1] = s0y;
      if (cont) {
        a.s1[pofs] = s1x;
        a.s1[pofs + 1] = s1y;
      }
      if (a.p0) {  // block means: single-frame block of this frame; pair block ending here
        const float inv0 = __fdiv_rn(1.0f, (float)(hc * wc));
        const float m0x = __fmul_rn(s0x, inv0), m0y = __fmul_rn(s0y, inv0);
        // quad-interleaved [slot][c/4][tile][4]: a warp of the selector reading 32 consecutive
        // tiles' channel quad is one contiguous 512-byte run
        const long long qofs = head * a.part_head_stride + (((long long)slot * (d >> 2) + (c >> 2)) * a.n_tiles + tile) * 4 +
                               (c & 3);
        a.p0[qofs] = m0x;
        a.p0[qofs + 1] = m0y;
        unsigned bad = (isfinite(m0x) && isfinite(m0y)) ? 0u : 1u;
        if (cont) {
          const float inv1 = __fdiv_rn(1.0f, (float)(2 * hc * wc));
          const float m1x = __fmul_rn(s1x, inv1), m1y = __fmul_rn(s1y, inv1);
          a.p1[qofs] = m1x;
          a.p1[qofs + 1] = m1y;
          if (!(isfinite(m1x) && isfinite(m1y))) bad |= 2u;
        }
        if (bad && a.pflag) atomicOr(a.pflag + head * a.norm2_head_stride + (long long)slot * a.n_tiles + tile, bad);
      }
      if (fi == 0 && cnt == 2) {  // frame B continues frame A's sequence
        s1x = s0x;
        s1y = s0y;
      }
    }
  }
  // |row| bounds of src (max squared row norm per frame-tile): two threads per row
  if (a.norm2) {
    __shared__ float wmax_t[kPPThreads / 32];
    const int r = tid >> 1, half = tid & 1, cpt = d >> 1;  // channels per thread
    for (int fi = 0; fi < cnt; ++fi) {
      const uint8_t* st = stage(fi, 0);
      float acc4[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // four independent chains
#pragma unroll 8
      for (int c = half * cpt; c < (half + 1) * cpt; c += 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(st + at(r, c));
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x = __uint_as_float(w4[e] << 16), y = __uint_as_float(w4[e] & 0xffff0000u);
          acc4[e] = fmaf(x, x, fmaf(y, y, acc4[e]));
        }
      }
      float acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
#pragma unroll
      for (int o = 2; o < 32; o <<= 1) acc = fmaxf(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if ((tid & 31) == 0) wmax_t[tid >> 5] = acc;
      __syncthreads();
      if (tid == 0) {
        float mx = wmax_t[0];
#pragma unroll
        for (int w = 1; w < kPPThreads / 32; ++w) mx = fmaxf(mx, wmax_t[w]);
        a.norm2[head * a.norm2_head_stride + (long long)slots.s[f0 + fi] * a.n_tiles + tile] = mx;
      }
      __syncthreads();
    }
  }
  if constexpr (ROPE) fence_proxy_async_smem();  // rotated tiles: generic writes -> async-proxy reads
  __syncthreads();
  if (tid == 0) {
    for (int fi = 0; fi < cnt; ++fi) {
      const long long to = head * a.dst_head_stride + ((long long)slots.s[f0 + fi] * a.n_tiles + tile) * tile_bytes;
      for (int t = 0; t < nt; ++t) bulk_s2g((t == 0 ? a.dst : a.dst2) + to, stage(fi, t), tile_bytes);
    }
    bulk_commit();
    bulk_wait_read();  // shared memory stays valid until the copies have read it
  }
}

template <bool ROPE>
__global__ void __launch_bounds__(kPPThreads) pack_pool_kernel(const __grid_constant__ PackPoolArgs a,
                                                               const __grid_constant__ PoolGroups groups,
                                                               const __grid_constant__ SlotList slots) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) uint8_t sm_pp[];
  if (a.use_tma)
    pack_pool_tma<ROPE>(a, groups, slots, blockIdx.x, blockIdx.y, blockIdx.z, sm_pp);
  else
    pack_pool_body<ROPE>(a, groups, slots, blockIdx.x, blockIdx.y, blockIdx.z, sm_pp);
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

// out-of-line variant for mask kinds other than "all" (keeps the selector's unrolled
// candidate loop small; kind 0 never calls it)
__device__ __noinline__ bool coarse_allowed_masked(const DevGeom& g, const DevMask& m, int qtr, int qtile, int ktr,
                                                   int ktile) {
  return coarse_allowed(g, m, qtr, qtile, ktr, ktile);
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
  const float* k_p0;        // ring block means (PackPoolArgs::p0 / p1, same layout as k_s0 / k_s1)
  const float* k_p1;
  const unsigned* k_flag;   // [slot][n_tiles] non-finite bits of k_p0 / k_p1
  long long k_flag_head_stride;

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

__device__ inline uint32_t order_score(float s) {  // order_key's upper half; 0 = no candidate
  uint32_t u = __float_as_uint(s == 0.0f ? 0.0f : s);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Coarse scores over shared-memory tiles of kScQ pooled queries x kScK pooled keys, row
// stride d+4 floats (16-byte aligned rows; the 4-float skew spreads the 8 rows one LDS.128
// wavefront touches over all banks).  Thread t owns queries 2*(t/16) + {0,1} and keys
// t%16 + 16*{0..3}: 8 independent exact chains, 6 LDS.128 per 4 channels.  Every chain is
// the reference's sequential fp32 order (see file header): channels ascending, separate
// multiply and add from 0.0f, then the 1/sqrt(d) multiply.
constexpr int kScQ = 16, kScK = 64, kScThreads = 128;

__device__ inline void chain4(float& acc, const float4& a, const float4& b) {
  acc = __fadd_rn(acc, __fmul_rn(a.x, b.x));
  acc = __fadd_rn(acc, __fmul_rn(a.y, b.y));
  acc = __fadd_rn(acc, __fmul_rn(a.z, b.z));
  acc = __fadd_rn(acc, __fmul_rn(a.w, b.w));
}

__global__ void __launch_bounds__(kScThreads) coarse_score_kernel(DevGeom g, DevMask m, SelectParams p,
                                                                 float* __restrict__ scores) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) float smf[];
  const int d = g.d, ld = d + 4, d4 = d >> 2;
  float* pq = smf;              // [kScQ][d+4]
  float* pk = smf + kScQ * ld;  // [kScK][d+4]
  const int kb0 = blockIdx.x * kScK, qb0 = blockIdx.y * kScQ, head = blockIdx.z;
  const int tid = threadIdx.x;
  // per staged row: source pointer and 1/count (rows past the grid stage zeros)
  __shared__ const float* row_src[kScQ + kScK];
  __shared__ float row_inv[kScQ + kScK];
  if (tid < kScQ + kScK) {
    const int r = tid;
    const float* src = nullptr;
    int cnt_tok = 1;
    if (r < kScQ) {
      const int qb = qb0 + r;
      if (qb < g.bnq) {
        const int qtr = qb / g.n_tiles, qtile = qb - qtr * g.n_tiles;
        const int qcnt = g.q_tr_count[qtr];
        const int qf = g.q_tr_first[qtr] + qcnt - 1;
        src = (qcnt == 2 ? p.q_s1 : p.q_s0) + head * p.q_head_stride + ((long long)qf * g.n_tiles + qtile) * d;
        cnt_tok = qcnt * tile_h_count(g, qtile) * tile_w_count(g, qtile);
      }
    } else {
      const int kb = kb0 + r - kScQ;
      if (kb < g.bnk) {
        const int ktr = kb / g.n_tiles, ktile = kb - ktr * g.n_tiles;
        const int kcnt = g.k_tr_count[ktr];
        const int kf = g.k_tr_first[ktr] + kcnt - 1;
        src = (kcnt == 2 ? p.k_s1 : p.k_s0) + head * p.k_head_stride +
              ((long long)g.k_slot[kf] * g.n_tiles + ktile) * d;
        cnt_tok = kcnt * tile_h_count(g, ktile) * tile_w_count(g, ktile);
      }
    }
    row_src[r] = src;
    row_inv[r] = __fdiv_rn(1.0f, (float)cnt_tok);
  }
  __syncthreads();
  // stage: warp w copies rows w, w+4, ...; lane = float4 column; kB rows in flight
  bool fin = true;
  constexpr int kB = 10, kRows = kScQ + kScK, kWarps = kScThreads / 32;
  const int warp = tid >> 5, lane = tid & 31;
  for (int c4 = lane; c4 < d4; c4 += 32) {
#pragma unroll 1
    for (int r0 = warp; r0 < kRows; r0 += kB * kWarps) {
      float4 v[kB];
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const int r = r0 + j * kWarps;
        const float* src = r < kRows ? row_src[r] : nullptr;
        v[j] = src ? __ldg(reinterpret_cast<const float4*>(src) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const int r = r0 + j * kWarps;
        if (r < kRows) {
          const float inv = row_inv[r];
          float4 w = v[j];
          w.x = __fmul_rn(w.x, inv);
          w.y = __fmul_rn(w.y, inv);
          w.z = __fmul_rn(w.z, inv);
          w.w = __fmul_rn(w.w, inv);
          fin = fin && isfinite(w.x) && isfinite(w.y) && isfinite(w.z) && isfinite(w.w);
          *reinterpret_cast<float4*>(smf + r * ld + c4 * 4) = w;
        }
      }
    }
  }
  if (!fin) atomicOr(p.err, kErrShape);
  __syncthreads();
  const int kq = tid & 15, qg = tid >> 4;
  const float* q0 = pq + (2 * qg) * ld;
  const float* q1 = q0 + ld;
  const float* k0 = pk + kq * ld;
  float acc[2][4] = {};
#pragma unroll 4
  for (int c = 0; c < d; c += 4) {
    const float4 a0 = *reinterpret_cast<const float4*>(q0 + c);
    const float4 a1 = *reinterpret_cast<const float4*>(q1 + c);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 b = *reinterpret_cast<const float4*>(k0 + 16 * j * ld + c);
      chain4(acc[0][j], a0, b);
      chain4(acc[1][j], a1, b);
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int qb = qb0 + 2 * qg + i;
    if (qb >= g.bnq) continue;
    float* row = scores + ((long long)head * g.bnq + qb) * g.bnk;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int kb = kb0 + kq + 16 * j;
      if (kb < g.bnk) row[kb] = __fmul_rn(acc[i][j], p.scale);
    }
  }
}

// Top-k per (head, q-block): one warp each, the row's candidates held in registers
// (NPER per lane, key block kb = 32*i + lane).  Candidates are the coarse-allowed key
// blocks other than the diagonal, ranked by (score desc, id asc) == the reference's
// stable_sort (sparse.cpp:103-130).  The diagonal block (if allowed) is forced first and
// counts toward k.  Threshold T = the kprime-th largest orderable score, by a 32-round
// bitwise search whose counts are ballot popcounts (no shuffles); all candidates above T
// are taken, and the lowest ids among those equal to T fill the rest — exactly the
// stable-sort prefix.  A ballot compaction emits ascending ids.
constexpr int kTopkWarps = 8;

// Top-k of one (head, q-block) row by one warp, the row's candidates held in registers
// (NPER per lane, key block kb = 32*i + lane).  Candidates are the coarse-allowed key blocks
// other than the diagonal, ranked by (score desc, id asc) == the reference's stable_sort
// (sparse.cpp:103-130).  The diagonal block (if allowed) is forced first and counts toward
// k.  Threshold T = the kprime-th largest orderable score, by a 32-round bitwise search
// whose counts are ballot popcounts (no shuffles); all candidates above T are taken, and
// the lowest ids among those equal to T fill the rest — exactly the stable-sort prefix.  A
// ballot compaction emits ascending ids.  `sc` (global or shared) holds the row's scores.
// Threshold of a warp's candidates by radix select: the kprime-th largest order score (with
// multiplicity) in four 8-bit digit rounds, each a shared-memory histogram of the candidates
// that match the digits fixed so far (`hist`: 256 words per warp) and a suffix scan over the
// lanes' 8-bin slices.  Same T and take_eq as the 32-round bit search; requires
// 0 < kprime < number of candidates.
template <int NPER>
__device__ __forceinline__ uint32_t kth_largest_radix(const uint32_t (&os)[NPER], int kprime, unsigned* hist,
                                                      int& take_eq) {
  const int lane = threadIdx.x & 31;
  uint32_t prefix = 0u, pmask = 0u;
  int need = kprime;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    reinterpret_cast<uint4*>(hist)[2 * lane] = make_uint4(0u, 0u, 0u, 0u);
    reinterpret_cast<uint4*>(hist)[2 * lane + 1] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NPER; ++i)
      if (os[i] != 0u && (os[i] & pmask) == prefix) atomicAdd(&hist[(os[i] >> shift) & 255u], 1u);
    __syncwarp();
    const uint4 h0 = reinterpret_cast<const uint4*>(hist)[2 * lane];
    const uint4 h1 = reinterpret_cast<const uint4*>(hist)[2 * lane + 1];
    const int c[8] = {(int)h0.x, (int)h0.y, (int)h0.z, (int)h0.w, (int)h1.x, (int)h1.y, (int)h1.z, (int)h1.w};
    int local = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) local += c[j];
    int suf = local;  // candidates with digit >= 8 * lane
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_down_sync(0xffffffffu, suf, o);
      if (lane + o < 32) suf += v;
    }
    const int above = suf - local;  // candidates with digit >= 8 * (lane + 1)
    const bool mine = above < need && suf >= need;
    const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
    int dg = 0, a = above;
    if (mine) {
      dg = -1;
#pragma unroll
      for (int j = 7; j >= 0; --j)
        if (dg < 0) {
          if (a + c[j] >= need) dg = j;
          else a += c[j];
        }
      dg += 8 * lane;
    }
    dg = __shfl_sync(0xffffffffu, dg, src);
    a = __shfl_sync(0xffffffffu, a, src);
    need -= a;
    prefix |= (uint32_t)dg << shift;
    pmask |= 255u << shift;
    __syncwarp();
  }
  take_eq = need;
  return prefix;
}

template <int NPER>
__device__ __forceinline__ void topk_core(const DevGeom& g, const DevMask& m, const SelectParams& p, int qb, int head,
                                          const float (&sv)[NPER], unsigned* hist) {
  const int lane = threadIdx.x & 31;
  const int bnk = g.bnk;
  const int qtr = qb / g.n_tiles, qtile = qb - qtr * g.n_tiles;
  const long long row = (long long)head * g.bnq + qb;
  int dg = -1;
  if (g.q_tr_diag[qtr] >= 0) dg = g.q_tr_diag[qtr] * g.n_tiles + qtile;
  uint32_t os[NPER];
  bool dg_ok = false;
  int n_cand = 0;
  // Locality window: coarse-allowed depends on the (query tile, key tile) pair only, so the
  // row's allowed key tiles are one bit table (in the radix histogram's space, which is not in
  // use yet), built 32 tiles per step; the candidates then walk their key tile incrementally
  const bool loc_table = m.kind == 1 && hist != nullptr && g.n_tiles <= 32 * 256;
  int kt = lane % g.n_tiles;  // key tile of candidate kb = 32 * i + lane
  if (loc_table) {
    const int qh0 = 8 * (qtile / g.tiles_w), qw0 = 8 * (qtile % g.tiles_w);
    const int qhc = tile_h_count(g, qtile), qwc = tile_w_count(g, qtile);
    for (int t0 = 0; t0 < g.n_tiles; t0 += 32) {
      const int t = t0 + lane;
      bool a = false;
      if (t < g.n_tiles) {
        const int kth = t / g.tiles_w, ktw = t - kth * g.tiles_w;
        a = range_overlap(m.mode, qh0, qhc, 8 * kth, tile_h_count(g, t), m.extent_h, g.rows) &&
            range_overlap(m.mode, qw0, qwc, 8 * ktw, tile_w_count(g, t), m.extent_w, g.cols);
      }
      const unsigned w = __ballot_sync(0xffffffffu, a);
      if (lane == 0) hist[t0 >> 5] = w;
    }
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const int kb = 32 * i + lane;
    bool al = kb < bnk;
    if (loc_table) {
      if (i > 0) {
        kt += 32;
        while (kt >= g.n_tiles) kt -= g.n_tiles;
      }
      al = al && ((hist[kt >> 5] >> (kt & 31)) & 1u);
    } else if (m.kind != 0 && al) {
      const int ktr = kb / g.n_tiles, ktile = kb - ktr * g.n_tiles;
      al = coarse_allowed_masked(g, m, qtr, qtile, ktr, ktile);
    }
    if (kb < bnk) {
      if (p.coarse) p.coarse[row * bnk + kb] = sv[i];
      if (p.allowed) p.allowed[row * bnk + kb] = al ? 1 : 0;
    }
    if (al && kb == dg) dg_ok = true;
    os[i] = (al && kb != dg) ? order_score(sv[i]) : 0u;
    n_cand += __popc(__ballot_sync(0xffffffffu, os[i] != 0u));
  }
  if (!__any_sync(0xffffffffu, dg_ok)) dg = -1;
  if (loc_table) __syncwarp();  // the table's reads before the radix histogram reuses its space
  const long long kp64 = p.topk - (dg >= 0 ? 1 : 0);
  const int kprime = kp64 > (long long)INT32_MAX ? INT32_MAX : (int)kp64;
  uint32_t T = 1u;  // every candidate
  int take_eq = 1 << 30;
  if (kprime <= 0) {
    T = 0xFFFFFFFFu;
    take_eq = 0;
  } else if (kprime < n_cand && hist) {
    T = kth_largest_radix<NPER>(os, kprime, hist, take_eq);
  } else if (kprime < n_cand) {
    uint32_t prefix = 0u;
#pragma unroll 1
    for (int bit = 31; bit >= 0; --bit) {
      const uint32_t trial = prefix | (1u << bit);
      int cnt = 0;
#pragma unroll
      for (int i = 0; i < NPER; ++i) cnt += __popc(__ballot_sync(0xffffffffu, os[i] >= trial));
      if (cnt >= kprime) prefix = trial;
    }
    T = prefix;
    int gt = 0;
#pragma unroll
    for (int i = 0; i < NPER; ++i) gt += __popc(__ballot_sync(0xffffffffu, os[i] > T));
    take_eq = kprime - gt;
  }
  int* out = p.sel + row * p.cap;
  const unsigned lt = (1u << lane) - 1u;
  int total = 0, eq_seen = 0;
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const int kb = 32 * i + lane;
    const bool eq = os[i] != 0u && os[i] == T;
    const unsigned be = __ballot_sync(0xffffffffu, eq);
    const bool f = (os[i] != 0u && os[i] > T) || (eq && eq_seen + __popc(be & lt) < take_eq) || (kb == dg);
    eq_seen += __popc(be);
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (f) {
      const int pos = total + __popc(bal & lt);
      if (pos < p.cap) out[pos] = kb;
    }
    total += __popc(bal);
  }
  for (int i = total + lane; i < p.cap; i += 32) out[i] = -1;
  if (lane == 0) {
    p.sel_count[row] = total;
    if (p.diag) p.diag[row] = dg;
    if (total > p.cap) atomicOr(p.err, kErrInvariant);
  }
}

// topk_core of a row whose scores are in memory (global or shared)
template <int NPER>
__device__ __forceinline__ void topk_row(const DevGeom& g, const DevMask& m, const SelectParams& p, int qb, int head,
                                         const float* sc, unsigned* hist = nullptr) {
  const int lane = threadIdx.x & 31;
  float sv[NPER];
#pragma unroll
  for (int i = 0; i < NPER; ++i) {  // all loads in flight before any use
    const int kb = 32 * i + lane;
    sv[i] = kb < g.bnk ? sc[kb] : 0.0f;
  }
  topk_core<NPER>(g, m, p, qb, head, sv, hist);
}



template <int NPER>
__global__ void __launch_bounds__(kTopkWarps * 32) topk_select_kernel(const __grid_constant__ DevGeom g,
                                                                     const __grid_constant__ DevMask m,
                                                                     const __grid_constant__ SelectParams p,
                                                                     const float* __restrict__ scores) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5;
  const int qb = blockIdx.x * kTopkWarps + warp;
  if (qb >= g.bnq) return;
  const int head = blockIdx.y;
  __shared__ __align__(16) unsigned hist[kTopkWarps][256];
  topk_row<NPER>(g, m, p, qb, head, scores + ((long long)head * g.bnq + qb) * g.bnk, hist[warp]);
}

// ---------------------------------------------------------------------------------------
// Streaming front end of one layer-step (ring append + mask builder) in two launches:
//   ring_pack_kernel   blocks [0, heads*n_tiles): KVCache::append of the new frame's K tile
//                      (swizzled ring slot, pooled partials, |k| bounds); then the query
//                      frames' tiles (packed for the tensor cores, pooled partials, |q|
//                      bounds); the last heads*n_tiles blocks: the new frame's V tile
//                      (swizzled ring slot only).  Independent inputs, one pass over HBM; one 16 KB tile per block
//                      keeps ~13 blocks (208 KB of loads in flight) on every SM.
//   mask_select_kernel kFrontQB q-blocks of one head per block: pooled queries, coarse scores
//                      against the ring's pooled keys streamed through shared memory in
//                      kFrontKC-block chunks (exact sequential chains, P/src/tensor.cpp:121-151,
//                      sparse.cpp:97-99), top-k with the forced diagonal (topk_row).
// ---------------------------------------------------------------------------------------
constexpr int kFrontQB = 6;  // q-blocks (pooled query rows) per mask-select block (2-8 measured; 6 fills 132 SMs)
constexpr int kFrontQP = kFrontQB <= 2 ? 2 : (kFrontQB <= 4 ? 4 : 8);  // query slots per channel (transposed tile)
constexpr int kFrontThreads = 256; // one key block per thread (strided past 256)

struct FrontArgs {
  PackPoolArgs kv;   // append K: src = k, dst = ring slot, partials + |k| bounds (src null: no append)
  PackPoolArgs v;    // append V: src = v, dst = ring slot, pack only (s0 null)
  PoolGroups kv_pg;
  SlotList kv_sl;
  PackPoolArgs q;    // query frames: packed tiles + pooled partials into the workspace
  PoolGroups q_pg;
  SlotList q_sl;
  int heads, n_tiles, q_trows;
};

inline size_t ring_pack_smem(int d, int max_q_cnt, size_t rope_bytes) {
  return pack_pool_smem(d, max_q_cnt, false) + rope_bytes;
}

template <bool ROPE>
__global__ void __launch_bounds__(kPPThreads, 12) ring_pack_kernel(const __grid_constant__ FrontArgs fa) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) uint8_t sm_rp[];
  const int n_append = fa.kv.src != nullptr ? fa.heads * fa.n_tiles : 0;
  int b = blockIdx.x;
  auto run = [&](const PackPoolArgs& a, const PoolGroups& pg, const SlotList& sl, int tile, int grp, int head,
                 bool rope) {
    if (a.use_tma) {
      if (rope) pack_pool_tma<ROPE>(a, pg, sl, tile, grp, head, sm_rp);
      else pack_pool_tma<false>(a, pg, sl, tile, grp, head, sm_rp);
    } else {
      if (rope) pack_pool_body<ROPE>(a, pg, sl, tile, grp, head, sm_rp);
      else pack_pool_body<false>(a, pg, sl, tile, grp, head, sm_rp);
    }
  };
  // K tiles, then query tiles (both pool and bound), then V tiles (copy only) last: the
  // launch's last partial wave is then made of the cheapest blocks
  if (b < n_append) {
    const int head = b / fa.n_tiles;
    run(fa.kv, fa.kv_pg, fa.kv_sl, b - head * fa.n_tiles, 0, head, true);
    return;
  }
  b -= n_append;
  const int per_head = fa.q_trows * fa.n_tiles;
  if (b < fa.heads * per_head) {
    const int head = b / per_head, rem = b - head * per_head, qtr = rem / fa.n_tiles;
    run(fa.q, fa.q_pg, fa.q_sl, rem - qtr * fa.n_tiles, qtr, head, true);
    return;
  }
  b -= fa.heads * per_head;
  const int head = b / fa.n_tiles;  // V: never rotated
  run(fa.v, fa.kv_pg, fa.kv_sl, b - head * fa.n_tiles, 0, head, false);
}

inline size_t mask_select_smem(int d, int bnk) {
  return (size_t)d * kFrontQP * 4 + (size_t)kFrontQB * bnk * 4 + (size_t)kFrontQB * 256 * 4;
}

// Coarse scores + top-k of kFrontQB (head, q-block) rows per block.  Thread t owns key blocks
// t, t + 256, ...: it streams the key block's mean (the ring's p0 / p1 row, written by the
// append pass with its non-finite bits) from L2 and runs the kFrontQB query chains on it,
// scalar products and the adds in packed pairs (FADD2; per chain the reference's exact order --
// channels ascending, separate multiply and add from 0.0f, then the 1/sqrt(d) multiply; P/src/tensor.cpp:121-151,
// sparse.cpp:97-99); the pooled queries (S / count, scaled here) sit transposed in shared
// memory, [channel][query slot], so one channel's queries are one broadcast load.  Scores go
// to shared memory; warp r then selects row r (topk_row, radix threshold).
template <int NPER>
__global__ void __launch_bounds__(kFrontThreads) mask_select_kernel(const __grid_constant__ DevGeom g,
                                                                    const __grid_constant__ DevMask m,
                                                                    const __grid_constant__ SelectParams p) {
  static_assert(kFrontQB >= 1 && kFrontQB <= 8 && kFrontQB * 32 <= kFrontThreads, "one warp per row for top-k");
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) float sm_ms[];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int per_head = (g.bnq + kFrontQB - 1) / kFrontQB;
  const int head = blockIdx.x / per_head;
  const int qb0 = (blockIdx.x - head * per_head) * kFrontQB;
  const int nqb = min(kFrontQB, g.bnq - qb0);
  const int d = g.d, d4 = d >> 2, bnk = g.bnk;
  float* qT = sm_ms;                                          // [d][kFrontQP]
  unsigned* hist = reinterpret_cast<unsigned*>(qT + d * kFrontQP);   // [kFrontQB][256] (16 B aligned)
  float* sc = reinterpret_cast<float*>(hist + kFrontQB * 256);         // [kFrontQB][bnk]
  bool fin = true;
  // pooled queries: S1 (two-frame rows) or S0, times 1/count (avg_pool_blocks' final scale)
  for (int idx = tid; idx < kFrontQP * d4; idx += kFrontThreads) {
    const int r = idx / d4, c4 = idx - r * d4;
    float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < nqb) {
      const int qb = qb0 + r, qtr = qb / g.n_tiles, qtile = qb - qtr * g.n_tiles;
      const int qcnt = g.q_tr_count[qtr], qf = g.q_tr_first[qtr] + qcnt - 1;
      const float* src = (qcnt == 2 ? p.q_s1 : p.q_s0) + head * p.q_head_stride + ((long long)qf * g.n_tiles + qtile) * d;
      const float inv = __fdiv_rn(1.0f, (float)(qcnt * tile_h_count(g, qtile) * tile_w_count(g, qtile)));
      w = __ldg(reinterpret_cast<const float4*>(src) + c4);
      w.x = __fmul_rn(w.x, inv);
      w.y = __fmul_rn(w.y, inv);
      w.z = __fmul_rn(w.z, inv);
      w.w = __fmul_rn(w.w, inv);
      fin = fin && isfinite(w.x) && isfinite(w.y) && isfinite(w.z) && isfinite(w.w);
    }
    qT[(4 * c4 + 0) * kFrontQP + r] = w.x;
    qT[(4 * c4 + 1) * kFrontQP + r] = w.y;
    qT[(4 * c4 + 2) * kFrontQP + r] = w.z;
    qT[(4 * c4 + 3) * kFrontQP + r] = w.w;
  }
  __syncthreads();
  // NK key blocks of this thread scored together: one load of each channel's queries serves
  // NK * kFrontQB chains (bnk > 256: 2 keys per pass; the headline's bnk <= 256 has one)
  auto score = [&](auto nk_tag, int kb0) {
    constexpr int NK = decltype(nk_tag)::value;
    constexpr int kBatch = NK == 1 ? 8 : 4;  // channel quads per key in flight per batch
    const float4* kr[NK];
#pragma unroll
    for (int e = 0; e < NK; ++e) {
      const int kb = kb0 + e * kFrontThreads;
      const int ktr = kb / g.n_tiles, ktile = kb - ktr * g.n_tiles;
      const int kcnt = g.k_tr_count[ktr], kf = g.k_tr_first[ktr] + kcnt - 1;
      const long long slot_tile = (long long)g.k_slot[kf] * g.n_tiles + ktile;
      if (p.k_flag[head * p.k_flag_head_stride + slot_tile] & (kcnt == 2 ? 2u : 1u)) fin = false;
      // block mean rows are channel-quad interleaved ([slot][d/4][tile][4]): quad j of this key
      // block is kr[j * n_tiles], and the warp's 32 consecutive key blocks read one 512-byte run
      kr[e] = reinterpret_cast<const float4*>((kcnt == 2 ? p.k_p1 : p.k_p0) + head * p.k_head_stride +
                                              ((long long)g.k_slot[kf] * d4 * g.n_tiles + ktile) * 4);
    }
    const int qs = g.n_tiles;  // float4 stride between channel quads
    float acc[NK][kFrontQP];
#pragma unroll
    for (int e = 0; e < NK; ++e)
#pragma unroll
      for (int r = 0; r < kFrontQP; ++r) acc[e][r] = 0.0f;
    auto channel = [&](const float (&k)[NK], int c) {
      float qv[kFrontQP];
      if constexpr (kFrontQP == 2) {
        const float2 t = *reinterpret_cast<const float2*>(qT + c * kFrontQP);
        qv[0] = t.x;
        qv[1] = t.y;
      } else {
#pragma unroll
        for (int r4 = 0; r4 < kFrontQP; r4 += 4) {
          const float4 t = *reinterpret_cast<const float4*>(qT + c * kFrontQP + r4);
          qv[r4] = t.x;
          qv[r4 + 1] = t.y;
          qv[r4 + 2] = t.z;
          qv[r4 + 3] = t.w;
        }
      }
#pragma unroll
      for (int e = 0; e < NK; ++e) {
#pragma unroll
        for (int r = 0; r + 1 < kFrontQB; r += 2)
          padd_rn(acc[e][r], acc[e][r + 1], __fmul_rn(qv[r], k[e]), __fmul_rn(qv[r + 1], k[e]));
        if constexpr (kFrontQB & 1)
          acc[e][kFrontQB - 1] = __fadd_rn(acc[e][kFrontQB - 1], __fmul_rn(qv[kFrontQB - 1], k[e]));
      }
    };
    // the rows in batches of channel quads, the next batch's loads in flight meanwhile
    float4 cur[NK][kBatch], nxt[NK][kBatch];
#pragma unroll
    for (int e = 0; e < NK; ++e)
#pragma unroll
      for (int j = 0; j < kBatch; ++j) cur[e][j] = __ldg(kr[e] + (long long)j * qs);
#pragma unroll 1
    for (int b = 0; b < d4; b += kBatch) {
#pragma unroll
      for (int e = 0; e < NK; ++e)
#pragma unroll
        for (int j = 0; j < kBatch; ++j)
          nxt[e][j] = b + kBatch + j < d4 ? __ldg(kr[e] + (long long)(b + kBatch + j) * qs) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {  // d4 is 16 or 32: every batch is whole (no branch between quads)
        const int c = 4 * (b + j);
        float kx[NK], ky[NK], kz[NK], kw[NK];
#pragma unroll
        for (int e = 0; e < NK; ++e) {
          kx[e] = cur[e][j].x;
          ky[e] = cur[e][j].y;
          kz[e] = cur[e][j].z;
          kw[e] = cur[e][j].w;
        }
        channel(kx, c);
        channel(ky, c + 1);
        channel(kz, c + 2);
        channel(kw, c + 3);
      }
#pragma unroll
      for (int e = 0; e < NK; ++e)
#pragma unroll
        for (int j = 0; j < kBatch; ++j) cur[e][j] = nxt[e][j];
    }
#pragma unroll
    for (int e = 0; e < NK; ++e)
#pragma unroll
      for (int r = 0; r < kFrontQB; ++r) sc[r * bnk + kb0 + e * kFrontThreads] = __fmul_rn(acc[e][r], p.scale);
  };
  int kb = tid;
  for (; kb + kFrontThreads < bnk; kb += 2 * kFrontThreads) score(std::integral_constant<int, 2>{}, kb);
  if (kb < bnk) score(std::integral_constant<int, 1>{}, kb);
  if (!fin) atomicOr(p.err, kErrShape);
  __syncthreads();
  if (warp < nqb) topk_row<NPER>(g, m, p, qb0 + warp, head, sc + warp * bnk, hist + warp * 256);
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
  pdl_wait();
  pdl_trigger();
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

// ---------------------------------------------------------------------------------------
// per-frame attention mass for scored eviction (frame_attention_mass, P/src/kv_cache.cpp:
// 170-206) from the fp32 coarse scores the selector already wrote, in three small passes
// spread over the whole GPU (one CTA per head measured 66 us; fp64 exp chains are long):
//   frame_mass_rows_kernel   warp per (head, q-block): max over coarse-allowed key blocks,
//                            sum of exp(s - max) in fp64 (rows with no allowed block are
//                            marked and skipped, kv_cache.cpp:179-181);
//   frame_mass_blocks_kernel CTA per (head, 32 key blocks): warp w sums q-blocks w, w+8, ...
//                            of exp(s - max) / denom, then a fixed-order 8-way combine
//                            (deterministic; kv_cache.cpp:184-190);
//   frame_mass_frames_kernel warp per (head, key frame): the mass of every block of its
//                            temporal row, split over member tokens (kv_cache.cpp:193-203).
// Device exp and the summation order differ from the reference in the last ulps (1e-12 rel).
// ---------------------------------------------------------------------------------------
constexpr int kMassThreads = 256;

__global__ void __launch_bounds__(kMassThreads) frame_mass_rows_kernel(const __grid_constant__ DevGeom g,
                                                                       const __grid_constant__ DevMask m,
                                                                       const float* __restrict__ coarse,
                                                                       double* __restrict__ rmax,
                                                                       double* __restrict__ rden, int heads) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * (kMassThreads / 32) + (threadIdx.x >> 5);  // head * bnq + qb
  if (row >= (long long)heads * g.bnq) return;
  const int qb = (int)(row % g.bnq);
  const int qtr = qb / g.n_tiles, qtile = qb - qtr * g.n_tiles;
  const float* sc = coarse + row * g.bnk;
  double mx = -INFINITY;
  for (int kb = lane; kb < g.bnk; kb += 32)
    if (coarse_allowed(g, m, qtr, qtile, kb / g.n_tiles, kb % g.n_tiles)) mx = fmax(mx, (double)sc[kb]);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double den = 0.0;
  if (mx != -INFINITY)
    for (int kb = lane; kb < g.bnk; kb += 32)
      if (coarse_allowed(g, m, qtr, qtile, kb / g.n_tiles, kb % g.n_tiles)) den += exp((double)sc[kb] - mx);
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  if (lane == 0) {
    rmax[row] = mx;
    rden[row] = den;
  }
}

__global__ void __launch_bounds__(kMassThreads) frame_mass_blocks_kernel(const __grid_constant__ DevGeom g,
                                                                         const __grid_constant__ DevMask m,
                                                                         const float* __restrict__ coarse,
                                                                         const double* __restrict__ rmax,
                                                                         const double* __restrict__ rden,
                                                                         double* __restrict__ bmass) {
  pdl_wait();
  pdl_trigger();
  __shared__ double part[kMassThreads / 32][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int head = blockIdx.y;
  const int kb = blockIdx.x * 32 + lane;
  const int ktr = kb / g.n_tiles, ktile = kb - ktr * g.n_tiles;
  const float* sc = coarse + (long long)head * g.bnq * g.bnk;
  double acc = 0.0;
  if (kb < g.bnk)
    for (int qb = warp; qb < g.bnq; qb += kMassThreads / 32) {
      const double mx = rmax[(long long)head * g.bnq + qb];
      if (mx == -INFINITY) continue;
      const int qtr = qb / g.n_tiles, qtile = qb - qtr * g.n_tiles;
      if (coarse_allowed(g, m, qtr, qtile, ktr, ktile))
        acc += exp((double)sc[(long long)qb * g.bnk + kb] - mx) / rden[(long long)head * g.bnq + qb];
    }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && kb < g.bnk) {
    double t = part[0][lane];
#pragma unroll
    for (int w = 1; w < kMassThreads / 32; ++w) t += part[w][lane];
    bmass[(long long)head * g.bnk + kb] = t;
  }
}

__global__ void __launch_bounds__(128) frame_mass_frames_kernel(const __grid_constant__ DevGeom g,
                                                                const double* __restrict__ bmass,
                                                                double* __restrict__ mass, int heads) {
  pdl_wait();
  pdl_trigger();
  // warp per (head, key frame); lanes stride the tiles of the frame's temporal row
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (i >= heads * g.nkf) return;
  const int head = i / g.nkf, f = i - head * g.nkf;
  int tr = 0;
  while (tr + 1 < g.nk_trows && g.k_tr_first[tr + 1] <= f) ++tr;
  const double* bm = bmass + (long long)head * g.bnk + (long long)tr * g.n_tiles;
  double acc = 0.0;
  for (int tile = lane; tile < g.n_tiles; tile += 32) {
    const double b = bm[tile];
    if (b == 0.0) continue;
    const int tok = tile_h_count(g, tile) * tile_w_count(g, tile);
    acc += b / (double)(tok * g.k_tr_count[tr]) * (double)tok;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) mass[i] = acc;
}

// ---------------------------------------------------------------------------------------
// token-mask builders: build_segment_mask / build_causal_mask
// (P/src/mask.cpp:67-101) straight into MaskMatrix words ([L][(L+63)/64] uint64, bit j of
// row i = mask(i, j), P/include/vsr/mask.hpp:16-59).  Byte work, HBM-write bound: the labels
// are staged in shared memory once per CTA; a warp builds 32 consecutive words of a row with
// two ballots per word (lane b tests keys 64w+b and 64w+32+b, conflict-free), keeps word
// w in lane w%32 and stores the 32 words as one coalesced 256 B run.
// kind 0: segment (seg[i] == seg[j]); kind 1: causal (frame[j] <= frame[i] + lookahead).
// ---------------------------------------------------------------------------------------
constexpr int kMaskThreads = 256;

// KIND 0 segment: ballots over the labels.  KIND 1 causal: frames are non-decreasing (host
// checked), so row i's allowed keys are the prefix [0, p) with p = #{j : frame[j] <= frame[i]
// + lookahead} (mask.cpp:96-98); p comes from a binary search in shared memory and every
// word is closed-form (all ones / partial / zero) — pure write bandwidth.
// KIND 2: segment rows — row s of the output is segment s's row (li = s, nrows = #segments);
// token_rows_copy_kernel then gives token i the row of seg[i] (rows of one segment are equal).
template <int KIND>
__global__ void __launch_bounds__(kMaskThreads) token_mask_kernel(const int* __restrict__ labels, int L,
                                                                  int lookahead,
                                                                  unsigned long long* __restrict__ bits,
                                                                  int nrows) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ int tm_lab[];
  for (int j = threadIdx.x; j < L; j += kMaskThreads) tm_lab[j] = labels[j];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int wpr = (L + 63) >> 6;
  // 32-word runs per row; causal rows are one task each (one binary search per row)
  const int groups = KIND == 1 ? 1 : (wpr + 31) >> 5;
  const int total = nrows * groups;
  const int nwarps = gridDim.x * (kMaskThreads / 32);
  for (int task = blockIdx.x * (kMaskThreads / 32) + (threadIdx.x >> 5); task < total; task += nwarps) {
    const int i = task / groups;
    const int w0 = (task - i * groups) << 5;
    unsigned long long mine = 0;
    if constexpr (KIND == 0 || KIND == 2) {
      const int li = KIND == 2 ? i : tm_lab[i];
      const int un = min(32, wpr - w0);
      for (int u = 0; u < un; ++u) {
        const int j0 = ((w0 + u) << 6) + lane, j1 = j0 + 32;
        const unsigned lo = __ballot_sync(0xffffffffu, j0 < L && tm_lab[j0] == li);
        const unsigned hi = __ballot_sync(0xffffffffu, j1 < L && tm_lab[j1] == li);
        if (lane == u) mine = ((unsigned long long)hi << 32) | lo;
      }
    } else {
      const int limit = tm_lab[i] + lookahead;
      int lo = 0, hi = L;  // first j with frame[j] > limit
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (tm_lab[mid] <= limit) lo = mid + 1; else hi = mid;
      }
      for (int w = lane; w < wpr; w += 32) {
        const int b0 = w << 6;
        bits[(long long)i * wpr + w] = lo >= b0 + 64 ? ~0ull : (lo <= b0 ? 0ull : ((1ull << (lo - b0)) - 1ull));
      }
      continue;
    }
    if (w0 + lane < wpr) bits[(long long)i * wpr + w0 + lane] = mine;
  }
}

__global__ void __launch_bounds__(kMaskThreads) token_rows_copy_kernel(const int* __restrict__ seg, int L,
                                                                       const unsigned long long* __restrict__ rows,
                                                                       unsigned long long* __restrict__ bits) {
  pdl_wait();
  pdl_trigger();
  const int wpr = (L + 63) >> 6;
  const long long total = (long long)L * wpr;
  for (long long e = (long long)blockIdx.x * kMaskThreads + threadIdx.x; e < total;
       e += (long long)gridDim.x * kMaskThreads) {
    const int i = (int)(e / wpr), w = (int)(e - (long long)i * wpr);
    bits[e] = rows[(long long)seg[i] * wpr + w];
  }
}

}  // namespace fvsr

namespace fvsr {
// ---------------------------------------------------------------------------------------
// Tile-major attention output ([unit][64 * fpu rows][d], the head-parallel shard layout) ->
// token-major [heads][nq * rows * cols][d].  Unit u = head * (ntr * tiles) + trow * tiles +
// tile; row r of a unit is frame trow * fpu + r / 64, tile row (r % 64) / 8, column r % 8.
// One thread per 16-byte chunk; padding rows of ragged tiles are skipped.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) untile_kernel(const uint16_t* __restrict__ tiles, long long units, int fpu,
                                                     int nq, int rows, int cols, int d,
                                                     uint16_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int tw = (cols + 7) / 8, n_tiles = tw * ((rows + 7) / 8), ntr = nq / fpu;
  const int chunks = d / 8, urows = 64 * fpu;
  const long long total = units * urows * chunks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / chunks;
    const int ch = (int)(i - row * chunks);
    const long long u = row / urows;
    const int r = (int)(row - u * urows);
    const int head = (int)(u / (ntr * n_tiles));
    const int rem = (int)(u - (long long)head * ntr * n_tiles);
    const int trow = rem / n_tiles, tile = rem - trow * n_tiles;
    const int f = trow * fpu + r / 64, rr = r % 64;
    const int h = (tile / tw) * 8 + rr / 8, w = (tile % tw) * 8 + rr % 8;
    if (h >= rows || w >= cols) continue;
    const long long dst = ((long long)(head * nq + f) * rows * cols + (long long)h * cols + w) * d + ch * 8;
    *reinterpret_cast<uint4*>(out + dst) = *reinterpret_cast<const uint4*>(tiles + row * d + ch * 8);
  }
}
}  // namespace fvsr

namespace fvsr {
// ---------------------------------------------------------------------------------------
// rms_norm (P/src/stream.cpp:86-99): y = x * 1/sqrt(mean(x^2) + 1e-6) * gain, one warp per
// token row: fp32 residual stream in, bf16 out (the projection GEMMs' operand).  The sum of
// squares is an fp32 warp tree (the reference sums in double; the difference is far below
// the bf16 rounding of y).
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) rms_norm_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                                                       long long n, int D, uint16_t* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const long long row = blockIdx.x * 8ll + (threadIdx.x >> 5);
  if (row >= n) return;
  const float4* xr = reinterpret_cast<const float4*>(x + row * D);
  float acc = 0.0f;
  for (int c = lane; c < D / 4; c += 32) {
    const float4 v = xr[c];
    acc = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, acc))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  const float inv = (float)(1.0 / sqrt((double)acc / (double)D + 1e-6));
  const float4* gr = reinterpret_cast<const float4*>(gain);
  uint2* yr = reinterpret_cast<uint2*>(y + row * D);
  for (int c = lane; c < D / 4; c += 32) {
    const float4 v = xr[c], g = gr[c];
    const __nv_bfloat162 a = __floats2bfloat162_rn(v.x * inv * g.x, v.y * inv * g.y);
    const __nv_bfloat162 b = __floats2bfloat162_rn(v.z * inv * g.z, v.w * inv * g.w);
    uint2 w;
    w.x = *reinterpret_cast<const uint32_t*>(&a);
    w.y = *reinterpret_cast<const uint32_t*>(&b);
    yr[c] = w;
  }
}
}  // namespace fvsr

/*
 * fvsr_b200.h — C-ABI of the B200-native FlashVSR block-sparse streaming attention.
 *
 * This is the drop-in boundary for the reference's hot-path operator API
 * (P = /root/reference/proj):
 *
 *   fvsr_plan_sparse            replaces vsr::plan_sparse            P/include/vsr/sparse.hpp:45-52
 *                                                                     (P/src/sparse.cpp:72-139)
 *   fvsr_sparse_attention_exec  replaces vsr::sparse_attention_exec  P/include/vsr/sparse.hpp:59-64
 *                                                                     (P/src/sparse.cpp:208-254)
 *   fvsr_sparsity_report        replaces vsr::sparsity_report        P/include/vsr/sparse.hpp:66
 *   fvsr_ring_*                 replace vsr::KVCache append / sliding evict / frames and the
 *                               per-step concat_rows context assembly
 *                               P/include/vsr/kv_cache.hpp:27-73, P/src/kv_cache.cpp:39-106,
 *                               P/src/stream.cpp:154-164,244-249
 *   fvsr_ring_attention         replaces head_attention for every head of one layer
 *                               P/src/stream.cpp:175-194 (called at :251)
 *
 * Conventions
 *   - Plain pointers and sizes only.  Tensors are bf16 bit patterns (uint16_t) in DEVICE
 *     memory unless a name ends in _host.  Token order is the reference's TokenGrid order:
 *     frame-major, then row-major inside a frame (P/include/vsr/grid.hpp:17-20).
 *   - Multi-head tensors are head-major: q is [heads][Lq][d], k/v are [heads][Lk][d].
 *   - Every call is stream-ordered on the cudaStream_t passed in (NULL = legacy default
 *     stream) and never allocates device memory once the context's workspace has grown to
 *     the largest shape seen.  Different streams are independent, which replaces the
 *     reference's `threads` argument (P/src/sparse.cpp:229-253).
 *   - Errors: every entry point returns an fvsr_status.  Host-detectable contract
 *     violations are returned immediately, mirroring the reference's VSR_REQUIRE checks
 *     (same exception taxonomy, P/include/vsr/common.hpp:10-48).  Data-dependent errors
 *     found on the device (non-finite pooled values -> SHAPE, a softmax row with no
 *     reachable key -> DEGENERATE) are latched in the context's device error word and
 *     reported by fvsr_check_errors() (which synchronizes the stream), or immediately by
 *     any call made with FVSR_FLAG_SYNC_CHECK.
 *   - fvsr_last_error() returns a thread-local message for the last failing call.
 *   - There is no CPU fallback: without a usable sm_100 device every compute entry point
 *     returns FVSR_E_CUDA.
 */
#ifndef FVSR_B200_H
#define FVSR_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FVSR_API __attribute__((visibility("default")))
#else
#define FVSR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define FVSR_ABI_VERSION 1

typedef struct CUstream_st* fvsr_stream_t; /* == cudaStream_t */

typedef enum {
  FVSR_OK = 0,
  FVSR_E_SHAPE = 1,       /* vsr::ShapeError */
  FVSR_E_CONFIG = 2,      /* vsr::ConfigError */
  FVSR_E_DEGENERATE = 3,  /* vsr::DegenerateRowError */
  FVSR_E_EMPTY_BLOCK = 4, /* vsr::EmptyBlockError */
  FVSR_E_INVARIANT = 5,   /* vsr::InvariantError */
  FVSR_E_CUDA = 6,        /* CUDA runtime / no sm_100 device */
  FVSR_E_NOMEM = 8        /* device allocation failed */
} fvsr_status;

/* Token grid: absolute, strictly increasing frame ids (HOST array) over rows x cols.
 * == vsr::TokenGrid (P/include/vsr/grid.hpp:22-46). */
typedef struct {
  const int32_t* frame_ids;
  int32_t n_frames;
  int32_t rows;
  int32_t cols;
} fvsr_grid;

typedef enum {
  FVSR_MASK_ALL = 0,      /* MaskMatrix::all_allowed (P/include/vsr/mask.hpp:21-23) */
  FVSR_MASK_LOCALITY = 1, /* build_locality_mask, analytic on device (P/src/mask.cpp:109-147) */
  FVSR_MASK_BITMASK = 2   /* explicit MaskMatrix words, DEVICE pointer [Lq][words_per_row] */
} fvsr_mask_kind;

typedef enum {
  FVSR_LOCALITY_PRESERVED = 0, /* LocalityWindow::Mode::boundary_preserved */
  FVSR_LOCALITY_TRUNCATED = 1  /* LocalityWindow::Mode::boundary_truncated */
} fvsr_locality_mode;

/* Token mask descriptor == vsr::MaskMatrix / vsr::LocalityWindow (P/include/vsr/mask.hpp:16-97).
 * Locality frame extents are the grid's rows/cols (make_stream_locality, P/src/stream.cpp). */
typedef struct {
  int32_t kind;
  int32_t mode;
  int32_t extent_h;
  int32_t extent_w;
  const uint64_t* bits;  /* FVSR_MASK_BITMASK only */
  int64_t words_per_row; /* FVSR_MASK_BITMASK only: (Lk + 63) / 64 */
} fvsr_mask;

/* FVSR_FLAG_SYNC_CHECK: synchronize and check the device error word after every call.
 * FVSR_FLAG_NO_TMA: stage the ring append / query pack with 1-D bulk copies instead of
 * tensor-map TMA (the fallback when the driver's tensor-map entry point is unavailable). */
enum { FVSR_FLAG_SYNC_CHECK = 1, FVSR_FLAG_NO_TMA = 2 };

/* Output layouts of fvsr_ring_attention. */
enum {
  FVSR_OUT_TOKEN_MAJOR = 0, /* [heads][Lq][d] in TokenGrid order */
  FVSR_OUT_TILE_MAJOR = 1   /* [unit - unit_begin][64][d], one 8x8 query tile per unit (padding rows
                               included): each rank's shard is contiguous for the NCCL all-gather */
};

/* Eviction strategies == vsr::EvictStrategy (P/include/vsr/kv_cache.hpp:12). */
enum { FVSR_EVICT_SLIDING = 0, FVSR_EVICT_UNIFORM = 1, FVSR_EVICT_HEAD_WISE = 2 };

/* Kernel classes timed by fvsr_ctx_timing_enable.  A ring step's front (FVSR_TIME_FRONT) is
 * also split into its two launches: FVSR_TIME_PACK (ring append + query pack) and
 * FVSR_TIME_SELECT (coarse scores + top-k). */
enum {
  FVSR_TIME_APPEND = 0,
  FVSR_TIME_MASK_BUILDER = 1,
  FVSR_TIME_ATTENTION = 2,
  FVSR_TIME_FRONT = 3,
  FVSR_TIME_PACK = 4,
  FVSR_TIME_SELECT = 5
};

typedef struct fvsr_ctx fvsr_ctx;
typedef struct fvsr_ring fvsr_ring;

/* ---- library / context ------------------------------------------------------------- */
FVSR_API int32_t fvsr_abi_version(void);
/* Experiment macros the library was built with ("" for the product build). */
FVSR_API const char* fvsr_build_flags(void);
FVSR_API const char* fvsr_last_error(void);
/* Binds to the current CUDA device; fails with FVSR_E_CUDA unless it is sm_100. */
FVSR_API int32_t fvsr_ctx_create(fvsr_ctx** out);
FVSR_API void fvsr_ctx_destroy(fvsr_ctx* ctx);
/* Call flags (FVSR_FLAG_*) applied to every later call on this context. */
FVSR_API int32_t fvsr_ctx_set_flags(fvsr_ctx* ctx, int32_t flags);
/* Synchronizes `stream`, reads and clears the device error word. */
FVSR_API int32_t fvsr_check_errors(fvsr_ctx* ctx, fvsr_stream_t stream);
/* Number of kernel launches this context has issued (instrumentation for benches). */
FVSR_API int64_t fvsr_ctx_launch_count(const fvsr_ctx* ctx);
/* When enabled, every append / mask-builder / attention call records a CUDA-event span on
 * its own stream; fvsr_ctx_timing_read synchronizes the device and returns the summed
 * milliseconds and span count of one class (FVSR_TIME_*), optionally clearing all spans. */
FVSR_API int32_t fvsr_ctx_timing_enable(fvsr_ctx* ctx, int32_t enable);
FVSR_API int32_t fvsr_ctx_timing_read(fvsr_ctx* ctx, int32_t kind, double* total_ms, int64_t* count,
                                      int32_t clear);
/* Executed (mask-allowed, selected-block) token pairs counted by the attention kernel since
 * the last read — the reference's sparsity_report definition; synchronizes and resets. */
FVSR_API int32_t fvsr_ctx_read_pairs(fvsr_ctx* ctx, uint64_t* executed_pairs);
/* Key tiles the attention kernel issued since the last read (and how many of them carried
 * 128 key rows: two-frame blocks or two paired single-frame blocks); resets the counters.
 * Tile-level tensor work = tiles x (QK^T 2*128*NQ*d) + PV over the valid key rows. */
FVSR_API int32_t fvsr_ctx_read_tiles(fvsr_ctx* ctx, uint64_t* tiles, uint64_t* full_tiles);

/* ---- geometry (host only) ----------------------------------------------------------- */
/* Block counts of partition_blocks(grid_q) / partition_blocks(grid_k) (P/src/partition.cpp:38-62). */
FVSR_API int32_t fvsr_block_counts(const fvsr_grid* grid_q, const fvsr_grid* grid_k, int32_t* bnq,
                          int32_t* bnk);

/* ---- drop-in operator API (flat device tensors) ------------------------------------- */
/* plan_sparse: per head, pool q/k per (2,8,8) block in exact sequential fp32, score block
 * pairs (sequential dot, no FMA, x 1/sqrt(d)), restrict to coarse-allowed pairs, keep the
 * top-k with the forced diagonal (ties toward the lower id).  Outputs (DEVICE):
 *   sel       [heads][bnq][cap]  ascending key-block ids, -1 padded; cap >= min(topk, bnk)
 *   sel_count [heads][bnq]
 *   diag      [heads][bnq]       diagonal block or -1 (SparsePlan::diagonal_block)
 *   coarse    [heads][bnq][bnk]  fp32 coarse scores (SparsePlan::coarse_scores) or NULL
 *   allowed   [heads][bnq][bnk]  uint8 coarse-allowed (SparsePlan::coarse_allowed) or NULL
 * Indices are bit-exact with the reference for identical (bf16-representable) inputs. */
FVSR_API int32_t fvsr_plan_sparse(fvsr_ctx* ctx, const uint16_t* q, const uint16_t* k, int32_t heads,
                         int32_t d, const fvsr_grid* grid_q, const fvsr_grid* grid_k,
                         const fvsr_mask* mask, int64_t topk, int32_t cap, int32_t* sel,
                         int32_t* sel_count, int32_t* diag, float* coarse, uint8_t* allowed,
                         fvsr_stream_t stream);

/* fvsr_plan_sparse on fp32 inputs (q, k: DEVICE fp32 [heads][L][d]): the reference's own
 * inputs, pooled exactly as avg_pool_blocks does, so the plan (indices, coarse scores) is
 * bit-exact with vsr::plan_sparse on ANY fp32 data (the C++ drop-in layer plans this way). */
FVSR_API int32_t fvsr_plan_sparse_f32(fvsr_ctx* ctx, const float* q, const float* k, int32_t heads,
                         int32_t d, const fvsr_grid* grid_q, const fvsr_grid* grid_k,
                         const fvsr_mask* mask, int64_t topk, int32_t cap, int32_t* sel,
                         int32_t* sel_count, int32_t* diag, float* coarse, uint8_t* allowed,
                         fvsr_stream_t stream);

/* sparse_attention_exec: exact softmax attention restricted to each query block's
 * selected key blocks and the token mask, tcgen05 tensor cores, fp32 online softmax,
 * bf16 out [heads][Lq][d].  Rows outside [row_begin, row_end) are written as zeros
 * (row_end < 0 means "to the end").  d must be 64 or 128. */
FVSR_API int32_t fvsr_sparse_attention_exec(fvsr_ctx* ctx, const uint16_t* q, const uint16_t* k,
                                   const uint16_t* v, int32_t heads, int32_t d,
                                   const fvsr_grid* grid_q, const fvsr_grid* grid_k,
                                   const fvsr_mask* mask, int32_t cap, const int32_t* sel,
                                   const int32_t* sel_count, float scale, int64_t row_begin,
                                   int64_t row_end, uint16_t* out, fvsr_stream_t stream);

/* sparsity_report: per head (DEVICE outputs, uint64 [heads]) executed token pairs, dense
 * (mask-allowed) token pairs, selected and coarse-allowed block pairs.  executed_flops of
 * the reference == executed_pairs * (2d+2) (P/src/sparse.cpp:268-281). */
FVSR_API int32_t fvsr_sparsity_report(fvsr_ctx* ctx, int32_t heads, const fvsr_grid* grid_q,
                             const fvsr_grid* grid_k, const fvsr_mask* mask, int32_t cap,
                             const int32_t* sel, const int32_t* sel_count,
                             uint64_t* executed_pairs, uint64_t* dense_pairs,
                             uint64_t* selected_blocks, uint64_t* allowed_blocks,
                             fvsr_stream_t stream);

/* ---- token-mask builders (DEVICE MaskMatrix words for FVSR_MASK_BITMASK) -------------- */
/* build_segment_mask (P/src/mask.cpp:67-84): bits [L][(L+63)/64] (DEVICE), allowed iff
 * seg[i] == seg[j].  seg: HOST [L]; ids must be >= 0 and contiguous (FVSR_E_CONFIG). */
FVSR_API int32_t fvsr_build_segment_mask(fvsr_ctx* ctx, const int32_t* seg, int64_t L, uint64_t* bits,
                                fvsr_stream_t stream);
/* build_causal_mask (P/src/mask.cpp:86-101): allowed iff frame[j] <= frame[i] + lookahead.
 * frame: HOST [L], non-decreasing; lookahead >= 0 (FVSR_E_CONFIG otherwise). */
FVSR_API int32_t fvsr_build_causal_mask(fvsr_ctx* ctx, const int32_t* frame, int64_t L, int32_t lookahead,
                               uint64_t* bits, fvsr_stream_t stream);

/* ---- device ring-buffer KV cache (streaming) ---------------------------------------- */
/* window_frames + 1 slots per (layer, head): the current frame is appended before
 * attention, exactly as step() does (P/src/stream.cpp:228-229; KVCache::validate allows
 * window + 1, P/src/kv_cache.cpp:144).  K/V live tile-major and pre-swizzled for the
 * tensor-core kernel; per-frame-tile pooled partial sums are kept so the mask builder never
 * re-reads cached keys. */
FVSR_API int32_t fvsr_ring_create(fvsr_ctx* ctx, int32_t layers, int32_t heads, int32_t d, int32_t rows,
                         int32_t cols, int32_t window_frames, fvsr_ring** out);
FVSR_API void fvsr_ring_destroy(fvsr_ring* ring);
/* KVCache::append for every head of `layer`: k, v are [heads][rows*cols][d] (DEVICE). */
FVSR_API int32_t fvsr_ring_append(fvsr_ctx* ctx, fvsr_ring* ring, int32_t layer, int32_t frame_id,
                         const uint16_t* k, const uint16_t* v, fvsr_stream_t stream);
/* Fused RoPE: from now on fvsr_ring_append rotates K and fvsr_ring_attention
 * rotates Q at their absolute (frame, row, col) positions inside the pack/pool pass, before
 * pooling and the tensor-core layout — apply_rope (P/src/rope.cpp:30-62) as make_frame_kv /
 * step call it (P/src/stream.cpp:134-152, 240), without an HBM round trip.  Inputs are then
 * the un-rotated projections.  theta0 > 1; axis_split = channels for (t, h, w), positive,
 * even, summing to d (NULL = RopeConfig::split_default: d/2, d/4, d/4).  Rotation is fp32
 * without FMA from the reference's float-rounded double cos/sin, then bf16 RNE: bit-exact
 * with bf16(apply_rope(x)).  At most 4 query frames per fvsr_ring_attention call. */
FVSR_API int32_t fvsr_ring_set_rope(fvsr_ring* ring, double theta0, const int32_t* axis_split);
/* KVCache::evict with the sliding_window strategy (P/src/kv_cache.cpp:100-106). */
FVSR_API int32_t fvsr_ring_evict_sliding(fvsr_ring* ring, int32_t layer);
/* Sliding eviction down to `keep` frames (oldest first).  Chunked streaming of Tq frames per
 * step (the paper's 2-latent chunks) creates the ring with window_frames = W + Tq - 1 and
 * calls this with keep = W before appending each chunk. */
FVSR_API int32_t fvsr_ring_evict_keep(fvsr_ring* ring, int32_t layer, int32_t keep);
/* KVCache::frame_ids (identical for every head under sliding eviction). */
FVSR_API int32_t fvsr_ring_frame_ids(const fvsr_ring* ring, int32_t layer, int32_t* ids, int32_t cap,
                            int32_t* n);
/* The frame ids head `head` of `layer` retains (head-wise eviction lets heads diverge;
 * fvsr_ring_frame_ids reports head 0). */
FVSR_API int32_t fvsr_ring_frame_ids_head(const fvsr_ring* ring, int32_t layer, int32_t head, int32_t* ids,
                                          int32_t cap, int32_t* n);

/* head_attention for heads [0, heads) of `layer`: queries of frames q_frame_ids (usually
 * the current frame) against the ring's context.  q is [heads][nq*rows*cols][d] (DEVICE),
 * out likewise.  sel/sel_count (DEVICE, optional) receive the plan as fvsr_plan_sparse would.
 * unit_begin/unit_end restrict the work to a range of (head, q-tile) units, unit =
 * head * (nq * tiles) + frame * tiles + tile (head-parallel sharding; pass 0, -1 for all);
 * rows of units outside the range are left untouched.  out_layout: FVSR_OUT_*. */
FVSR_API int32_t fvsr_ring_attention(fvsr_ctx* ctx, fvsr_ring* ring, int32_t layer, const uint16_t* q,
                            const int32_t* q_frame_ids, int32_t nq, const fvsr_mask* mask,
                            int64_t topk, float scale, int64_t unit_begin, int64_t unit_end,
                            uint16_t* out, int32_t out_layout, int32_t sel_cap, int32_t* sel,
                            int32_t* sel_count, fvsr_stream_t stream);

/* One streaming layer-step of step() (P/src/stream.cpp:228-256) on device: KVCache::append of
 * frame `frame_id`'s K/V (k, v: [heads][rows*cols][d] bf16, as fvsr_ring_append) followed by
 * head_attention for the query frames (as fvsr_ring_attention, whose arguments these are).
 * The append and the query pack + pool share one kernel launch (independent inputs, one pass
 * over HBM), coarse scores + top-k a second, then the sparse attention kernel: three launches
 * per layer-step.  The ring keeps the new frame; evict afterwards as with fvsr_ring_append. */
FVSR_API int32_t fvsr_ring_step(fvsr_ctx* ctx, fvsr_ring* ring, int32_t layer, int32_t frame_id, const uint16_t* k,
                                const uint16_t* v, const uint16_t* q, const int32_t* q_frame_ids, int32_t nq,
                                const fvsr_mask* mask, int64_t topk, float scale, int64_t unit_begin,
                                int64_t unit_end, uint16_t* out, int32_t out_layout, int32_t sel_cap, int32_t* sel,
                                int32_t* sel_count, fvsr_stream_t stream);

/* Strided tensor layout in elements: head h, token t of a tensor starts at
 * h * head_stride + t * token_stride.  {0, 0} = [heads][tokens][d] (head_stride = tokens * d,
 * token_stride = d); {d, heads * d} reads / writes a projection GEMM's [tokens][heads * d]
 * matrix in place (no per-head split or transpose pass).  Strides are multiples of 8. */
typedef struct {
  int64_t head_stride;
  int64_t token_stride;
} fvsr_layout;

/* fvsr_ring_step with strided K/V, Q and output layouts (token-major output, all units):
 * the DiT block's K/V projection [tokens][2 * heads * d] feeds the ring append directly
 * (make_frame_kv's per-head slice_cols + apply_rope, P/src/stream.cpp:134-152, fused into
 * the append's gather), Q likewise, and the attention writes [tokens][heads * d] for the
 * output projection (P/src/stream.cpp:252-259). */
FVSR_API int32_t fvsr_ring_step_layout(fvsr_ctx* ctx, fvsr_ring* ring, int32_t layer, int32_t frame_id,
                                       const uint16_t* k, const uint16_t* v, fvsr_layout kv_layout, const uint16_t* q,
                                       fvsr_layout q_layout, const int32_t* q_frame_ids, int32_t nq,
                                       const fvsr_mask* mask, int64_t topk, float scale, uint16_t* out,
                                       fvsr_layout out_layout, fvsr_stream_t stream);

/* ---- scored eviction ------------------------------------------------- */
/* frame_attention_mass (P/src/kv_cache.cpp:170-206; declared P/include/vsr/kv_cache.hpp:79):
 * per head and key frame (grid_k order), the coarse-score softmax mass of every q-block
 * (fp64, coarse-allowed blocks only) summed into key blocks and split over their member
 * tokens' frames.  coarse: DEVICE fp32 [heads][bnq][bnk] (fvsr_plan_sparse's output);
 * mass: DEVICE double [heads][grid_k->n_frames].  Within 1e-12 relative of the reference
 * (device exp and reduction order differ in the last ulps). */
FVSR_API int32_t fvsr_frame_attention_mass(fvsr_ctx* ctx, int32_t heads, const fvsr_grid* grid_q,
                                  const fvsr_grid* grid_k, const fvsr_mask* mask,
                                  const float* coarse, double* mass, fvsr_stream_t stream);
/* The same for the plan of the preceding fvsr_ring_attention on this ctx (same layer, same
 * q frames and mask, stream order; call before evicting): head_attention's frame_scores
 * (P/src/stream.cpp:190).  mass: DEVICE double [heads][n] aligned with fvsr_ring_frame_ids. */
FVSR_API int32_t fvsr_ring_frame_mass(fvsr_ctx* ctx, fvsr_ring* ring, int32_t layer,
                             const int32_t* q_frame_ids, int32_t nq, const fvsr_mask* mask,
                             double* mass, fvsr_stream_t stream);
/* KVCache::evict (P/src/kv_cache.cpp:97-137): FVSR_EVICT_SLIDING ignores scores;
 * FVSR_EVICT_UNIFORM sums HOST scores [heads][n] (aligned with fvsr_ring_frame_ids) over heads
 * and drops the lowest-scored non-newest frames (older first on ties) from every head.
 * FVSR_EVICT_HEAD_WISE drops each head's own lowest-scored frames, so the heads' retained sets
 * may diverge (each (layer, head) has its own frame table; later steps run one launch per run
 * of heads with identical sets).  FVSR_EVICT_UNIFORM on diverged sets: FVSR_E_INVARIANT
 * (kv_cache.cpp:119-122).  NULL scores while over budget on a scored strategy: FVSR_E_CONFIG
 * (kv_cache.cpp:112-113). */
FVSR_API int32_t fvsr_ring_evict(fvsr_ring* ring, int32_t layer, int32_t strategy, const double* scores);

/* rms_norm (P/src/stream.cpp:86-99) of the DiT block: x fp32 [n][D] (DEVICE), gain fp32 [D],
 * y = x / sqrt(mean(x^2) + 1e-6) * gain as bf16 [n][D] (the projection GEMMs' operand). */
FVSR_API int32_t fvsr_rms_norm(fvsr_ctx* ctx, const float* x, const float* gain, int64_t n, int32_t D, uint16_t* y,
                               fvsr_stream_t stream);

/* Tile-major attention output -> token-major (the head-parallel gather's last step):
 * tiles [units][64 * frames_per_unit][d] bf16 (FVSR_OUT_TILE_MAJOR, unit = head * (nq /
 * frames_per_unit * tiles) + temporal row * tiles + tile) -> out [heads][nq * rows * cols][d];
 * frames_per_unit 2 for paired query frames (2m, 2m+1).  DEVICE buffers, 16-byte aligned. */
FVSR_API int32_t fvsr_untile(fvsr_ctx* ctx, const uint16_t* tiles, int64_t units, int32_t frames_per_unit, int32_t nq,
                             int32_t rows, int32_t cols, int32_t d, uint16_t* out, fvsr_stream_t stream);

/* One streaming layer-step from HOST buffers (the end-to-end path): H2D copy of the new
 * frame's q/k/v ([heads][rows*cols][d] bf16; pinned memory recommended), ring append,
 * sliding evict, attention, D2H copy of out.  Returns after enqueueing; the host output is
 * valid once `stream` is synchronized. */
FVSR_API int32_t fvsr_ring_step_host(fvsr_ctx* ctx, fvsr_ring* ring, int32_t layer, int32_t frame_id,
                            const uint16_t* q_host, const uint16_t* k_host,
                            const uint16_t* v_host, const fvsr_mask* mask, int64_t topk,
                            float scale, uint16_t* out_host, fvsr_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FVSR_B200_H */

/* TEST INFRASTRUCTURE ONLY — CPU oracle for the FlashVSR block-sparse hot path.
 *
 * Plain-C restatement of the reference algorithm (P = /root/reference/proj):
 *   fp_partition   <- partition_blocks        P/src/partition.cpp:38-62
 *   fp_plan        <- plan_sparse             P/src/sparse.cpp:72-133
 *                     avg_pool_blocks         P/src/tensor.cpp:161-186
 *                     matmul (+ finite check) P/src/tensor.cpp:121-151
 *                     coarse_allowed_mask     P/src/sparse.cpp:47-70
 *                     build_locality_mask     P/src/mask.cpp:109-147
 *   fp_exec        <- exec_block_range        P/src/sparse.cpp:141-206
 *                     sparse_attention_exec   P/src/sparse.cpp:208-254
 *   fp_report      <- sparsity_report         P/src/sparse.cpp:256-285
 * Pinned against the compiled reference (oracle/_ref) and the committed golden
 * fixtures in tests/golden/ (see tests/test_oracle.py).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 */
#ifndef FVSR_PORT_H
#define FVSR_PORT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error taxonomy of P/include/vsr/common.hpp:10-48 */
enum { FP_OK = 0, FP_SHAPE = 1, FP_CONFIG = 2, FP_DEGENERATE = 3, FP_EMPTY_BLOCK = 4,
       FP_INVARIANT = 5, FP_NOMEM = 8 };

typedef struct { /* TokenGrid, P/include/vsr/grid.hpp:22-46 */
  const int* frame_ids;
  int n_frames;
  int rows;
  int cols;
} fp_grid;

typedef struct { /* MaskMatrix::all_allowed | LocalityWindow | explicit bits */
  int kind;      /* 0 all-allowed, 1 locality window, 2 bitmask */
  int mode;      /* 0 boundary_preserved, 1 boundary_truncated */
  int extent_h;
  int extent_w;
  const uint64_t* bits; /* kind 2: [Lq][words_per_row] */
  long words_per_row;
} fp_mask;

/* vsr::Rng(seed) gaussian_f stream (P/include/vsr/rng.hpp:12-53): mt19937_64 plus the
 * explicit Box-Muller pair, n draws in TensorF32::gaussian order (tensor.cpp:39-43). */
void fp_gaussian(uint64_t seed, float* out, long n);

/* Block count of partition_blocks(grid). */
int fp_block_count(const fp_grid* g, int* nblocks);

/* assignment[L] (token -> block id), keys[nblocks][3] = (t_row, h_tile, w_tile). */
int fp_partition(const fp_grid* g, int* assignment, int* keys, int* nblocks);

/* plan_sparse.  sel is [bnq][cap] ascending, -1 padded; coarse [bnq][bnk] (may be
 * NULL); allowed [bnq][bnk] (may be NULL). */
int fp_plan(const float* q, const float* k, int d, const fp_grid* gq, const fp_grid* gk,
            const fp_mask* m, long topk, int cap, int* sel, int* sel_count, int* diag,
            float* coarse, uint8_t* allowed);

/* sparse_attention_exec with threads = 1.  row_end < 0 means SIZE_MAX. */
int fp_exec(const float* q, const float* k, const float* v, int d, const fp_grid* gq,
            const fp_grid* gk, const fp_mask* m, int cap, const int* sel,
            const int* sel_count, float scale, long row_begin, long row_end, float* out);

/* sparsity_report: executed and dense token pairs, selected/allowed block pairs. */
int fp_report(const fp_grid* gq, const fp_grid* gk, const fp_mask* m, int cap,
              const int* sel, const int* sel_count, uint64_t* executed_pairs,
              uint64_t* dense_pairs, uint64_t* selected_blocks, uint64_t* allowed_blocks);

#ifdef __cplusplus
}
#endif
#endif

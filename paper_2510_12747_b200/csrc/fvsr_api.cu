// fvsr_api.cu — host implementation of the C-ABI declared in include/fvsr_b200.h.
//
// One translation unit: the kernels are included below so the library builds with a
// single nvcc invocation and no relocatable device code.  Host checks mirror the
// reference's VSR_REQUIRE contracts (P = /root/reference/proj) and return the same
// exception taxonomy as status codes.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fvsr_b200.h"
#include "fvsr_common.cuh"
#include "kernel_attn.cu"
#include "kernels_plan.cu"

using namespace fvsr;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define FVSR_CUDA(call)                                                                     \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) return fail(FVSR_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define FVSR_TRY(expr)          \
  do {                          \
    int st_ = (expr);           \
    if (st_ != FVSR_OK) return st_; \
  } while (0)

int status_from_bits(unsigned bits) {
  for (int code = 1; code < 8; ++code)
    if (bits & (1u << code)) return code;
  return FVSR_OK;
}

const char* device_error_message(int code) {
  switch (code) {
    case FVSR_E_SHAPE: return "non-finite pooled value in plan_sparse (matmul finite check, P/src/tensor.cpp:126-127)";
    case FVSR_E_DEGENERATE: return "sparse_attention_exec: a query row has no allowed keys in its selected blocks";
    case FVSR_E_INVARIANT: return "selection list out of range or longer than cap";
    default: return "device error";
  }
}

}  // namespace

struct fvsr_ctx {
  int device = 0;
  int flags = 0;
  unsigned* d_err = nullptr;
  unsigned long long* d_pairs = nullptr;  // executed token pairs, accumulated by the attention kernel
  unsigned long long* d_tiles = nullptr;  // [2] key tiles issued / of them with 128 key rows
  // optional CUDA-event spans per kernel class (fvsr_ctx_timing_enable)
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Span { cudaEvent_t a, b; int kind; };
  std::vector<Span> spans;
  long long launches = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // staging for fvsr_ring_step_host
  void* stage = nullptr;
  size_t stage_bytes = 0;
  // coarse block scores for the top-k pass (plan / ring attention without a user buffer)
  float* d_scores = nullptr;
  size_t scores_cap = 0;
  // shape of the scores the last two-kernel selection left in d_scores (fvsr_ring_frame_mass)
  int scores_heads = 0, scores_bnq = 0, scores_bnk = 0;
  // the last ring step's runs of heads with identical frame tables and their score slices
  struct ScoreRun {
    int h0, h1, bnq, bnk;
    size_t off;  // floats into d_scores
  };
  std::vector<ScoreRun> score_runs;
  // which ring attention call produced d_scores (fvsr_ring_frame_mass refuses any other):
  // ring, layer, the layer's frame-set generation, query frame ids and the mask descriptor
  struct ScoreStamp {
    const void* ring = nullptr;
    int layer = -1;
    unsigned long long gen = 0;
    std::vector<int> qids;
    fvsr_mask mask{};
    bool operator==(const ScoreStamp& o) const {
      const bool both_all = mask.kind == FVSR_MASK_ALL && o.mask.kind == FVSR_MASK_ALL;
      return ring == o.ring && layer == o.layer && gen == o.gen && qids == o.qids &&
             (both_all || (mask.kind == o.mask.kind && mask.mode == o.mask.mode && mask.extent_h == o.mask.extent_h && mask.extent_w == o.mask.extent_w &&
             mask.bits == o.mask.bits && mask.words_per_row == o.mask.words_per_row));
    }
  } stamp;
  // fp64 scratch of the frame-mass passes
  double* d_mass_scratch = nullptr;
  size_t mass_scratch_cap = 0;
};

struct fvsr_ring {
  int layers, heads, d, rows, cols, window, slots, tiles_w, tiles_h, n_tiles;
  size_t tile_bytes;
  uint8_t* k = nullptr;
  uint8_t* v = nullptr;
  float* s0 = nullptr;
  float* s1 = nullptr;
  float* kn2 = nullptr;  // max squared key-row norm per (layer, head, slot, tile)
  float* p0 = nullptr;   // block means S0 / count, S1 / count (the mask builder's pooled keys)
  float* p1 = nullptr;
  unsigned* kfl = nullptr;  // per (layer, head, slot, tile): non-finite bits of p0 / p1
  // fused RoPE (fvsr_ring_set_rope): device (cos, sin) tables per axis position
  bool rope = false;
  double rope_theta0 = 10000.0;
  int rope_split[3] = {0, 0, 0};
  float2* rope_t = nullptr;  // [rope_t_cap][split0/2]
  float2* rope_h = nullptr;  // [rows][split1/2]
  float2* rope_w = nullptr;  // [cols][split2/2]
  int rope_t_cap = 0;
  // Frame tables.  KVCache keeps one list of frames per (layer, head) (P/include/vsr/
  // kv_cache.hpp:72); head-wise eviction lets the heads of a layer diverge.  The owning ring
  // keeps htab/hused per (layer, head); every operation runs on VIEWS, one per run of
  // consecutive heads with identical tables (one view for all heads unless they diverged):
  // a view is a shallow copy whose heads are [head0, head0 + heads) of the heads_total
  // stored heads and whose ctx[layer] / used[layer] are the run's table.
  using Table = std::vector<std::pair<int, int>>;     // (frame_id, slot), ascending ids
  std::vector<std::vector<Table>> htab;               // owning ring: [layer][head]
  std::vector<std::vector<std::vector<char>>> hused;  // owning ring: [layer][head][slot] occupancy
  std::vector<Table> ctx;                             // view: [layer] the run's table
  std::vector<std::vector<char>> used;                // view: [layer] the run's slot occupancy
  std::vector<unsigned long long> gen;                // per layer: bumped on every append / evict
  int head0 = 0, heads_total = 0;
  long long kv_head_stride() const { return (long long)slots * n_tiles * (long long)tile_bytes; }
  long long part_head_stride() const { return (long long)slots * n_tiles * d; }
  long long hbase(int l) const { return (long long)l * heads_total + head0; }
  uint8_t* k_layer(int l) const { return k + hbase(l) * kv_head_stride(); }
  uint8_t* v_layer(int l) const { return v + hbase(l) * kv_head_stride(); }
  float* s0_layer(int l) const { return s0 + hbase(l) * part_head_stride(); }
  float* s1_layer(int l) const { return s1 + hbase(l) * part_head_stride(); }
  long long kn2_head_stride() const { return (long long)slots * n_tiles; }
  float* kn2_layer(int l) const { return kn2 + hbase(l) * kn2_head_stride(); }
  float* p0_layer(int l) const { return p0 + hbase(l) * part_head_stride(); }
  float* p1_layer(int l) const { return p1 + hbase(l) * part_head_stride(); }
  unsigned* kfl_layer(int l) const { return kfl + hbase(l) * kn2_head_stride(); }
  // the append pass's outputs besides the swizzled tiles
  void append_outputs(int l, PackPoolArgs& a) const {
    a.s0 = s0_layer(l);
    a.s1 = s1_layer(l);
    a.part_head_stride = part_head_stride();
    a.ext_s0 = s0_layer(l);
    a.norm2 = kn2_layer(l);
    a.norm2_head_stride = kn2_head_stride();
    a.p0 = p0_layer(l);
    a.p1 = p1_layer(l);
    a.pflag = kfl_layer(l);
  }
};

namespace {
// runs [h0, h1) of consecutive heads of `layer` with identical frame tables
std::vector<std::pair<int, int>> head_runs(const fvsr_ring* r, int layer) {
  std::vector<std::pair<int, int>> out;
  const auto& t = r->htab[layer];
  int h0 = 0;
  for (int h = 1; h <= r->heads; ++h)
    if (h == r->heads || t[h] != t[h0]) {
      out.emplace_back(h0, h);
      h0 = h;
    }
  return out;
}
// view of heads [h0, h1) at `layer` (see fvsr_ring)
fvsr_ring ring_view(const fvsr_ring* r, int layer, int h0, int h1) {
  fvsr_ring v;
  v.layers = r->layers;
  v.heads = h1 - h0;
  v.d = r->d;
  v.rows = r->rows;
  v.cols = r->cols;
  v.window = r->window;
  v.slots = r->slots;
  v.tiles_w = r->tiles_w;
  v.tiles_h = r->tiles_h;
  v.n_tiles = r->n_tiles;
  v.tile_bytes = r->tile_bytes;
  v.k = r->k;
  v.v = r->v;
  v.s0 = r->s0;
  v.s1 = r->s1;
  v.kn2 = r->kn2;
  v.p0 = r->p0;
  v.p1 = r->p1;
  v.kfl = r->kfl;
  v.rope = r->rope;
  v.rope_theta0 = r->rope_theta0;
  for (int i = 0; i < 3; ++i) v.rope_split[i] = r->rope_split[i];
  v.rope_t = r->rope_t;
  v.rope_h = r->rope_h;
  v.rope_w = r->rope_w;
  v.rope_t_cap = r->rope_t_cap;
  v.ctx.assign(r->layers, {});
  v.used.assign(r->layers, {});
  v.ctx[layer] = r->htab[layer][h0];
  v.used[layer] = r->hused[layer][h0];
  v.gen = r->gen;
  v.head0 = r->head0 + h0;
  v.heads_total = r->heads_total;
  return v;
}
// the view's table changes -> every head of its run
void ring_commit(fvsr_ring* r, const fvsr_ring& v, int layer, int h0, int h1) {
  for (int h = h0; h < h1; ++h) {
    r->htab[layer][h] = v.ctx[layer];
    r->hused[layer][h] = v.used[layer];
  }
  r->gen[layer] = std::max(r->gen[layer], v.gen[layer]);
}
}  // namespace

namespace {

// ---------------------------------------------------------------------------------------
// validation and geometry
// ---------------------------------------------------------------------------------------
int check_grid(const fvsr_grid* g, const char* what) {
  if (!g) return fail(FVSR_E_CONFIG, "%s: null grid", what);
  // TokenGrid constructor, P/include/vsr/grid.hpp:48-57
  if (g->n_frames < 1 || g->rows < 1 || g->cols < 1 || !g->frame_ids)
    return fail(FVSR_E_CONFIG, "TokenGrid: empty extents (%s)", what);
  if (g->n_frames > kMaxFrames)
    return fail(FVSR_E_CONFIG, "%s: %d frames exceeds the kernel limit of %d", what, g->n_frames, kMaxFrames);
  for (int i = 0; i < g->n_frames; ++i) {
    if (g->frame_ids[i] < 0) return fail(FVSR_E_CONFIG, "TokenGrid: negative frame id");
    if (i > 0 && g->frame_ids[i] <= g->frame_ids[i - 1])
      return fail(FVSR_E_CONFIG, "TokenGrid: frame ids must be strictly increasing");
  }
  return FVSR_OK;
}

long long grid_tokens(const fvsr_grid* g) { return (long long)g->n_frames * g->rows * g->cols; }

int build_geom(const fvsr_grid* gq, const fvsr_grid* gk, int d, const int* k_slots, DevGeom& g) {
  FVSR_TRY(check_grid(gq, "grid_q"));
  FVSR_TRY(check_grid(gk, "grid_k"));
  if (gq->rows != gk->rows || gq->cols != gk->cols)
    return fail(FVSR_E_CONFIG, "query and key grids must share rows/cols (%dx%d vs %dx%d)", gq->rows, gq->cols,
                gk->rows, gk->cols);
  std::memset(&g, 0, sizeof(g));
  g.rows = gq->rows;
  g.cols = gq->cols;
  g.tiles_w = (g.cols + 7) / 8;
  g.tiles_h = (g.rows + 7) / 8;
  g.n_tiles = g.tiles_w * g.tiles_h;
  g.d = d;
  const long long N = (long long)g.rows * g.cols;
  // temporal rows: consecutive frames sharing frame/2 (kBlockT = 2, P/include/vsr/partition.hpp:11)
  auto trows = [&](const fvsr_grid* gr, int* first, int* count, int* ftr, int& ntr) {
    ntr = 0;
    for (int i = 0; i < gr->n_frames; ++i) {
      if (i > 0 && gr->frame_ids[i] / 2 == gr->frame_ids[i - 1] / 2) {
        count[ntr - 1] = 2;
      } else {
        first[ntr] = i;
        count[ntr] = 1;
        ++ntr;
      }
      if (ftr) ftr[i] = ntr - 1;
    }
  };
  trows(gq, g.q_tr_first, g.q_tr_count, g.q_frame_tr, g.nq_trows);
  trows(gk, g.k_tr_first, g.k_tr_count, nullptr, g.nk_trows);
  g.nqf = gq->n_frames;
  g.nkf = gk->n_frames;
  g.bnq = g.nq_trows * g.n_tiles;
  g.bnk = g.nk_trows * g.n_tiles;
  for (int i = 0; i < g.nqf; ++i) g.q_frame_tok0[i] = (int)(i * N);
  for (int i = 0; i < g.nkf; ++i) {
    g.k_frame_tok0[i] = (int)(i * N);
    g.k_slot[i] = k_slots ? k_slots[i] : i;
  }
  for (int a = 0; a < g.nq_trows; ++a) {
    const int key = gq->frame_ids[g.q_tr_first[a]] / 2;
    g.q_tr_diag[a] = -1;
    for (int b = 0; b < g.nk_trows; ++b)
      if (gk->frame_ids[g.k_tr_first[b]] / 2 == key) g.q_tr_diag[a] = b;
  }
  if (N * std::max(g.nqf, g.nkf) > (long long)INT32_MAX)
    return fail(FVSR_E_CONFIG, "grid too large for 32-bit token indices");
  return FVSR_OK;
}

int build_mask(const fvsr_mask* m, const DevGeom& g, long long lk, DevMask& dm) {
  std::memset(&dm, 0, sizeof(dm));
  dm.frame_h = g.rows;
  dm.frame_w = g.cols;
  if (!m || m->kind == FVSR_MASK_ALL) {
    dm.kind = 0;
    dm.extent_h = dm.extent_w = 1;
    return FVSR_OK;
  }
  dm.kind = m->kind;
  dm.mode = m->mode;
  dm.extent_h = m->extent_h;
  dm.extent_w = m->extent_w;
  if (m->kind == FVSR_MASK_LOCALITY) {
    // build_locality_mask, P/src/mask.cpp:113-116
    if (m->extent_h < 1 || m->extent_w < 1) return fail(FVSR_E_CONFIG, "build_locality_mask: extents must be >= 1");
    if (m->extent_h > g.rows || m->extent_w > g.cols)
      return fail(FVSR_E_CONFIG, "build_locality_mask: extent larger than frame");
    if (m->mode != FVSR_LOCALITY_PRESERVED && m->mode != FVSR_LOCALITY_TRUNCATED)
      return fail(FVSR_E_CONFIG, "locality mode must be preserved (0) or truncated (1)");
    return FVSR_OK;
  }
  if (m->kind == FVSR_MASK_BITMASK) {
    if (!m->bits) return fail(FVSR_E_SHAPE, "bitmask mask without bits");
    if (m->words_per_row != (lk + 63) / 64) return fail(FVSR_E_SHAPE, "mask shape mismatch (words_per_row)");
    dm.bits = m->bits;
    dm.words_per_row = m->words_per_row;
    return FVSR_OK;
  }
  return fail(FVSR_E_CONFIG, "unknown mask kind %d", m->kind);
}

void* ws_get(fvsr_ctx* ctx, size_t bytes, int* st) {
  if (bytes > ctx->ws_bytes) {
    if (ctx->ws) cudaFree(ctx->ws);
    ctx->ws = nullptr;
    ctx->ws_bytes = 0;
    if (cudaMalloc(&ctx->ws, bytes) != cudaSuccess) {
      *st = fail(FVSR_E_NOMEM, "workspace allocation of %zu bytes failed", bytes);
      return nullptr;
    }
    ctx->ws_bytes = bytes;
  }
  *st = FVSR_OK;
  return ctx->ws;
}

struct Carve {
  uint8_t* base;
  size_t off = 0;
  explicit Carve(void* b) : base(static_cast<uint8_t*>(b)) {}
  template <typename T>
  T* take(size_t n) {
    off = (off + 1023) & ~size_t(1023);
    T* p = reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    return p;
  }
  static size_t need(std::initializer_list<size_t> sizes) {
    size_t o = 0;
    for (size_t s : sizes) o = ((o + 1023) & ~size_t(1023)) + s;
    return o + 1024;
  }
};

int after_launch(fvsr_ctx* ctx, cudaStream_t s, int nlaunch) {
  ctx->launches += nlaunch;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FVSR_E_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  if (ctx->flags & FVSR_FLAG_SYNC_CHECK) return fvsr_check_errors(ctx, reinterpret_cast<fvsr_stream_t>(s));
  return FVSR_OK;
}

// Kernel launch with programmatic stream serialization (PDL): the grid may be scheduled while
// the previous kernel of the stream drains; every kernel of this library calls pdl_wait()
// before touching global state, so the overlap covers launch latency and prologues only.
// FVSR_PDL=0 disables it (plain stream order).
// Only the attention kernel (one persistent CTA per SM, long prologue) is launched this way:
// small many-CTA kernels launched early pile onto the first SMs that free up.
template <typename... KArgs, typename... Args>
cudaError_t launch_kp(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                      Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  // programmatic dependent launch for the kernels that ask for it (the mask selector and the
  // attention: their prologues overlap the predecessor's tail).  On every kernel it measured
  // worse (139.3 vs 135.0 us per step): early-resident append blocks crowd the attention's tail.
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  return launch_kp(false, kern, grid, block, smem, s, std::forward<Args>(args)...);
}

// Dynamic shared-memory opt-in above 48 KB, cached per (device, kernel): the attribute is a
// per-device property, so a process driving several GPUs configures each one.
template <typename K>
int ensure_smem(K* kern, size_t bytes) {
  if (bytes <= 48 * 1024) return FVSR_OK;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  FVSR_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, reinterpret_cast<const void*>(kern)}];
  if (bytes > have) {
    FVSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
  }
  return FVSR_OK;
}

// Prefer the largest shared-memory carveout for a kernel whose occupancy is bounded by it
// (once per device and kernel).
template <typename K>
int ensure_carveout(K* kern) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, bool> done;
  int dev = 0;
  FVSR_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  bool& d = done[{dev, reinterpret_cast<const void*>(kern)}];
  if (!d) {
    FVSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    d = true;
  }
  return FVSR_OK;
}

// Tensor map of a token-major bf16 source for the TMA pack/pool path: 5-D (channel, col, row,
// frame, head), box (64, 8, 8, 1, 1), 128-byte swizzle, zero fill past the edges.  false when
// the driver entry point is missing or the layout does not meet TMA's alignment rules (the
// caller then keeps the bulk-copy path).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    cudaGetLastError();
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
bool encode_src_map(const fvsr_ctx* ctx, CUtensorMap* m, const void* src, int d, int rows, int cols, int frames,
                    int heads, long long token_stride, long long head_stride) {
  if (ctx->flags & FVSR_FLAG_NO_TMA) return false;
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn || !src || (d != 64 && d != 128)) return false;
  const long long ts = token_stride ? token_stride : d;
  const long long fs = (long long)rows * cols * ts;
  const long long hs = head_stride ? head_stride : fs * frames;
  if (reinterpret_cast<uintptr_t>(src) % 16 != 0 || (ts * 2) % 16 != 0 || (hs * 2) % 16 != 0) return false;
  const cuuint64_t dims[5] = {(cuuint64_t)d, (cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)frames, (cuuint64_t)heads};
  const cuuint64_t strides[4] = {(cuuint64_t)(ts * 2), (cuuint64_t)(cols * ts * 2), (cuuint64_t)(fs * 2),
                                 (cuuint64_t)(hs * 2)};
  const cuuint32_t box[5] = {64, 8, 8, 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(src), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int launch_pack_pool(const PackPoolArgs& a, const PoolGroups& pg, const SlotList& sl, dim3 grid, int max_cnt,
                     cudaStream_t s) {
  if (a.d % 8 != 0) return fail(FVSR_E_CONFIG, "pack_pool: head_dim must be a multiple of 8 (got %d)", a.d);
  if ((reinterpret_cast<uintptr_t>(a.src) | reinterpret_cast<uintptr_t>(a.src2)) % 16 != 0)
    return fail(FVSR_E_CONFIG, "pack_pool: token-major inputs must be 16-byte aligned");
  const size_t smem = pack_pool_smem(a.d, max_cnt, a.src2 != nullptr) +
                      (a.rope_t ? (size_t)(max_cnt * (a.rope_dt / 2) + 8 * (a.rope_dh / 2) + 8 * (a.rope_dw / 2)) *
                                      sizeof(float2)
                                : 0);
  // the RoPE variant is a separate instantiation so the plain pack/pool pass is unchanged
  auto kern = a.rope_t ? pack_pool_kernel<true> : pack_pool_kernel<false>;
  FVSR_TRY(ensure_smem(kern, smem));
  FVSR_CUDA(launch_k(kern, dim3(grid), dim3(kPPThreads), smem, s, a, pg, sl));
  return FVSR_OK;
}

int ctx_reserve_scores(fvsr_ctx* ctx, size_t n) {
  if (ctx->scores_cap >= n) return FVSR_OK;
  if (ctx->d_scores) cudaFree(ctx->d_scores);
  ctx->d_scores = nullptr;
  ctx->scores_cap = 0;
  if (cudaMalloc(&ctx->d_scores, n * sizeof(float)) != cudaSuccess)
    return fail(FVSR_E_CUDA, "cudaMalloc(%zu) for coarse scores failed", n * sizeof(float));
  ctx->scores_cap = n;
  return FVSR_OK;
}

int npow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// ---- CUDA-event spans on the launching stream ------------------------------------------
struct SpanGuard {
  fvsr_ctx* ctx;
  cudaStream_t s;
  int kind;
  cudaEvent_t a = nullptr;
  cudaEvent_t take() {
    if (ctx->ev_used == ctx->ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ctx->ev_pool.push_back(e);
    }
    return ctx->ev_pool[ctx->ev_used++];
  }
  SpanGuard(fvsr_ctx* c, cudaStream_t st, int k) : ctx(c), s(st), kind(k) {
    if (ctx->timing) {
      a = take();
      cudaEventRecord(a, s);
    }
  }
  ~SpanGuard() {
    if (ctx->timing && a) {
      cudaEvent_t b = take();
      cudaEventRecord(b, s);
      ctx->spans.push_back({a, b, kind});
    }
  }
};

// ---- launch helpers ---------------------------------------------------------------------
void launch_pack(const uint16_t* src, long long src_head_stride, int heads, int nframes, const DevGeom& g,
                 uint8_t* dst, long long dst_head_stride, const int* slots, cudaStream_t s) {
  SlotList sl{};
  for (int i = 0; i < nframes; ++i) sl.s[i] = slots ? slots[i] : i;
  dim3 grid(g.n_tiles, nframes, heads);
  (void)launch_k(pack_frames_kernel, grid, dim3(256), 0, s, src, src_head_stride, g.rows, g.cols, g.tiles_w,
                 g.n_tiles, g.d, dst, dst_head_stride, sl);
}

// Pooled partials for the t_rows of a frame list.
template <typename T>
void launch_pool_trows(const T* src, long long src_head_stride, int heads, const int* tr_first,
                       const int* tr_count, int ntr, const DevGeom& g, const int* slots, float* s0, float* s1,
                       long long part_head_stride, cudaStream_t s) {
  PoolGroups pg{};
  SlotList sl{};
  int nf = 0;
  for (int a = 0; a < ntr; ++a) {
    pg.first[a] = tr_first[a];
    pg.count[a] = tr_count[a];
    pg.ext_slot[a] = -1;
    nf = std::max(nf, tr_first[a] + tr_count[a]);
  }
  for (int i = 0; i < nf; ++i) sl.s[i] = slots ? slots[i] : i;
  dim3 grid(g.n_tiles, ntr, heads);
  const int threads = std::min(256, ((g.d + 31) / 32) * 32);
  (void)launch_k(pool_partials_kernel<T>, grid, dim3(threads), 0, s, src, src_head_stride, g.rows, g.cols, g.tiles_w,
                 g.n_tiles, g.d, pg, sl, s0, s1, part_head_stride, nullptr);
}

int launch_select(fvsr_ctx* ctx, const DevGeom& g, const DevMask& dm, int heads, const float* q_s0,
                  const float* q_s1, long long q_head_stride, const float* k_s0, const float* k_s1,
                  long long k_head_stride, float scale, long long topk, int cap, int* sel, int* sel_count,
                  int* diag, float* coarse, uint8_t* allowed, cudaStream_t s) {
  SelectParams p{};
  p.q_s0 = q_s0;
  p.q_s1 = q_s1;
  p.q_head_stride = q_head_stride;
  p.k_s0 = k_s0;
  p.k_s1 = k_s1;
  p.k_head_stride = k_head_stride;
  p.scale = scale;
  p.topk = topk;
  p.cap = cap;
  p.npow2 = npow2(g.bnk);
  p.sel = sel;
  p.sel_count = sel_count;
  p.diag = diag;
  p.coarse = coarse;
  p.allowed = allowed;
  p.err = ctx->d_err;
  if (g.d % 4 != 0) return fail(FVSR_E_CONFIG, "plan_sparse: head_dim must be a multiple of 4 (got %d)", g.d);
  // coarse scores -> workspace (L2-resident, heads*bnq*bnk floats), then per-row top-k
  const size_t n_scores = (size_t)heads * g.bnq * g.bnk;
  float* scores = coarse;
  ctx->scores_heads = ctx->scores_bnq = ctx->scores_bnk = 0;
  if (!scores) {
    if (ctx_reserve_scores(ctx, n_scores) != FVSR_OK) return FVSR_E_CUDA;
    scores = ctx->d_scores;
    ctx->scores_heads = heads;
    ctx->scores_bnq = g.bnq;
    ctx->scores_bnk = g.bnk;
  }
  p.coarse = nullptr;  // the score kernel writes `scores` directly
  if (g.d % 4 != 0) return fail(FVSR_E_CONFIG, "plan_sparse: head_dim must be a multiple of 4 (got %d)", g.d);
  const size_t smem_sc = (size_t)(kScQ + kScK) * (g.d + 4) * 4;
  FVSR_TRY(ensure_smem(coarse_score_kernel, smem_sc));
  dim3 gs((g.bnk + kScK - 1) / kScK, (g.bnq + kScQ - 1) / kScQ, heads);
  FVSR_CUDA(launch_k(coarse_score_kernel, dim3(gs), dim3(kScThreads), smem_sc, s, g, dm, p, scores));
  dim3 gt((g.bnq + kTopkWarps - 1) / kTopkWarps, heads);
  if (g.bnk <= 32 * 8)
    FVSR_CUDA(launch_k(topk_select_kernel<8>, dim3(gt), dim3(kTopkWarps * 32), 0, s, g, dm, p, scores));
  else if (g.bnk <= 32 * 32)
    FVSR_CUDA(launch_k(topk_select_kernel<32>, dim3(gt), dim3(kTopkWarps * 32), 0, s, g, dm, p, scores));
  else if (g.bnk <= 32 * 128)
    FVSR_CUDA(launch_k(topk_select_kernel<128>, dim3(gt), dim3(kTopkWarps * 32), 0, s, g, dm, p, scores));
  else
    return fail(FVSR_E_CONFIG, "too many key blocks (%d > 4096) for the selector", g.bnk);
  return FVSR_OK;
}

template <int D, int NQ, int MK>
int launch_attn_dqm(const DevGeom& g, const DevMask& dm, const AttnParams& p, int sms, cudaStream_t s) {
  using Cfg = AttnCfg<D, NQ>;
  FVSR_TRY(ensure_smem(sparse_attn_kernel<D, NQ, MK>, Cfg::kBytes));
  const long long units = p.unit_end - p.unit_begin;
  if (units <= 0) return FVSR_OK;
  // persistent CTAs, round robin over whole units: as many as the waves need (792 units on 148
  // SMs -> 6 waves -> 132 CTAs), so no SM holds one unit more than the others.  Every unit is
  // processed whole by one CTA: its output does not depend on the launch's other units.
  const long long waves = (units + sms - 1) / sms;
  const unsigned grid = (unsigned)((units + waves - 1) / waves);
  FVSR_CUDA(launch_kp(true, sparse_attn_kernel<D, NQ, MK>, dim3(grid), dim3(Cfg::kThreads), Cfg::kBytes, s, g, dm, p));
  return FVSR_OK;
}

template <int D, int NQ>
int launch_attn_dq(const DevGeom& g, const DevMask& dm, const AttnParams& p, int sms, cudaStream_t s) {
  if (dm.kind == 0) return launch_attn_dqm<D, NQ, 0>(g, dm, p, sms, s);
  if (dm.kind == 1) return launch_attn_dqm<D, NQ, 1>(g, dm, p, sms, s);
  return launch_attn_dqm<D, NQ, 2>(g, dm, p, sms, s);
}

bool trows_uniform(const DevGeom& g) {
  for (int a = 1; a < g.nq_trows; ++a)
    if (g.q_tr_count[a] != g.q_tr_count[0]) return false;
  return true;
}

// One persistent launch per query-tile height: NQ=64 for temporal rows holding one query
// frame, NQ=128 for rows holding two.  unit_begin/unit_end index the unit space
// head * (n_trows * tiles) + trow * tiles + tile and require uniform rows.
int launch_attention(fvsr_ctx* ctx, const DevGeom& g, const DevMask& dm, AttnParams p, int heads,
                     long long unit_begin, long long unit_end, cudaStream_t s) {
  if (g.d != 64 && g.d != 128)
    return fail(FVSR_E_CONFIG, "sparse_attention_exec: head_dim %d unsupported (64 or 128)", g.d);
  // key-tile descriptors: 5-bit frame index (31 = empty half), 5-bit tile row, 6-bit tile column
  if (g.nkf > kMaxKeyFrames)
    return fail(FVSR_E_CONFIG, "sparse_attention_exec: %d key frames exceeds the kernel limit of %d", g.nkf,
                kMaxKeyFrames);
  if (g.tiles_h > kMaxTilesH || g.tiles_w > kMaxTilesW)
    return fail(FVSR_E_CONFIG, "sparse_attention_exec: frame of %dx%d tokens exceeds the kernel limit of %dx%d",
                g.rows, g.cols, 8 * kMaxTilesH, 8 * kMaxTilesW);
  const bool uniform = trows_uniform(g);
  int sms = 0;
  FVSR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  SpanGuard sg(ctx, s, FVSR_TIME_ATTENTION);
  for (int nq = 1; nq <= 2; ++nq) {
    p.n_trows = 0;
    for (int a = 0; a < g.nq_trows; ++a)
      if (g.q_tr_count[a] == nq) p.trow_list[p.n_trows++] = a;
    if (!p.n_trows) continue;
    const long long total = (long long)heads * p.n_trows * g.n_tiles;
    p.unit_begin = uniform ? std::max(0ll, unit_begin) : 0;
    p.unit_end = uniform ? (unit_end < 0 ? total : std::min(unit_end, total)) : total;
    int st;
    if (g.d == 128)
      st = nq == 1 ? launch_attn_dq<128, 64>(g, dm, p, sms, s) : launch_attn_dq<128, 128>(g, dm, p, sms, s);
    else
      st = nq == 1 ? launch_attn_dq<64, 64>(g, dm, p, sms, s) : launch_attn_dq<64, 128>(g, dm, p, sms, s);
    FVSR_TRY(st);
    ctx->launches += 1;
  }
  return FVSR_OK;
}

int check_ctx(fvsr_ctx* ctx) {
  if (!ctx) return fail(FVSR_E_CONFIG, "null context");
  int dev = -1;
  FVSR_CUDA(cudaGetDevice(&dev));
  if (dev != ctx->device) FVSR_CUDA(cudaSetDevice(ctx->device));
  return FVSR_OK;
}

}  // namespace

// =========================================================================================
// C-ABI
// =========================================================================================
extern "C" {

int32_t fvsr_abi_version(void) { return FVSR_ABI_VERSION; }

#ifndef FVSR_BUILD_FLAGS
#define FVSR_BUILD_FLAGS ""
#endif
const char* fvsr_build_flags(void) { return FVSR_BUILD_FLAGS; }

const char* fvsr_last_error(void) { return g_last_error.c_str(); }

int32_t fvsr_ctx_create(fvsr_ctx** out) {
  if (!out) return fail(FVSR_E_CONFIG, "null output pointer");
  *out = nullptr;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(FVSR_E_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
  cudaDeviceProp prop{};
  FVSR_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10 || prop.minor != 0)
    return fail(FVSR_E_CUDA, "fvsr_b200 requires an sm_100 (B200) device; found sm_%d%d (%s)", prop.major, prop.minor,
                prop.name);
  auto* c = new fvsr_ctx();
  c->device = dev;
  if (cudaMalloc(&c->d_err, sizeof(unsigned)) != cudaSuccess ||
      cudaMalloc(&c->d_pairs, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&c->d_tiles, 2 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaFree(c->d_err);
    cudaFree(c->d_pairs);
    delete c;
    return fail(FVSR_E_NOMEM, "error word allocation failed");
  }
  cudaMemset(c->d_err, 0, sizeof(unsigned));
  cudaMemset(c->d_pairs, 0, sizeof(unsigned long long));
  cudaMemset(c->d_tiles, 0, 2 * sizeof(unsigned long long));
  *out = c;
  return FVSR_OK;
}

void fvsr_ctx_destroy(fvsr_ctx* ctx) {
  if (!ctx) return;
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_pairs);
  cudaFree(ctx->d_tiles);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->stage) cudaFree(ctx->stage);
  if (ctx->d_scores) cudaFree(ctx->d_scores);
  if (ctx->d_mass_scratch) cudaFree(ctx->d_mass_scratch);
  delete ctx;
}

int32_t fvsr_ctx_set_flags(fvsr_ctx* ctx, int32_t flags) {
  if (!ctx) return fail(FVSR_E_CONFIG, "null context");
  ctx->flags = flags;
  return FVSR_OK;
}

int64_t fvsr_ctx_launch_count(const fvsr_ctx* ctx) { return ctx ? ctx->launches : 0; }

int32_t fvsr_ctx_timing_enable(fvsr_ctx* ctx, int32_t enable) {
  if (!ctx) return fail(FVSR_E_CONFIG, "null context");
  ctx->timing = enable != 0;
  return FVSR_OK;
}

int32_t fvsr_ctx_timing_read(fvsr_ctx* ctx, int32_t kind, double* total_ms, int64_t* count, int32_t clear) {
  FVSR_TRY(check_ctx(ctx));
  FVSR_CUDA(cudaDeviceSynchronize());
  double ms = 0.0;
  int64_t n = 0;
  for (const auto& sp : ctx->spans) {
    if (sp.kind != kind) continue;
    float e = 0.f;
    FVSR_CUDA(cudaEventElapsedTime(&e, sp.a, sp.b));
    ms += e;
    ++n;
  }
  if (total_ms) *total_ms = ms;
  if (count) *count = n;
  if (clear) {
    ctx->spans.clear();
    ctx->ev_used = 0;
  }
  return FVSR_OK;
}

int32_t fvsr_ctx_read_pairs(fvsr_ctx* ctx, uint64_t* executed_pairs) {
  FVSR_TRY(check_ctx(ctx));
  FVSR_CUDA(cudaDeviceSynchronize());
  unsigned long long v = 0;
  FVSR_CUDA(cudaMemcpy(&v, ctx->d_pairs, sizeof(v), cudaMemcpyDeviceToHost));
  FVSR_CUDA(cudaMemset(ctx->d_pairs, 0, sizeof(v)));
  if (executed_pairs) *executed_pairs = v;
  return FVSR_OK;
}

int32_t fvsr_ctx_read_tiles(fvsr_ctx* ctx, uint64_t* tiles, uint64_t* full_tiles) {
  FVSR_TRY(check_ctx(ctx));
  FVSR_CUDA(cudaDeviceSynchronize());
  unsigned long long v[2] = {0, 0};
  FVSR_CUDA(cudaMemcpy(v, ctx->d_tiles, sizeof(v), cudaMemcpyDeviceToHost));
  FVSR_CUDA(cudaMemset(ctx->d_tiles, 0, sizeof(v)));
  if (tiles) *tiles = v[0];
  if (full_tiles) *full_tiles = v[1];
  return FVSR_OK;
}

int32_t fvsr_check_errors(fvsr_ctx* ctx, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  FVSR_CUDA(cudaStreamSynchronize(s));
  unsigned bits = 0;
  FVSR_CUDA(cudaMemcpy(&bits, ctx->d_err, sizeof(bits), cudaMemcpyDeviceToHost));
  if (bits) FVSR_CUDA(cudaMemset(ctx->d_err, 0, sizeof(unsigned)));
  const int code = status_from_bits(bits);
  if (code) return fail(code, "%s", device_error_message(code));
  return FVSR_OK;
}

int32_t fvsr_block_counts(const fvsr_grid* grid_q, const fvsr_grid* grid_k, int32_t* bnq, int32_t* bnk) {
  DevGeom g;
  FVSR_TRY(build_geom(grid_q, grid_k, 1, nullptr, g));
  if (bnq) *bnq = g.bnq;
  if (bnk) *bnk = g.bnk;
  return FVSR_OK;
}

}  // extern "C"
namespace {
template <typename T>
int plan_sparse_impl(fvsr_ctx* ctx, const T* q, const T* k, int32_t heads, int32_t d,
                         const fvsr_grid* grid_q, const fvsr_grid* grid_k, const fvsr_mask* mask, int64_t topk,
                         int32_t cap, int32_t* sel, int32_t* sel_count, int32_t* diag, float* coarse,
                         uint8_t* allowed, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!q || !k || !sel || !sel_count) return fail(FVSR_E_SHAPE, "plan_sparse: null tensor");
  if (heads < 1 || d < 1) return fail(FVSR_E_SHAPE, "plan_sparse: heads and head_dim must be >= 1");
  DevGeom g;
  FVSR_TRY(build_geom(grid_q, grid_k, d, nullptr, g));
  DevMask dm;
  FVSR_TRY(build_mask(mask, g, grid_tokens(grid_k), dm));
  if (topk < 1) return fail(FVSR_E_CONFIG, "plan_sparse: topk must be >= 1");  // sparse.cpp:83
  if (cap < std::min<long long>(topk, g.bnk))
    return fail(FVSR_E_SHAPE, "plan_sparse: cap %d < min(topk, bnk) = %lld", cap, std::min<long long>(topk, g.bnk));
  const long long Lq = grid_tokens(grid_q), Lk = grid_tokens(grid_k);
  const size_t qpart = (size_t)heads * g.nqf * g.n_tiles * d, kpart = (size_t)heads * g.nkf * g.n_tiles * d;
  int st;
  void* ws = ws_get(ctx, Carve::need({qpart * 4, qpart * 4, kpart * 4, kpart * 4}), &st);
  if (!ws) return st;
  Carve cv(ws);
  float* qs0 = cv.take<float>(qpart);
  float* qs1 = cv.take<float>(qpart);
  float* ks0 = cv.take<float>(kpart);
  float* ks1 = cv.take<float>(kpart);
  launch_pool_trows(q, Lq * d, heads, g.q_tr_first, g.q_tr_count, g.nq_trows, g, nullptr, qs0, qs1,
                    (long long)g.nqf * g.n_tiles * d, s);
  launch_pool_trows(k, Lk * d, heads, g.k_tr_first, g.k_tr_count, g.nk_trows, g, nullptr, ks0, ks1,
                    (long long)g.nkf * g.n_tiles * d, s);
  const float scale = 1.0f / std::sqrt(static_cast<float>(d));  // sparse.cpp:97
  FVSR_TRY(launch_select(ctx, g, dm, heads, qs0, qs1, (long long)g.nqf * g.n_tiles * d, ks0, ks1,
                         (long long)g.nkf * g.n_tiles * d, scale, topk, cap, sel, sel_count, diag, coarse, allowed, s));
  return after_launch(ctx, s, 4);
}
}  // namespace
extern "C" {

int32_t fvsr_plan_sparse(fvsr_ctx* ctx, const uint16_t* q, const uint16_t* k, int32_t heads, int32_t d,
                         const fvsr_grid* grid_q, const fvsr_grid* grid_k, const fvsr_mask* mask, int64_t topk,
                         int32_t cap, int32_t* sel, int32_t* sel_count, int32_t* diag, float* coarse,
                         uint8_t* allowed, fvsr_stream_t stream) {
  return plan_sparse_impl(ctx, q, k, heads, d, grid_q, grid_k, mask, topk, cap, sel, sel_count, diag, coarse, allowed,
                          stream);
}

int32_t fvsr_plan_sparse_f32(fvsr_ctx* ctx, const float* q, const float* k, int32_t heads, int32_t d,
                             const fvsr_grid* grid_q, const fvsr_grid* grid_k, const fvsr_mask* mask, int64_t topk,
                             int32_t cap, int32_t* sel, int32_t* sel_count, int32_t* diag, float* coarse,
                             uint8_t* allowed, fvsr_stream_t stream) {
  return plan_sparse_impl(ctx, q, k, heads, d, grid_q, grid_k, mask, topk, cap, sel, sel_count, diag, coarse, allowed,
                          stream);
}

int32_t fvsr_sparse_attention_exec(fvsr_ctx* ctx, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                                   int32_t heads, int32_t d, const fvsr_grid* grid_q, const fvsr_grid* grid_k,
                                   const fvsr_mask* mask, int32_t cap, const int32_t* sel,
                                   const int32_t* sel_count, float scale, int64_t row_begin, int64_t row_end,
                                   uint16_t* out, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!q || !k || !v || !sel || !sel_count || !out) return fail(FVSR_E_SHAPE, "sparse_attention_exec: null tensor");
  if (heads < 1) return fail(FVSR_E_SHAPE, "sparse_attention_exec: heads must be >= 1");
  if (d != 64 && d != 128)
    return fail(FVSR_E_CONFIG, "sparse_attention_exec: head_dim %d unsupported by the tensor-core kernel (64, 128)", d);
  if (cap < 1) return fail(FVSR_E_SHAPE, "sparse_attention_exec: cap must be >= 1");
  DevGeom g;
  FVSR_TRY(build_geom(grid_q, grid_k, d, nullptr, g));
  DevMask dm;
  FVSR_TRY(build_mask(mask, g, grid_tokens(grid_k), dm));
  const long long Lq = grid_tokens(grid_q), Lk = grid_tokens(grid_k);
  if (row_end < 0 || row_end > Lq) row_end = Lq;  // sparse.cpp:224
  if (row_begin < 0 || row_begin > row_end)
    return fail(FVSR_E_CONFIG, "sparse_attention_exec: empty or inverted row range");  // :225
  const size_t tb = (size_t)d * 128;
  const size_t qbytes = (size_t)heads * g.nqf * g.n_tiles * tb, kbytes = (size_t)heads * g.nkf * g.n_tiles * tb;
  int st;
  void* ws = ws_get(ctx, Carve::need({qbytes, kbytes, kbytes}), &st);
  if (!ws) return st;
  Carve cv(ws);
  uint8_t* qp = cv.take<uint8_t>(qbytes);
  uint8_t* kp = cv.take<uint8_t>(kbytes);
  uint8_t* vp = cv.take<uint8_t>(kbytes);
  launch_pack(q, Lq * d, heads, g.nqf, g, qp, (long long)g.nqf * g.n_tiles * tb, nullptr, s);
  launch_pack(k, Lk * d, heads, g.nkf, g, kp, (long long)g.nkf * g.n_tiles * tb, nullptr, s);
  launch_pack(v, Lk * d, heads, g.nkf, g, vp, (long long)g.nkf * g.n_tiles * tb, nullptr, s);
  AttnParams p{};
  p.q = qp;
  p.q_head_stride = (long long)g.nqf * g.n_tiles * tb;
  p.k = kp;
  p.v = vp;
  p.kv_head_stride = (long long)g.nkf * g.n_tiles * tb;
  p.sel = sel;
  p.sel_count = sel_count;
  p.cap = cap;
  p.out = out;
  p.out_head_stride = Lq * d;
  p.row_begin = row_begin;
  p.row_end = row_end;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.unit_begin = 0;
  p.out_tile_major = 0;
  p.err = ctx->d_err;
  p.pairs = ctx->d_pairs;
  p.tiles = ctx->d_tiles;
  FVSR_TRY(launch_attention(ctx, g, dm, p, heads, 0, -1, s));
  return after_launch(ctx, s, 3);
}

int32_t fvsr_sparsity_report(fvsr_ctx* ctx, int32_t heads, const fvsr_grid* grid_q, const fvsr_grid* grid_k,
                             const fvsr_mask* mask, int32_t cap, const int32_t* sel, const int32_t* sel_count,
                             uint64_t* executed_pairs, uint64_t* dense_pairs, uint64_t* selected_blocks,
                             uint64_t* allowed_blocks, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!sel || !sel_count || !executed_pairs || !dense_pairs || !selected_blocks || !allowed_blocks)
    return fail(FVSR_E_SHAPE, "sparsity_report: null tensor");
  DevGeom g;
  FVSR_TRY(build_geom(grid_q, grid_k, 1, nullptr, g));
  DevMask dm;
  FVSR_TRY(build_mask(mask, g, grid_tokens(grid_k), dm));
  for (uint64_t* o : {executed_pairs, dense_pairs, selected_blocks, allowed_blocks})
    FVSR_CUDA(cudaMemsetAsync(o, 0, sizeof(uint64_t) * heads, s));
  dim3 grid(g.bnq, heads);
  FVSR_CUDA(launch_k(sparsity_count_kernel, dim3(grid), dim3(128), 0, s, g, dm, sel, sel_count, cap,
                                             reinterpret_cast<unsigned long long*>(executed_pairs),
                                             reinterpret_cast<unsigned long long*>(dense_pairs),
                                             reinterpret_cast<unsigned long long*>(selected_blocks),
                                             reinterpret_cast<unsigned long long*>(allowed_blocks)));
  return after_launch(ctx, s, 1);
}

// ---- ring ---------------------------------------------------------------------------------
int32_t fvsr_ring_create(fvsr_ctx* ctx, int32_t layers, int32_t heads, int32_t d, int32_t rows, int32_t cols,
                         int32_t window_frames, fvsr_ring** out) {
  FVSR_TRY(check_ctx(ctx));
  if (!out) return fail(FVSR_E_CONFIG, "null output pointer");
  *out = nullptr;
  if (layers < 1 || heads < 1 || window_frames < 1)
    return fail(FVSR_E_CONFIG, "KVCache: empty extents");  // kv_cache.cpp:31
  if (rows < 1 || cols < 1) return fail(FVSR_E_CONFIG, "TokenGrid: empty extents");
  if (d != 64 && d != 128) return fail(FVSR_E_CONFIG, "ring: head_dim %d unsupported (64 or 128)", d);
  if (window_frames + 1 > kMaxKeyFrames)
    return fail(FVSR_E_CONFIG, "ring: window %d exceeds the kernel limit of %d frames", window_frames, kMaxKeyFrames - 1);
  if ((rows + 7) / 8 > kMaxTilesH || (cols + 7) / 8 > kMaxTilesW)
    return fail(FVSR_E_CONFIG, "ring: frame of %dx%d tokens exceeds the kernel limit of %dx%d", rows, cols,
                8 * kMaxTilesH, 8 * kMaxTilesW);
  auto* r = new fvsr_ring();
  r->layers = layers;
  r->heads = heads;
  r->d = d;
  r->rows = rows;
  r->cols = cols;
  r->window = window_frames;
  r->slots = window_frames + 1;
  r->tiles_w = (cols + 7) / 8;
  r->tiles_h = (rows + 7) / 8;
  r->n_tiles = r->tiles_w * r->tiles_h;
  r->tile_bytes = (size_t)d * 128;
  const size_t kvb = (size_t)layers * heads * r->kv_head_stride();
  const size_t pb = (size_t)layers * heads * r->part_head_stride() * sizeof(float);
  const size_t nb = (size_t)layers * heads * r->kn2_head_stride() * sizeof(float);
  if (cudaMalloc(&r->k, kvb) != cudaSuccess || cudaMalloc(&r->v, kvb) != cudaSuccess ||
      cudaMalloc(&r->s0, pb) != cudaSuccess || cudaMalloc(&r->s1, pb) != cudaSuccess ||
      cudaMalloc(&r->kn2, nb) != cudaSuccess || cudaMalloc(&r->p0, pb) != cudaSuccess ||
      cudaMalloc(&r->p1, pb) != cudaSuccess || cudaMalloc(&r->kfl, nb) != cudaSuccess) {
    fvsr_ring_destroy(r);
    return fail(FVSR_E_NOMEM, "ring allocation of %zu bytes failed", 2 * kvb + 4 * pb + 2 * nb);
  }
  r->htab.assign(layers, std::vector<fvsr_ring::Table>(heads));
  r->hused.assign(layers, std::vector<std::vector<char>>(heads, std::vector<char>(r->slots, 0)));
  r->gen.assign(layers, 0);
  r->heads_total = heads;
  *out = r;
  return FVSR_OK;
}

void fvsr_ring_destroy(fvsr_ring* ring) {
  if (!ring) return;
  cudaFree(ring->k);
  cudaFree(ring->v);
  cudaFree(ring->s0);
  cudaFree(ring->s1);
  cudaFree(ring->kn2);
  cudaFree(ring->p0);
  cudaFree(ring->p1);
  cudaFree(ring->kfl);
  cudaFree(ring->rope_t);
  cudaFree(ring->rope_h);
  cudaFree(ring->rope_w);
  delete ring;
}

// ---- fused RoPE tables (apply_rope, P/src/rope.cpp:30-62) ------------------------------------
namespace {
// (cos, sin) of pos * theta0^(-2i/d_axis) for pos in [p0, p1): the reference's double math,
// rounded to float exactly as apply_rope does
std::vector<float2> rope_table(double theta0, int d_axis, int p0, int p1) {
  std::vector<float2> t((size_t)(p1 - p0) * (d_axis / 2));
  for (int p = p0; p < p1; ++p)
    for (int i = 0; i < d_axis / 2; ++i) {
      const double inv_freq = std::pow(theta0, -2.0 * i / static_cast<double>(d_axis));
      const double angle = 1.0 * p * inv_freq;
      t[(size_t)(p - p0) * (d_axis / 2) + i] = make_float2(static_cast<float>(std::cos(angle)),
                                                           static_cast<float>(std::sin(angle)));
    }
  return t;
}

// frame ids [0, need) covered by the t-axis table (grown on demand; synchronous, rare)
int rope_reserve_t(fvsr_ring* r, int need) {
  if (need <= r->rope_t_cap) return FVSR_OK;
  int cap = std::max(need, std::max(1024, 2 * r->rope_t_cap));
  const std::vector<float2> t = rope_table(r->rope_theta0, r->rope_split[0], 0, cap);
  float2* d = nullptr;
  if (cudaMalloc(&d, t.size() * sizeof(float2)) != cudaSuccess)
    return fail(FVSR_E_NOMEM, "rope table allocation failed");
  FVSR_CUDA(cudaMemcpy(d, t.data(), t.size() * sizeof(float2), cudaMemcpyHostToDevice));
  if (r->rope_t) {
    FVSR_CUDA(cudaDeviceSynchronize());  // in-flight kernels may still read the old table
    cudaFree(r->rope_t);
  }
  r->rope_t = d;
  r->rope_t_cap = cap;
  return FVSR_OK;
}

int rope_args(fvsr_ring* r, const int* fids, int n, PackPoolArgs& a) {
  if (!r->rope) return FVSR_OK;
  if (n > 4) return fail(FVSR_E_CONFIG, "fused RoPE: at most 4 query frames per call (got %d)", n);
  int mx = 0;
  for (int i = 0; i < n; ++i) mx = std::max(mx, fids[i]);
  FVSR_TRY(rope_reserve_t(r, mx + 1));
  a.rope_t = r->rope_t;
  a.rope_h = r->rope_h;
  a.rope_w = r->rope_w;
  a.rope_dt = r->rope_split[0];
  a.rope_dh = r->rope_split[1];
  a.rope_dw = r->rope_split[2];
  for (int i = 0; i < n; ++i) a.rope_fid[i] = fids[i];
  return FVSR_OK;
}
}  // namespace

int32_t fvsr_ring_set_rope(fvsr_ring* r, double theta0, const int32_t* axis_split) {
  if (!r) return fail(FVSR_E_CONFIG, "null ring");
  int split[3];
  if (axis_split) {
    for (int i = 0; i < 3; ++i) split[i] = axis_split[i];
  } else {  // RopeConfig::split_default (P/src/rope.cpp:11-17), StreamConfig::rope (stream.cpp:8-10)
    split[0] = r->d / 2;
    split[1] = r->d / 4;
    split[2] = r->d / 4;
  }
  // RopeConfig::validate (P/src/rope.cpp:19-28)
  int sum = 0;
  for (int part : split) {
    if (part <= 0 || part % 2 != 0) return fail(FVSR_E_CONFIG, "RopeConfig: axis split parts must be positive and even");
    sum += part;
  }
  if (sum != r->d) return fail(FVSR_E_CONFIG, "RopeConfig: axis split must sum to dim");
  if (!(theta0 > 1.0)) return fail(FVSR_E_CONFIG, "RopeConfig: theta0 must exceed 1");
  if (kPPThreads % (r->d / 2) != 0) return fail(FVSR_E_CONFIG, "fused RoPE: head_dim %d unsupported", r->d);
  r->rope_theta0 = theta0;
  for (int i = 0; i < 3; ++i) r->rope_split[i] = split[i];
  FVSR_CUDA(cudaDeviceSynchronize());
  cudaFree(r->rope_t);
  cudaFree(r->rope_h);
  cudaFree(r->rope_w);
  r->rope_t = r->rope_h = r->rope_w = nullptr;
  r->rope_t_cap = 0;
  const std::vector<float2> th = rope_table(theta0, split[1], 0, r->rows);
  const std::vector<float2> tw = rope_table(theta0, split[2], 0, r->cols);
  if (cudaMalloc(&r->rope_h, th.size() * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&r->rope_w, tw.size() * sizeof(float2)) != cudaSuccess)
    return fail(FVSR_E_NOMEM, "rope table allocation failed");
  FVSR_CUDA(cudaMemcpy(r->rope_h, th.data(), th.size() * sizeof(float2), cudaMemcpyHostToDevice));
  FVSR_CUDA(cudaMemcpy(r->rope_w, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice));
  r->rope = true;
  return rope_reserve_t(r, 1);
}

}  // extern "C"
namespace {
// KVCache::append of one run of heads (a view; k, v point at its first head)
int ring_append_view(fvsr_ctx* ctx, fvsr_ring* r, int layer, int frame_id, const uint16_t* k, const uint16_t* v,
                     cudaStream_t s) {
  auto& c = r->ctx[layer];
  if (!c.empty() && frame_id <= c.back().first)
    return fail(FVSR_E_INVARIANT, "KVCache: frame ids must increase");  // kv_cache.cpp:42
  int slot = -1;
  for (int i = 0; i < r->slots; ++i)
    if (!r->used[layer][i]) { slot = i; break; }
  if (slot < 0)
    return fail(FVSR_E_INVARIANT, "KVCache: head retains more than window + current (evict before append)");
  int partner = -1;
  if ((frame_id & 1) && !c.empty() && c.back().first == frame_id - 1) partner = c.back().second;

  DevGeom g{};
  g.rows = r->rows;
  g.cols = r->cols;
  g.tiles_w = r->tiles_w;
  g.tiles_h = r->tiles_h;
  g.n_tiles = r->n_tiles;
  g.d = r->d;
  const long long N = (long long)r->rows * r->cols;
  SpanGuard sg(ctx, s, FVSR_TIME_APPEND);
  // one pass: K -> swizzled ring slot + pooled partials (S1 continues the even partner), V -> slot
  PackPoolArgs a{};
  a.src = k;
  a.src2 = v;
  a.src_head_stride = N * r->d;
  a.dst = r->k_layer(layer);
  a.dst2 = r->v_layer(layer);
  a.dst_head_stride = r->kv_head_stride();
  r->append_outputs(layer, a);
  a.rows = r->rows;
  a.cols = r->cols;
  a.tiles_w = r->tiles_w;
  a.n_tiles = r->n_tiles;
  a.d = r->d;
  FVSR_TRY(rope_args(r, &frame_id, 1, a));
  a.use_tma = encode_src_map(ctx, &a.tm, a.src, r->d, r->rows, r->cols, 1, r->heads, 0, a.src_head_stride) &&
              encode_src_map(ctx, &a.tm2, a.src2, r->d, r->rows, r->cols, 1, r->heads, 0, a.src_head_stride);
  PoolGroups pg{};
  pg.first[0] = 0;
  pg.count[0] = 1;
  pg.ext_slot[0] = partner;
  SlotList sl{};
  sl.s[0] = slot;
  FVSR_TRY(launch_pack_pool(a, pg, sl, dim3(r->n_tiles, 1, r->heads), 1, s));
  r->used[layer][slot] = 1;
  c.emplace_back(frame_id, slot);
  ++r->gen[layer];
  return FVSR_OK;
}
}  // namespace
extern "C" {

int32_t fvsr_ring_append(fvsr_ctx* ctx, fvsr_ring* r, int32_t layer, int32_t frame_id, const uint16_t* k,
                         const uint16_t* v, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!r || !k || !v) return fail(FVSR_E_SHAPE, "ring_append: null argument");
  if (layer < 0 || layer >= r->layers) return fail(FVSR_E_SHAPE, "KVCache: layer/head out of range");
  if (frame_id < 0) return fail(FVSR_E_CONFIG, "TokenGrid: negative frame id");
  if (r->rope) FVSR_TRY(rope_reserve_t(r, frame_id + 1));  // views never grow the shared table
  const long long hs = (long long)r->rows * r->cols * r->d;
  int launches = 0;
  for (auto [h0, h1] : head_runs(r, layer)) {
    fvsr_ring v_ = ring_view(r, layer, h0, h1);
    FVSR_TRY(ring_append_view(ctx, &v_, layer, frame_id, k + h0 * hs, v + h0 * hs, s));
    ring_commit(r, v_, layer, h0, h1);
    ++launches;
  }
  return after_launch(ctx, s, launches);
}

int32_t fvsr_ring_evict_sliding(fvsr_ring* r, int32_t layer) {
  if (!r) return fail(FVSR_E_CONFIG, "null ring");
  if (layer < 0 || layer >= r->layers) return fail(FVSR_E_SHAPE, "KVCache: layer out of range");
  for (int h = 0; h < r->heads; ++h) {
    auto& c = r->htab[layer][h];
    while ((int)c.size() > r->window) {  // kv_cache.cpp:100-106
      r->hused[layer][h][c.front().second] = 0;
      c.erase(c.begin());
      ++r->gen[layer];
    }
  }
  return FVSR_OK;
}

int32_t fvsr_ring_evict_keep(fvsr_ring* r, int32_t layer, int32_t keep) {
  if (!r) return fail(FVSR_E_CONFIG, "null ring");
  if (layer < 0 || layer >= r->layers) return fail(FVSR_E_SHAPE, "KVCache: layer out of range");
  if (keep < 0) return fail(FVSR_E_CONFIG, "ring_evict_keep: keep must be >= 0");
  for (int h = 0; h < r->heads; ++h) {
    auto& c = r->htab[layer][h];
    while ((int)c.size() > keep) {  // sliding: oldest first (kv_cache.cpp:100-106)
      r->hused[layer][h][c.front().second] = 0;
      c.erase(c.begin());
      ++r->gen[layer];
    }
  }
  return FVSR_OK;
}

int32_t fvsr_ring_frame_ids(const fvsr_ring* r, int32_t layer, int32_t* ids, int32_t cap, int32_t* n) {
  return fvsr_ring_frame_ids_head(r, layer, 0, ids, cap, n);
}

int32_t fvsr_ring_frame_ids_head(const fvsr_ring* r, int32_t layer, int32_t head, int32_t* ids, int32_t cap,
                                 int32_t* n) {
  if (!r) return fail(FVSR_E_CONFIG, "null ring");
  if (layer < 0 || layer >= r->layers || head < 0 || head >= r->heads)
    return fail(FVSR_E_SHAPE, "KVCache: layer/head out of range");
  const auto& c = r->htab[layer][head];
  if (n) *n = (int32_t)c.size();
  if ((int)c.size() > cap) return fail(FVSR_E_SHAPE, "frame id buffer too small");
  for (size_t i = 0; i < c.size(); ++i) ids[i] = c[i].first;
  return FVSR_OK;
}

}  // extern "C"

namespace {
// The new frame of a fused step (KVCache::append, P/src/kv_cache.cpp:39-47).
struct AppendSpec {
  const uint16_t* k;
  const uint16_t* v;
  int frame_id;
  fvsr_layout kv;  // {0, 0}: [heads][rows * cols][d]
};

// Ring attention of one layer-step: mask builder (one launch: optional ring append of the
// new frame, Q pack + pool, coarse scores, top-k) then the sparse attention kernel.
int ring_step_view(fvsr_ctx* ctx, fvsr_ring* r, int layer, const uint16_t* q, const int32_t* q_frame_ids, int nq,
                   const fvsr_mask* mask, int64_t topk, float scale, int64_t unit_begin, int64_t unit_end,
                   uint16_t* out, int out_layout, int sel_cap, int32_t* sel, int32_t* sel_count,
                   const AppendSpec* app, cudaStream_t s, fvsr_layout q_lay, fvsr_layout out_lay, float* coarse_out) {
  if (!r || !q || !out || !q_frame_ids) return fail(FVSR_E_SHAPE, "ring_attention: null argument");
  if (layer < 0 || layer >= r->layers) return fail(FVSR_E_SHAPE, "KVCache: layer out of range");
  auto& c = r->ctx[layer];
  int app_slot = -1, partner = -1;
  if (app) {  // fvsr_ring_append's contract (kv_cache.cpp:39-47)
    if (!app->k || !app->v) return fail(FVSR_E_SHAPE, "ring_append: null argument");
    if (app->frame_id < 0) return fail(FVSR_E_CONFIG, "TokenGrid: negative frame id");
    if (!c.empty() && app->frame_id <= c.back().first)
      return fail(FVSR_E_INVARIANT, "KVCache: frame ids must increase");  // kv_cache.cpp:42
    for (int i = 0; i < r->slots; ++i)
      if (!r->used[layer][i]) { app_slot = i; break; }
    if (app_slot < 0)
      return fail(FVSR_E_INVARIANT, "KVCache: head retains more than window + current (evict before append)");
    if ((app->frame_id & 1) && !c.empty() && c.back().first == app->frame_id - 1) partner = c.back().second;
  }
  if (c.empty() && !app) return fail(FVSR_E_CONFIG, "ring_attention: empty context");
  std::vector<int> kids, kslots;
  for (auto& fs : c) {
    kids.push_back(fs.first);
    kslots.push_back(fs.second);
  }
  if (app) {
    kids.push_back(app->frame_id);
    kslots.push_back(app_slot);
  }
  fvsr_grid gq{q_frame_ids, nq, r->rows, r->cols};
  fvsr_grid gk{kids.data(), (int)kids.size(), r->rows, r->cols};
  DevGeom g;
  FVSR_TRY(build_geom(&gq, &gk, r->d, kslots.data(), g));
  DevMask dm;
  FVSR_TRY(build_mask(mask, g, grid_tokens(&gk), dm));
  if (topk < 1) return fail(FVSR_E_CONFIG, "plan_sparse: topk must be >= 1");
  if (g.bnk > 32 * 128) return fail(FVSR_E_CONFIG, "too many key blocks (%d > 4096) for the selector", g.bnk);
  if (g.d % 8 != 0) return fail(FVSR_E_CONFIG, "pack_pool: head_dim must be a multiple of 8 (got %d)", g.d);
  const int cap_need = (int)std::min<long long>(topk, g.bnk);
  if (sel && sel_cap < cap_need) return fail(FVSR_E_SHAPE, "ring_attention: sel_cap < min(topk, bnk)");
  const int cap = sel ? sel_cap : cap_need;
  const int d = r->d;
  const long long Lq = grid_tokens(&gq);
  const size_t tb = r->tile_bytes;
  const size_t qbytes = (size_t)r->heads * g.nqf * g.n_tiles * tb;
  const size_t qpart = (size_t)r->heads * g.nqf * g.n_tiles * d;
  const size_t nsel = (size_t)r->heads * g.bnq;
  const size_t qn = (size_t)r->heads * g.nqf * g.n_tiles;
  int st;
  void* ws = ws_get(ctx, Carve::need({qbytes, qpart * 4, qpart * 4, nsel * cap * 4, nsel * 4, qn * 4}), &st);
  if (!ws) return st;
  Carve cv(ws);
  uint8_t* qp = cv.take<uint8_t>(qbytes);
  float* qs0 = cv.take<float>(qpart);
  float* qs1 = cv.take<float>(qpart);
  int* wsel = cv.take<int>(nsel * cap);
  int* wcnt = cv.take<int>(nsel);
  float* qn2 = cv.take<float>(qn);
  int* use_sel = sel ? sel : wsel;
  int* use_cnt = sel_count ? sel_count : wcnt;
  {
    SpanGuard sg(ctx, s, app ? FVSR_TIME_FRONT : FVSR_TIME_MASK_BUILDER);
    FrontArgs fa{};
    // append: K -> swizzled ring slot + pooled partials (S1 continues the even partner), V -> slot
    if (app) {
      PackPoolArgs& a = fa.kv;
      a.src = app->k;
      a.src_head_stride = app->kv.head_stride ? app->kv.head_stride : (long long)r->rows * r->cols * d;
      a.src_token_stride = app->kv.token_stride;
      a.dst = r->k_layer(layer);
      a.dst_head_stride = r->kv_head_stride();
      r->append_outputs(layer, a);
      a.rows = r->rows;
      a.cols = r->cols;
      a.tiles_w = r->tiles_w;
      a.n_tiles = r->n_tiles;
      a.d = d;
      FVSR_TRY(rope_args(r, &app->frame_id, 1, a));
      a.use_tma = encode_src_map(ctx, &a.tm, a.src, d, r->rows, r->cols, 1, r->heads, a.src_token_stride, a.src_head_stride);
      fa.kv_pg.first[0] = 0;
      fa.kv_pg.count[0] = 1;
      fa.kv_pg.ext_slot[0] = partner;
      fa.kv_sl.s[0] = app_slot;
      // V: the same tiles, packed only (no partials, no bounds, never rotated)
      PackPoolArgs& av = fa.v;
      av = a;
      av.src = app->v;
      av.dst = r->v_layer(layer);
      av.s0 = av.s1 = nullptr;
      av.ext_s0 = nullptr;
      av.norm2 = nullptr;
      av.p0 = av.p1 = nullptr;
      av.pflag = nullptr;
      av.use_tma = encode_src_map(ctx, &av.tm, av.src, d, r->rows, r->cols, 1, r->heads, av.src_token_stride,
                                  av.src_head_stride);
      if ((reinterpret_cast<uintptr_t>(a.src) | reinterpret_cast<uintptr_t>(av.src)) % 16 != 0)
        return fail(FVSR_E_CONFIG, "pack_pool: token-major inputs must be 16-byte aligned");
    }
    // one pass over Q: swizzled query tiles for the tensor cores + pooled partials for the plan
    PackPoolArgs& a = fa.q;
    a.src = q;
    a.src_head_stride = q_lay.head_stride ? q_lay.head_stride : Lq * d;
    a.src_token_stride = q_lay.token_stride;
    a.dst = qp;
    a.dst_head_stride = (long long)g.nqf * g.n_tiles * tb;
    a.s0 = qs0;
    a.s1 = qs1;
    a.part_head_stride = (long long)g.nqf * g.n_tiles * d;
    a.norm2 = qn2;
    a.norm2_head_stride = (long long)g.nqf * g.n_tiles;
    a.rows = g.rows;
    a.cols = g.cols;
    a.tiles_w = g.tiles_w;
    a.n_tiles = g.n_tiles;
    a.d = d;
    if (reinterpret_cast<uintptr_t>(q) % 16 != 0)
      return fail(FVSR_E_CONFIG, "pack_pool: token-major inputs must be 16-byte aligned");
    FVSR_TRY(rope_args(r, q_frame_ids, nq, a));
    a.use_tma = encode_src_map(ctx, &a.tm, q, d, g.rows, g.cols, g.nqf, r->heads, a.src_token_stride, a.src_head_stride);
    int max_cnt = 1;
    for (int t = 0; t < g.nq_trows; ++t) {
      fa.q_pg.first[t] = g.q_tr_first[t];
      fa.q_pg.count[t] = g.q_tr_count[t];
      fa.q_pg.ext_slot[t] = -1;
      max_cnt = std::max(max_cnt, g.q_tr_count[t]);
    }
    for (int i = 0; i < g.nqf; ++i) fa.q_sl.s[i] = i;
    fa.heads = r->heads;
    fa.n_tiles = g.n_tiles;
    fa.q_trows = g.nq_trows;
    SelectParams p{};
    p.q_s0 = qs0;
    p.q_s1 = qs1;
    p.q_head_stride = (long long)g.nqf * g.n_tiles * d;
    p.k_s0 = r->s0_layer(layer);
    p.k_s1 = r->s1_layer(layer);
    p.k_head_stride = r->part_head_stride();
    p.k_p0 = r->p0_layer(layer);
    p.k_p1 = r->p1_layer(layer);
    p.k_flag = r->kfl_layer(layer);
    p.k_flag_head_stride = r->kn2_head_stride();
    p.scale = 1.0f / std::sqrt(static_cast<float>(d));  // sparse.cpp:97
    p.topk = topk;
    p.cap = cap;
    p.npow2 = npow2(g.bnk);
    p.sel = use_sel;
    p.sel_count = use_cnt;
    p.coarse = coarse_out;  // kept for fvsr_ring_frame_mass
    p.err = ctx->d_err;
    const size_t rope_bytes =
        r->rope ? (size_t)(2 * (r->rope_split[0] / 2) + 8 * (r->rope_split[1] / 2) + 8 * (r->rope_split[2] / 2)) *
                      sizeof(float2)
                : 0;
    // launch 1: ring append + Q pack/pool (independent inputs, one pass)
    const size_t smem_p = ring_pack_smem(d, max_cnt, rope_bytes);
    const unsigned grid_p = (unsigned)((app ? 2 * r->heads * g.n_tiles : 0) + r->heads * g.nq_trows * g.n_tiles);
    auto kp = r->rope ? ring_pack_kernel<true> : ring_pack_kernel<false>;
    FVSR_TRY(ensure_smem(kp, smem_p));
    FVSR_TRY(ensure_carveout(kp));  // 12 blocks of ~18 KB resident per SM
    {
      SpanGuard sp(ctx, s, FVSR_TIME_PACK);
      FVSR_CUDA(launch_k(kp, dim3(grid_p), dim3(kPPThreads), smem_p, s, fa));
    }
    if (ctx->flags & FVSR_FLAG_SYNC_CHECK) {
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return fail(FVSR_E_CUDA, "ring_pack kernel: %s", cudaGetErrorString(e));
    }
    // launch 2: coarse scores + top-k (programmatic launch: its prologue overlaps launch 1's tail)
    const size_t smem_s = mask_select_smem(d, g.bnk);
    const unsigned grid_s = (unsigned)(r->heads * ((g.bnq + kFrontQB - 1) / kFrontQB));
    auto launch_s = [&](auto kern) -> int {
      FVSR_TRY(ensure_smem(kern, smem_s));
      FVSR_CUDA(launch_kp(true, kern, dim3(grid_s), dim3(kFrontThreads), smem_s, s, g, dm, p));
      return FVSR_OK;
    };
    SpanGuard ss(ctx, s, FVSR_TIME_SELECT);
    if (smem_s <= 200 * 1024) {
      st = g.bnk <= 256 ? launch_s(mask_select_kernel<8>)
                        : (g.bnk <= 1024 ? launch_s(mask_select_kernel<32>) : launch_s(mask_select_kernel<128>));
      FVSR_TRY(st);
      ctx->launches += 2;
    } else {  // score rows too long for shared memory: scores through L2, then the row selector
      FVSR_TRY(launch_select(ctx, g, dm, r->heads, qs0, qs1, p.q_head_stride, p.k_s0, p.k_s1, p.k_head_stride, p.scale,
                             topk, cap, use_sel, use_cnt, nullptr, coarse_out, nullptr, s));
      ctx->launches += 3;
    }
    if (ctx->flags & FVSR_FLAG_SYNC_CHECK) {  // debugging: attribute a fault to the front launches
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return fail(FVSR_E_CUDA, "mask_select kernel: %s", cudaGetErrorString(e));
    }
  }
  if (app) {  // the new frame is in the ring from here on
    r->used[layer][app_slot] = 1;
    c.emplace_back(app->frame_id, app_slot);
    ++r->gen[layer];
  }
  const long long units_total = (long long)r->heads * g.nq_trows * g.n_tiles;
  if (unit_end < 0 || unit_end > units_total) unit_end = units_total;
  if (unit_begin < 0 || unit_begin > unit_end) return fail(FVSR_E_CONFIG, "ring_attention: bad unit range");
  if (!trows_uniform(g) && (unit_begin != 0 || unit_end != units_total || out_layout == FVSR_OUT_TILE_MAJOR))
    return fail(FVSR_E_CONFIG, "ring_attention: unit ranges / tile-major output need query rows of equal height");
  AttnParams p{};
  p.q = qp;
  p.q_head_stride = (long long)g.nqf * g.n_tiles * tb;
  p.k = r->k_layer(layer);
  p.v = r->v_layer(layer);
  p.kv_head_stride = r->kv_head_stride();
  p.sel = use_sel;
  p.sel_count = use_cnt;
  p.cap = cap;
  p.out = out;
  p.out_head_stride = out_lay.head_stride ? out_lay.head_stride : Lq * d;
  p.out_token_stride = out_lay.token_stride;
  p.row_begin = 0;
  p.row_end = Lq;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out_tile_major = out_layout == FVSR_OUT_TILE_MAJOR ? 1 : 0;
  p.err = ctx->d_err;
  p.pairs = ctx->d_pairs;
  p.tiles = ctx->d_tiles;
  p.kn2 = r->kn2_layer(layer);
  p.kn2_head_stride = r->kn2_head_stride();
  p.qn2 = qn2;
  p.qn2_head_stride = (long long)g.nqf * g.n_tiles;
  FVSR_TRY(launch_attention(ctx, g, dm, p, r->heads, unit_begin, unit_end, s));
  return after_launch(ctx, s, 0);
}

// One layer-step over every run of heads with identical frame tables (one run unless
// head-wise eviction made the heads diverge; unit ranges / tile-major output need one run).
int ring_step_impl(fvsr_ctx* ctx, fvsr_ring* r, int layer, const uint16_t* q, const int32_t* q_frame_ids, int nq,
                   const fvsr_mask* mask, int64_t topk, float scale, int64_t unit_begin, int64_t unit_end,
                   uint16_t* out, int out_layout, int sel_cap, int32_t* sel, int32_t* sel_count,
                   const AppendSpec* app, cudaStream_t s, fvsr_layout q_lay = {0, 0},
                   fvsr_layout out_lay = {0, 0}) {
  if (!r || !q || !out || !q_frame_ids || nq < 1) return fail(FVSR_E_SHAPE, "ring_attention: null argument");
  if (layer < 0 || layer >= r->layers) return fail(FVSR_E_SHAPE, "KVCache: layer out of range");
  if (r->rope) {  // views never grow the shared RoPE table
    int mx = app ? app->frame_id : 0;
    for (int i = 0; i < nq; ++i) mx = std::max(mx, (int)q_frame_ids[i]);
    if (mx >= 0) FVSR_TRY(rope_reserve_t(r, mx + 1));
  }
  const auto runs = head_runs(r, layer);
  if (runs.size() > 1 && (unit_begin != 0 || unit_end >= 0 || out_layout == FVSR_OUT_TILE_MAJOR))
    return fail(FVSR_E_CONFIG,
                "ring_attention: the heads' frame sets diverge (head-wise eviction): unit ranges and tile-major "
                "output (head-parallel shards) need head-identical sets");
  // coarse-score slices of the runs (fvsr_ring_frame_mass reads them back)
  std::vector<fvsr_ctx::ScoreRun> sr;
  size_t total = 0;
  for (auto [h0, h1] : runs) {
    std::vector<int> kids;
    for (auto& fs : r->htab[layer][h0]) kids.push_back(fs.first);
    if (app) kids.push_back(app->frame_id);
    int bnq = 0, bnk = 0;
    if (!kids.empty()) {
      fvsr_grid gq{q_frame_ids, nq, r->rows, r->cols};
      fvsr_grid gk{kids.data(), (int)kids.size(), r->rows, r->cols};
      DevGeom g;
      if (build_geom(&gq, &gk, r->d, nullptr, g) == FVSR_OK) {
        bnq = g.bnq;
        bnk = g.bnk;
      }
    }
    sr.push_back({h0, h1, bnq, bnk, total});
    total += (size_t)(h1 - h0) * bnq * bnk;
  }
  if (ctx_reserve_scores(ctx, std::max<size_t>(1, total)) != FVSR_OK) return FVSR_E_CUDA;
  ctx->score_runs.clear();
  ctx->scores_heads = ctx->scores_bnq = ctx->scores_bnk = 0;
  const long long Lq = (long long)nq * r->rows * r->cols;
  const long long qhs = q_lay.head_stride ? q_lay.head_stride : Lq * r->d;
  const long long ohs = out_lay.head_stride ? out_lay.head_stride : Lq * r->d;
  for (const auto& run : sr) {
    fvsr_ring v = ring_view(r, layer, run.h0, run.h1);
    AppendSpec a{};
    if (app) {
      const long long khs = app->kv.head_stride ? app->kv.head_stride : (long long)r->rows * r->cols * r->d;
      a = *app;
      a.k += run.h0 * khs;
      a.v += run.h0 * khs;
    }
    FVSR_TRY(ring_step_view(ctx, &v, layer, q + run.h0 * qhs, q_frame_ids, nq, mask, topk, scale, unit_begin,
                            unit_end, out_layout == FVSR_OUT_TILE_MAJOR ? out : out + run.h0 * ohs, out_layout,
                            sel_cap, sel ? sel + (long long)run.h0 * run.bnq * sel_cap : nullptr,
                            sel_count ? sel_count + (long long)run.h0 * run.bnq : nullptr, app ? &a : nullptr, s,
                            q_lay, out_lay, ctx->d_scores + run.off));
    ring_commit(r, v, layer, run.h0, run.h1);
  }
  ctx->score_runs = sr;
  ctx->scores_heads = r->heads;
  ctx->scores_bnq = sr.empty() ? 0 : sr[0].bnq;
  ctx->scores_bnk = sr.empty() ? 0 : sr[0].bnk;
  ctx->stamp.ring = r;
  ctx->stamp.layer = layer;
  ctx->stamp.gen = r->gen[layer];
  ctx->stamp.qids.assign(q_frame_ids, q_frame_ids + nq);
  ctx->stamp.mask = mask ? *mask : fvsr_mask{};
  return FVSR_OK;
}
}  // namespace

extern "C" {

int32_t fvsr_ring_attention(fvsr_ctx* ctx, fvsr_ring* r, int32_t layer, const uint16_t* q,
                            const int32_t* q_frame_ids, int32_t nq, const fvsr_mask* mask, int64_t topk, float scale,
                            int64_t unit_begin, int64_t unit_end, uint16_t* out, int32_t out_layout,
                            int32_t sel_cap, int32_t* sel, int32_t* sel_count, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  return ring_step_impl(ctx, r, layer, q, q_frame_ids, nq, mask, topk, scale, unit_begin, unit_end, out, out_layout,
                        sel_cap, sel, sel_count, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

int32_t fvsr_ring_step(fvsr_ctx* ctx, fvsr_ring* r, int32_t layer, int32_t frame_id, const uint16_t* k,
                       const uint16_t* v, const uint16_t* q, const int32_t* q_frame_ids, int32_t nq,
                       const fvsr_mask* mask, int64_t topk, float scale, int64_t unit_begin, int64_t unit_end,
                       uint16_t* out, int32_t out_layout, int32_t sel_cap, int32_t* sel, int32_t* sel_count,
                       fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  const AppendSpec app{k, v, frame_id, {0, 0}};
  return ring_step_impl(ctx, r, layer, q, q_frame_ids, nq, mask, topk, scale, unit_begin, unit_end, out, out_layout,
                        sel_cap, sel, sel_count, &app, reinterpret_cast<cudaStream_t>(stream));
}

int32_t fvsr_ring_step_layout(fvsr_ctx* ctx, fvsr_ring* r, int32_t layer, int32_t frame_id, const uint16_t* k,
                              const uint16_t* v, fvsr_layout kv_layout, const uint16_t* q, fvsr_layout q_layout,
                              const int32_t* q_frame_ids, int32_t nq, const fvsr_mask* mask, int64_t topk, float scale,
                              uint16_t* out, fvsr_layout out_layout, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  if (!r) return fail(FVSR_E_SHAPE, "ring_step: null ring");
  for (const fvsr_layout* l : {&kv_layout, &q_layout, &out_layout})
    if (l->head_stride < 0 || l->token_stride < 0 || (l->token_stride && l->token_stride < r->d) ||
        (l->token_stride * 2) % 16 || (l->head_stride * 2) % 16)
      return fail(FVSR_E_CONFIG, "ring_step: layout strides must be >= d elements and 16-byte multiples");
  const AppendSpec app{k, v, frame_id, kv_layout};
  return ring_step_impl(ctx, r, layer, q, q_frame_ids, nq, mask, topk, scale, 0, -1, out, FVSR_OUT_TOKEN_MAJOR, 0,
                        nullptr, nullptr, &app, reinterpret_cast<cudaStream_t>(stream), q_layout, out_layout);
}

// ---- scored eviction ------------------------------------------------------
namespace {
int launch_frame_mass(fvsr_ctx* ctx, const DevGeom& g, const DevMask& dm, int heads, const float* coarse,
                      double* mass, cudaStream_t s) {
  // scratch: row max / denominators [heads][bnq], block masses [heads][bnk] (fp64)
  const size_t nrow = (size_t)heads * g.bnq, nblk = (size_t)heads * g.bnk;
  if (!ctx->d_mass_scratch || ctx->mass_scratch_cap < 2 * nrow + nblk) {
    cudaFree(ctx->d_mass_scratch);
    ctx->d_mass_scratch = nullptr;
    ctx->mass_scratch_cap = 0;
    if (cudaMalloc(&ctx->d_mass_scratch, (2 * nrow + nblk) * sizeof(double)) != cudaSuccess)
      return fail(FVSR_E_NOMEM, "frame_attention_mass: scratch allocation failed");
    ctx->mass_scratch_cap = 2 * nrow + nblk;
  }
  double* rmax = ctx->d_mass_scratch;
  double* rden = rmax + nrow;
  double* bmass = rden + nrow;
  const unsigned wpc = kMassThreads / 32;
  FVSR_CUDA(launch_k(frame_mass_rows_kernel, dim3((unsigned)((nrow + wpc - 1) / wpc)), dim3(kMassThreads), 0, s, g, dm,
                     coarse, rmax, rden, heads));
  FVSR_CUDA(launch_k(frame_mass_blocks_kernel, dim3((unsigned)((g.bnk + 31) / 32), (unsigned)heads),
                     dim3(kMassThreads), 0, s, g, dm, coarse, (const double*)rmax, (const double*)rden, bmass));
  const int nf = heads * g.nkf;
  FVSR_CUDA(launch_k(frame_mass_frames_kernel, dim3((unsigned)((nf + 3) / 4)), dim3(128), 0, s, g,
                     (const double*)bmass, mass, heads));
  return after_launch(ctx, s, 3);
}

// victim order for one head (P/src/kv_cache.cpp:81-93): lowest score first, older frame on
// ties, the newest frame exempt
std::vector<int> evict_victims(const std::vector<int>& ids, const double* score, size_t excess) {
  std::vector<size_t> idx;
  for (size_t i = 0; i + 1 < ids.size(); ++i) idx.push_back(i);
  std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
    if (score[a] != score[b]) return score[a] < score[b];
    return ids[a] < ids[b];
  });
  std::vector<int> out;
  for (size_t i = 0; i < excess && i < idx.size(); ++i) out.push_back(ids[idx[i]]);
  std::sort(out.begin(), out.end());
  return out;
}
}  // namespace

int32_t fvsr_frame_attention_mass(fvsr_ctx* ctx, int32_t heads, const fvsr_grid* grid_q, const fvsr_grid* grid_k,
                                  const fvsr_mask* mask, const float* coarse, double* mass, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  if (!coarse || !mass) return fail(FVSR_E_SHAPE, "frame_attention_mass: null tensor");
  if (heads < 1) return fail(FVSR_E_SHAPE, "frame_attention_mass: heads must be >= 1");
  DevGeom g;
  FVSR_TRY(build_geom(grid_q, grid_k, 4, nullptr, g));
  DevMask dm;
  FVSR_TRY(build_mask(mask, g, grid_tokens(grid_k), dm));
  return launch_frame_mass(ctx, g, dm, heads, coarse, mass, reinterpret_cast<cudaStream_t>(stream));
}

int32_t fvsr_ring_frame_mass(fvsr_ctx* ctx, fvsr_ring* r, int32_t layer, const int32_t* q_frame_ids, int32_t nq,
                             const fvsr_mask* mask, double* mass, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  if (!r || !q_frame_ids) return fail(FVSR_E_SHAPE, "ring_frame_mass: null argument");
  if (layer < 0 || layer >= r->layers) return fail(FVSR_E_SHAPE, "KVCache: layer out of range");
  fvsr_ctx::ScoreStamp want;
  want.ring = r;
  want.layer = layer;
  want.gen = r->gen[layer];
  want.qids.assign(q_frame_ids, q_frame_ids + nq);
  want.mask = mask ? *mask : fvsr_mask{};
  if (ctx->scores_heads != r->heads || ctx->score_runs.empty() || !(ctx->stamp == want))
    return fail(FVSR_E_CONFIG,
                "ring_frame_mass: the coarse scores on the context are not those of this ring, layer, frame set, "
                "query frames and mask (call right after fvsr_ring_attention of the same layer, before evicting)");
  if (!mass) return fail(FVSR_E_SHAPE, "ring_frame_mass: null output");
  // per run of heads with identical frame tables: its geometry, its score slice, its rows of mass
  for (const auto& run : ctx->score_runs) {
    const auto& c = r->htab[layer][run.h0];
    if (c.empty()) return fail(FVSR_E_CONFIG, "ring_frame_mass: empty context");
    std::vector<int> kids, kslots;
    for (auto& fs : c) {
      kids.push_back(fs.first);
      kslots.push_back(fs.second);
    }
    fvsr_grid gq{q_frame_ids, nq, r->rows, r->cols};
    fvsr_grid gk{kids.data(), (int)kids.size(), r->rows, r->cols};
    DevGeom g;
    FVSR_TRY(build_geom(&gq, &gk, r->d, kslots.data(), g));
    DevMask dm;
    FVSR_TRY(build_mask(mask, g, grid_tokens(&gk), dm));
    if (g.bnq != run.bnq || g.bnk != run.bnk) return fail(FVSR_E_CONFIG, "ring_frame_mass: stale score slices");
    FVSR_TRY(launch_frame_mass(ctx, g, dm, run.h1 - run.h0, ctx->d_scores + run.off,
                               mass + (size_t)run.h0 * kids.size(), reinterpret_cast<cudaStream_t>(stream)));
  }
  return FVSR_OK;
}

int32_t fvsr_ring_evict(fvsr_ring* r, int32_t layer, int32_t strategy, const double* scores) {
  if (!r) return fail(FVSR_E_CONFIG, "null ring");
  if (layer < 0 || layer >= r->layers) return fail(FVSR_E_SHAPE, "KVCache: layer out of range");
  if (strategy < FVSR_EVICT_SLIDING || strategy > FVSR_EVICT_HEAD_WISE)
    return fail(FVSR_E_CONFIG, "unknown eviction strategy: %d", strategy);
  if (strategy == FVSR_EVICT_SLIDING) return fvsr_ring_evict_sliding(r, layer);  // kv_cache.cpp:100-106
  bool over = false;  // kv_cache.cpp:108-111
  for (int h = 0; h < r->heads; ++h) over = over || (int)r->htab[layer][h].size() > r->window;
  if (!over) return FVSR_OK;
  if (!scores) return fail(FVSR_E_CONFIG, "KVCache: importance scores required for scored eviction");
  const size_t n = r->htab[layer][0].size();
  for (int h = 1; h < r->heads; ++h)
    if (r->htab[layer][h].size() != n) return fail(FVSR_E_SHAPE, "KVCache: score count must match retained frames");
  auto ids_of = [&](int h) {
    std::vector<int> ids;
    for (auto& fs : r->htab[layer][h]) ids.push_back(fs.first);
    return ids;
  };
  auto drop = [&](int h, int id) {
    auto& c = r->htab[layer][h];
    for (size_t i = 0; i < c.size(); ++i)
      if (c[i].first == id) {
        r->hused[layer][h][c[i].second] = 0;
        c.erase(c.begin() + (long)i);
        ++r->gen[layer];
        return;
      }
  };
  if (strategy == FVSR_EVICT_UNIFORM) {  // kv_cache.cpp:118-128: head scores summed, one decision
    const std::vector<int> ids = ids_of(0);
    for (int h = 1; h < r->heads; ++h)
      if (ids_of(h) != ids) return fail(FVSR_E_INVARIANT, "KVCache: uniform strategy requires head-identical sets");
    std::vector<double> total(n, 0.0);
    for (int h = 0; h < r->heads; ++h)
      for (size_t i = 0; i < n; ++i) total[i] += scores[(size_t)h * n + i];
    for (int id : evict_victims(ids, total.data(), n - (size_t)r->window))
      for (int h = 0; h < r->heads; ++h) drop(h, id);
    return FVSR_OK;
  }
  for (int h = 0; h < r->heads; ++h) {  // head_wise (kv_cache.cpp:130-135): per-head decisions
    const std::vector<int> ids = ids_of(h);
    if ((int)ids.size() <= r->window) continue;
    for (int id : evict_victims(ids, scores + (size_t)h * n, ids.size() - (size_t)r->window)) drop(h, id);
  }
  return FVSR_OK;
}

// ---- token-mask builders ----------------------------------------------------
namespace {
int launch_token_mask(fvsr_ctx* ctx, const int32_t* labels_host, long long L, int kind, int lookahead,
                      uint64_t* bits, cudaStream_t s, int n_segments = 0) {
  const size_t smem = (size_t)L * sizeof(int);
  if (smem > 200 * 1024) return fail(FVSR_E_CONFIG, "token mask: %lld tokens exceed the builder limit", L);
  const long long wpr = (L + 63) / 64;
  // few segments: build one row per segment, then copy rows (rows of a segment are equal)
  const bool by_segment = kind == 0 && n_segments > 0 && 4LL * n_segments <= L;
  const size_t lab_bytes = (smem + 255) / 256 * 256;
  const size_t row_bytes = by_segment ? (size_t)n_segments * wpr * 8 : 0;
  int st;
  void* ws = ws_get(ctx, lab_bytes + row_bytes, &st);
  if (!ws) return st;
  FVSR_CUDA(cudaMemcpyAsync(ws, labels_host, smem, cudaMemcpyHostToDevice, s));
  const int kk = by_segment ? 2 : kind;
  auto kern = kk == 0 ? token_mask_kernel<0> : (kk == 1 ? token_mask_kernel<1> : token_mask_kernel<2>);
  FVSR_TRY(ensure_smem(kern, smem));
  int sms = 148;
  (void)cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  const long long nrows = by_segment ? n_segments : L;
  const long long tasks = nrows * (kind == 1 ? 1 : (wpr + 31) / 32);
  const long long ctas = std::min<long long>((tasks + kMaskThreads / 32 - 1) / (kMaskThreads / 32), 4LL * sms);
  auto* rows = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(ws) + lab_bytes);
  FVSR_CUDA(launch_k(kern, dim3((unsigned)ctas), dim3(kMaskThreads), smem, s, static_cast<const int*>(ws), (int)L,
                     lookahead, by_segment ? rows : reinterpret_cast<unsigned long long*>(bits), (int)nrows));
  if (by_segment) {
    const long long words = L * wpr;
    const long long cc = std::min<long long>((words + kMaskThreads - 1) / kMaskThreads, 8LL * sms);
    FVSR_CUDA(launch_k(token_rows_copy_kernel, dim3((unsigned)cc), dim3(kMaskThreads), 0, s,
                       static_cast<const int*>(ws), (int)L, (const unsigned long long*)rows,
                       reinterpret_cast<unsigned long long*>(bits)));
    ctx->launches += 1;
  }
  // the host labels may be released on return (pageable copy is staged before returning)
  return after_launch(ctx, s, 1);
}
}  // namespace

int32_t fvsr_build_segment_mask(fvsr_ctx* ctx, const int32_t* seg, int64_t L, uint64_t* bits,
                                fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  if (!bits || (L > 0 && !seg)) return fail(FVSR_E_SHAPE, "build_segment_mask: null argument");
  // P/src/mask.cpp:69-78
  if (L < 1) return fail(FVSR_E_CONFIG, "build_segment_mask: no tokens labeled");
  int max_id = -1;
  for (long long i = 0; i < L; ++i) {
    if (seg[i] < 0) return fail(FVSR_E_CONFIG, "build_segment_mask: negative segment id");
    max_id = std::max(max_id, (int)seg[i]);
  }
  std::vector<char> seen((size_t)max_id + 1, 0);
  for (long long i = 0; i < L; ++i) seen[(size_t)seg[i]] = 1;
  for (char c : seen)
    if (!c) return fail(FVSR_E_CONFIG, "build_segment_mask: segment ids not contiguous");
  return launch_token_mask(ctx, seg, L, 0, 0, bits, reinterpret_cast<cudaStream_t>(stream), max_id + 1);
}

int32_t fvsr_build_causal_mask(fvsr_ctx* ctx, const int32_t* frame, int64_t L, int32_t lookahead, uint64_t* bits,
                               fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  if (!bits || (L > 0 && !frame)) return fail(FVSR_E_SHAPE, "build_causal_mask: null argument");
  if (L < 1) return fail(FVSR_E_SHAPE, "build_causal_mask: frame list length does not match L");
  // P/src/mask.cpp:89-92
  if (lookahead < 0) return fail(FVSR_E_CONFIG, "build_causal_mask: negative lookahead");
  for (long long i = 1; i < L; ++i)
    if (frame[i] < frame[i - 1]) return fail(FVSR_E_CONFIG, "build_causal_mask: frame indices must be non-decreasing");
  return launch_token_mask(ctx, frame, L, 1, lookahead, bits, reinterpret_cast<cudaStream_t>(stream));
}

int32_t fvsr_rms_norm(fvsr_ctx* ctx, const float* x, const float* gain, int64_t n, int32_t D, uint16_t* y,
                      fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  if (!x || !gain || !y) return fail(FVSR_E_SHAPE, "rms_norm: null tensor");
  if (n < 0 || D < 4 || D % 4) return fail(FVSR_E_SHAPE, "rms_norm: D must be a positive multiple of 4");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(gain)) % 16 || reinterpret_cast<uintptr_t>(y) % 8)
    return fail(FVSR_E_CONFIG, "rms_norm: misaligned buffers");
  if (n == 0) return FVSR_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  FVSR_CUDA(launch_k(rms_norm_kernel, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, s, x, gain, (long long)n, (int)D, y));
  return after_launch(ctx, s, 1);
}

int32_t fvsr_untile(fvsr_ctx* ctx, const uint16_t* tiles, int64_t units, int32_t frames_per_unit, int32_t nq,
                    int32_t rows, int32_t cols, int32_t d, uint16_t* out, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  if (!tiles || !out) return fail(FVSR_E_SHAPE, "untile: null tensor");
  if (units < 0 || rows < 1 || cols < 1 || d < 8 || d % 8 || (frames_per_unit != 1 && frames_per_unit != 2) ||
      nq < 1 || nq % frames_per_unit)
    return fail(FVSR_E_CONFIG, "untile: bad geometry");
  if ((reinterpret_cast<uintptr_t>(tiles) | reinterpret_cast<uintptr_t>(out)) % 16)
    return fail(FVSR_E_CONFIG, "untile: buffers must be 16-byte aligned");
  if (units == 0) return FVSR_OK;
  int sms = 148;
  (void)cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  FVSR_CUDA(launch_k(untile_kernel, dim3(4 * sms), dim3(256), 0, s, tiles, (long long)units, (int)frames_per_unit,
                     (int)nq, (int)rows, (int)cols, (int)d, out));
  return after_launch(ctx, s, 1);
}

int32_t fvsr_ring_step_host(fvsr_ctx* ctx, fvsr_ring* r, int32_t layer, int32_t frame_id, const uint16_t* q_host,
                            const uint16_t* k_host, const uint16_t* v_host, const fvsr_mask* mask, int64_t topk,
                            float scale, uint16_t* out_host, fvsr_stream_t stream) {
  FVSR_TRY(check_ctx(ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!r || !q_host || !k_host || !v_host || !out_host) return fail(FVSR_E_SHAPE, "ring_step_host: null argument");
  const size_t n = (size_t)r->heads * r->rows * r->cols * r->d;  // elements per tensor
  const size_t bytes = n * sizeof(uint16_t);
  if (ctx->stage_bytes < 4 * bytes) {
    if (ctx->stage) cudaFree(ctx->stage);
    ctx->stage = nullptr;
    ctx->stage_bytes = 0;
    if (cudaMalloc(&ctx->stage, 4 * bytes) != cudaSuccess) return fail(FVSR_E_NOMEM, "staging allocation failed");
    ctx->stage_bytes = 4 * bytes;
  }
  uint16_t* dq = static_cast<uint16_t*>(ctx->stage);
  uint16_t* dk = dq + n;
  uint16_t* dv = dk + n;
  uint16_t* dout = dv + n;
  FVSR_CUDA(cudaMemcpyAsync(dq, q_host, bytes, cudaMemcpyHostToDevice, s));
  FVSR_CUDA(cudaMemcpyAsync(dk, k_host, bytes, cudaMemcpyHostToDevice, s));
  FVSR_CUDA(cudaMemcpyAsync(dv, v_host, bytes, cudaMemcpyHostToDevice, s));
  const int32_t qids[1] = {frame_id};
  FVSR_TRY(fvsr_ring_step(ctx, r, layer, frame_id, dk, dv, dq, qids, 1, mask, topk, scale, 0, -1, dout,
                          FVSR_OUT_TOKEN_MAJOR, 0, nullptr, nullptr, stream));
  FVSR_TRY(fvsr_ring_evict_sliding(r, layer));
  FVSR_CUDA(cudaMemcpyAsync(out_host, dout, bytes, cudaMemcpyDeviceToHost, s));
  return FVSR_OK;
}

}  // extern "C"

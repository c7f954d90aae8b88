// kernel_attn.cu — block-sparse streaming attention on tcgen05 / TMEM (sm_100a).
//
// Replaces exec_block_range / sparse_attention_exec (P/src/sparse.cpp:141-254,
// P = /root/reference/proj): for each query row, exact softmax attention over the keys of
// its q-block's selected key blocks, filtered by the token mask, merged across blocks
// with a running max.  Rows outside [row_begin, row_end) are zero; a row whose selected
// blocks hold no allowed key latches DegenerateRowError (sparse.cpp:198-200).
//
// Work unit: one query tile position of one head and one temporal row — NQ = 64 query
// rows (one frame's 8x8 tile, the reference's streaming q-block) or NQ = 128 (the two
// frames of a (2,8,8) q-block, the paper's 2-latent chunk).  tcgen05 issues M in {64,128}
// and M=64 runs at half rate, so the kernel is TRANSPOSED: keys sit on the M=128 axis.
//     S^T[128 keys x NQ]  = K_tile[128 x d] . Q^T                 (K-major A, K-major B)
//     O^T[d x NQ]        += V_tile^T[d x 128] . P^T[128 keys x NQ] (MN-major A, MN-major B)
//
// Key tiles.  A selected block of two frames (2m, 2m+1 of one 8x8 tile) fills the 128 key
// rows of a tile: rows 0-63 frame 2m, rows 64-127 frame 2m+1.  A single-frame block (the
// current even frame, an odd frame whose partner was evicted) has 64 keys; consecutive
// single-frame blocks of a selection are PAIRED into one tile (rows 0-63 the first, 64-127
// the second), so every MMA tile and every softmax pass carries 128 real keys.  The order
// of the keys only changes fp32 rounding: the softmax is order-free.  A tile descriptor is
// two 16-bit halves (frame index, tile row, tile col), built per unit by the table builder.
//
// Softmax in the transposed layout: TMEM lane j holds key j's scores for all queries.
// Softmax warps = 4 lane quarters x NQ/32 column groups; a column group (4 warps, 128
// lanes) owns 32 query columns and keeps, per column, a running reference c (log2 units)
// and per-thread partial denominators.  Fixed-reference units (|q||k| bounds every score)
// keep c = 0; otherwise the reference only moves when a score exceeds it by > 8 (FA4-style
// lazy rescale), decided by one bar.red.or across the group per tile.
//
// Persistent CTAs (round-robin over units), 16 warps: 8 softmax (two ping-pong groups:
// tile t of a unit belongs to group t % 2), Q/K producer, QK issuer (+ TMEM allocator),
// V producer, PV issuer, and an epilogue warpgroup that merges the groups' O^T, stores the
// output and builds each unit's tables one unit ahead.
#include "fvsr_common.cuh"

namespace fvsr {

constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr int kInfoCap = 256;              // per-unit tile-descriptor table entries
constexpr float kBoundSlack = 64.0f;       // log2 units: p <= 2^64 keeps O, l and bf16 P finite
constexpr float kFixedBound = 60.0f;       // |s*scale*log2e| <= 60 for the unit: fixed reference 0
constexpr int kQkLead = 3;                 // QK(G) waits for PV(G - kQkLead) to be issued
constexpr uint32_t kHalfNone = 0xF800u;    // tile half without keys (frame index 31)
constexpr int kMaxKeyFrames = 31;          // frame index 31 marks an empty half
constexpr int kMaxTilesH = 32, kMaxTilesW = 64;  // tile coordinates of a 16-bit half

struct AttnParams {
  const uint8_t* q;          // packed q frame-tiles [heads][nqf][n_tiles]
  long long q_head_stride;   // bytes
  const uint8_t* k;          // packed k frame-tiles [heads][slots][n_tiles]
  const uint8_t* v;
  long long kv_head_stride;  // bytes
  const int* sel;            // [heads][bnq][cap]
  const int* sel_count;      // [heads][bnq]
  int cap;
  uint16_t* out;             // bf16 [heads][Lq][d] (token major) or [unit][NQ][d] (tile major)
  long long out_head_stride; // elements
  long long out_token_stride;// elements between consecutive tokens of a head (token major; 0: D)
  long long row_begin, row_end;
  float scale_log2;          // scale * log2(e)
  int n_trows;               // q temporal rows handled by this launch
  int trow_list[kMaxFrames]; // their indices in the geometry
  long long unit_begin, unit_end;  // [begin, end) of this launch's unit space
  int out_tile_major;        // 1: out is [unit - unit_begin][NQ][d]
  unsigned* err;
  unsigned long long* pairs; // += executed (mask-allowed, selected-block) token pairs
  unsigned long long* tiles; // [0] += key tiles issued, [1] += of them with 128 key rows
  // Optional score bounds (null = always vote): max squared key-row norm per (slot, tile) and
  // query-row norm per (q frame, tile).  |s| <= |q||k| lets a column group skip the rescale
  // vote when no score of a tile can exceed the word's references by more than kBoundSlack.
  const float* kn2;
  long long kn2_head_stride;  // elements
  const float* qn2;
  long long qn2_head_stride;  // elements
};

template <int D, int NQ>
struct AttnCfg {
  static constexpr int kSW = 8;                      // softmax warps (two warpgroups)
  static constexpr int kGroups = NQ == 64 ? 2 : 1;   // ping-pong softmax groups (tile parity)
  static constexpr int kWG = kSW / kGroups;          // warps per group
  static constexpr int kCGg = kWG / 4;               // column groups per group (4 lane quarters each)
  static constexpr int kCPT = NQ / kCGg;             // query columns per softmax thread
  static_assert(kCPT == 64, "columns per thread");
  static constexpr int kProducerWarp = kSW;          // Q and K tiles
  static constexpr int kQkWarp = kSW + 1;            // QK^T issuer (+ TMEM allocator)
  static constexpr int kVProducerWarp = kSW + 2;     // V tiles (decoupled so K runs ahead)
  static constexpr int kPvWarp = kSW + 3;            // PV issuer (own program order: QK never waits on P)
  static constexpr int kEpiWarp = kSW + 4;           // epilogue warpgroup (merge, normalise, store, tables)
  static constexpr int kThreads = kSW * 32 + 256;    // 16 warps
  static constexpr int kRegSoftmax = 184;            // setmaxnreg: 256 x 184 + 256 x 72 = 64K
  static constexpr int kRegOther = 256 - kRegSoftmax;
  static constexpr int kNS = NQ == 64 ? 4 : 2;       // S^T buffers in TMEM
  static constexpr int kNK = 2;                      // K stages (QK consumes them right away)
  static constexpr int kNV = 2;                      // V stages (released only after PV)
  static constexpr int kPB = 4;                      // pv_go / pv_done barrier ring (> kNV)
  static constexpr int kNP = NQ == 64 ? 4 : 1;       // P^T buffers
  static constexpr int kOB = 2;                      // O^T buffers per group (double-buffered units)
  static constexpr uint32_t kTileBytes = D * 128;    // one packed 64-row frame-tile
  static constexpr uint32_t kQSub = NQ * 128;        // Q sub-tile stride (NQ rows x 128 B)
  static constexpr uint32_t kQBytes = (D / 64) * kQSub;
  static constexpr uint32_t kKVBytes = 2 * kTileBytes;  // 128 rows
  static constexpr uint32_t kPBytes = NQ * 256;      // 128 keys x NQ bf16
  static constexpr uint32_t kOffQ = 0;
  static constexpr uint32_t kOffK = kOffQ + kQBytes;
  static constexpr uint32_t kOffV = kOffK + kNK * kKVBytes;
  static constexpr uint32_t kOffP = kOffV + kNV * kKVBytes;
  static constexpr uint32_t kOffS = kOffP + kNP * kPBytes;  // scratch
  static constexpr uint32_t kScratch = NQ == 64 ? 13312 : 16384;
  // scratch layout (bytes): barriers 256 | c [2][2][128] f32 | alpha [2][128] | l [2][2][128] |
  // f [2][128] | red [2][CGg][4][CPT] | win [2][32] i32 | info [2][cap] | kn2 [2][cap] | qn2 [2] |
  // c0 [2] | cmin [2][CGg][CPT/32] | unit [2][8] i32 | prog [2] | kmax [4]
  static constexpr uint32_t kScratchUsed =
      256 + 4 * (512 + 256 + 512 + 256) + 4 * (2 * kCGg * 4 * kCPT) + 4 * 64 + 8 * 2 * 256 + 16 +
      4 * (2 * kCGg * (kCPT / 32)) + 64 + 8 + 16;
  static_assert(kScratchUsed <= kScratch, "scratch budget");
  static constexpr uint32_t kOffE = kOffS + kScratch;         // epilogue staging chunk
  static constexpr uint32_t kEpiBytes = 4096;
  static constexpr int kEpiCols = kEpiBytes / (2 * D);        // query columns per staged chunk
  static constexpr uint32_t kBytes = kOffE + kEpiBytes + 1024;  // + alignment slack
  static constexpr uint32_t kTmemCols = 512;         // S x NS + O x groups x OB
  static_assert(kNS * NQ + kGroups * kOB * NQ <= 512, "TMEM budget");
  static_assert(kBytes <= 232448, "shared memory budget");
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32 pairs (FMUL2 / FADD2 on sm_100): a * s and a += b on two lanes of a pair.
__device__ __forceinline__ void fmul2(float& a0, float& a1, float s) {
  unsigned long long x;
  asm("{\n\t.reg .b64 s2;\n\tmov.b64 s2, {%3, %3};\n\tmov.b64 %0, {%1, %2};\n\t"
      "mul.rn.f32x2 %0, %0, s2;\n\t}"
      : "=l"(x)
      : "f"(a0), "f"(a1), "f"(s));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(x));
}
__device__ __forceinline__ void fadd2(float& a0, float& a1, float b0, float b1) {
  unsigned long long x;
  asm("{\n\t.reg .b64 b2;\n\tmov.b64 b2, {%3, %4};\n\tmov.b64 %0, {%1, %2};\n\t"
      "add.rn.f32x2 %0, %0, b2;\n\t}"
      : "=l"(x)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(x));
}

// Barrier over `n` threads that also ORs a predicate across them.
__device__ __forceinline__ bool bar_red_or(uint32_t id, uint32_t n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred pi, po;\n\tsetp.ne.u32 pi, %1, 0;\n\t"
      "bar.red.or.pred po, %2, %3, pi;\n\tselp.u32 %0, 1, 0, po;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

// Butterfly reduce-scatter of N (16, 32 or 64) per-thread column values across a warp:
// step s keeps the half selected by lane bit (4-s); with N=16 a final xor-1 combine merges
// lane pairs.  On return v[i], i < max(1, N/32), is the warp-wide reduction of column
// col(i) = N == 64 ? 2*lane + i : (N == 32 ? lane : lane >> 1).
template <int N, bool kMax>
__device__ __forceinline__ void warp_colreduce(float* v, int lane) {
  constexpr int kSteps = N >= 32 ? 5 : 4;
#pragma unroll
  for (int step = 0; step < kSteps; ++step) {
    const int half = (N / 2) >> step;
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
  if (N == 16) {
    const float recv = __shfl_xor_sync(0xffffffffu, v[0], 1);
    v[0] = kMax ? fmaxf(v[0], recv) : v[0] + recv;
  }
}
__device__ __forceinline__ int colreduce_col(int n, int lane, int i) {
  return n == 64 ? 2 * lane + i : (n == 32 ? lane : lane >> 1);
}

template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<32>(uint32_t taddr, uint32_t* r) {
  tmem_ld32(taddr, r);
}
template <>
__device__ __forceinline__ void tmem_ld<64>(uint32_t taddr, uint32_t* r) {
  tmem_ld32(taddr, r);
  tmem_ld32(taddr + 32, r + 32);
}
template <int N>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t* r);
template <>
__device__ __forceinline__ void tmem_st<32>(uint32_t taddr, const uint32_t* r) {
  tmem_st32(taddr, r);
}

// max of N values as a balanced tree (ILP instead of a serial chain)
template <int N>
__device__ __forceinline__ float tree_max(const float* v) {
  float t[N / 2];
#pragma unroll
  for (int i = 0; i < N / 2; ++i) t[i] = fmaxf(v[2 * i], v[2 * i + 1]);
#pragma unroll
  for (int w = N / 4; w >= 1; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) t[i] = fmaxf(t[2 * i], t[2 * i + 1]);
  return t[0];
}

// ---- key-tile descriptors -----------------------------------------------------------------
// A half (64 key rows) is 16 bits: [15:11] k-frame index in the grid (31: empty half),
// [10:6] tile row, [5:0] tile column.  A tile descriptor = half A | half B << 16.
__device__ __forceinline__ uint32_t half16(const DevGeom& g, int kf, int kt) {
  const int th = kt / g.tiles_w, tw = kt - th * g.tiles_w;
  return ((uint32_t)kf << 11) | ((uint32_t)th << 6) | (uint32_t)tw;
}
__device__ __forceinline__ bool block_single(const DevGeom& g, int kb) { return g.k_tr_count[kb / g.n_tiles] == 1; }
// one selected block on its own: A = its first frame, B = its partner frame or empty
__device__ __forceinline__ uint32_t block_desc(const DevGeom& g, int kb) {
  const int ktr = kb / g.n_tiles, kt = kb - ktr * g.n_tiles;
  const int f0 = g.k_tr_first[ktr];
  const uint32_t b = g.k_tr_count[ktr] == 2 ? half16(g, f0 + 1, kt) : kHalfNone;
  return half16(g, f0, kt) | (b << 16);
}
// two single-frame blocks in one tile
__device__ __forceinline__ uint32_t pair_desc(const DevGeom& g, int kb0, int kb1) {
  const int r0 = kb0 / g.n_tiles, r1 = kb1 / g.n_tiles;
  return half16(g, g.k_tr_first[r0], kb0 - r0 * g.n_tiles) |
         (half16(g, g.k_tr_first[r1], kb1 - r1 * g.n_tiles) << 16);
}
__device__ __forceinline__ bool half_empty(uint32_t h) { return ((h >> 11) & 31u) == 31u; }
// storage offset (in frame-tiles x kUnit) of a half's frame-tile
template <uint32_t kUnit>
__device__ __forceinline__ long long half_offset(const DevGeom& g, uint32_t h) {
  const int kt = (int)((h >> 6) & 31u) * g.tiles_w + (int)(h & 63u);
  return ((long long)g.k_slot[(h >> 11) & 31u] * g.n_tiles + kt) * kUnit;
}

// Locality window (build_locality_mask, P/src/mask.cpp:109-147) from the key side: bit r of the
// result is set when query coordinate p0 + r (r < 8) sees key coordinate k along an axis of
// length F with extent e.  Truncated: |k - p| <= e/2.  Preserved: the window start
// a(p) = clamp(p - e/2, 0, F - e) is monotone in p, so the p with a(p) <= k < a(p) + e are
// (p < e/2 and k < e) | (e/2 <= p <= F - e + e/2 and k - e + e/2 < p <= k + e/2) |
// (p > F - e + e/2 and k >= F - e): at most three intervals.
__device__ __forceinline__ uint32_t bit_interval(int a, int b, int p0) {  // bits of p in [a, b] n [p0, p0+7]
  const int lo = max(a, p0) - p0, hi = min(b, p0 + 7) - p0;
  return lo > hi ? 0u : ((2u << hi) - (1u << lo));
}
__device__ __forceinline__ uint32_t window_bits(int mode, int k, int p0, int e, int F) {
  const int r = e / 2;
  if (mode == 1) return bit_interval(k - r, k + r, p0);
  uint32_t bits = bit_interval(r - e + k + 1, k + r, p0) & bit_interval(r, F - e + r, p0);
  if (k < e) bits |= bit_interval(p0, r - 1, p0);
  if (k >= F - e) bits |= bit_interval(F - e + r + 1, p0 + 7, p0);
  return bits;
}

// MK: token-mask kind (0 all-allowed, 1 locality window, 2 explicit bitmask), fixed at
// compile time so the per-tile mask logic of the other kinds costs nothing.
template <int D, int NQ, int MK>
__global__ void __launch_bounds__(AttnCfg<D, NQ>::kThreads, 1)
    sparse_attn_kernel(const __grid_constant__ DevGeom g, const __grid_constant__ DevMask m,
                       const __grid_constant__ AttnParams p) {
  using Cfg = AttnCfg<D, NQ>;
  constexpr int SW = Cfg::kSW, kNS = Cfg::kNS, CPT = Cfg::kCPT, kGroups = Cfg::kGroups, WG = Cfg::kWG;
  constexpr int kNK = Cfg::kNK, kNV = Cfg::kNV, kNP = Cfg::kNP, kOB = Cfg::kOB, kPB = Cfg::kPB;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for SWIZZLE_128B, by offset so the compiler keeps the shared space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + Cfg::kOffQ;
  uint8_t* sK = smem + Cfg::kOffK;
  uint8_t* sV = smem + Cfg::kOffV;
  uint8_t* sP = smem + Cfg::kOffP;
  uint8_t* scratch = smem + Cfg::kOffS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(scratch);
  // Barrier protocol (one wait and one commit per tile in each MMA issuer):
  //   qk_go[G % NS]   K(G) landed (producer expect_tx + TMA bytes) and S buffer free
  //                   (arrivals of the tile's softmax group after reading S(G - NS))
  //   s_full[G % NS]  QK(G) complete (commit); also frees K stage G % NK for the producer
  //   pv_go[G % PB]   V(G) landed (V producer expect_tx + TMA bytes) and P(G) written
  //   pv_done[G % PB] PV(G) complete (commit); frees V stage and P buffer
  //   o_full / o_empty  per unit: all PVs done / epilogue read O
  //   tab_full[U & 1]  per-unit tables built (epilogue warpgroup, a unit ahead); every role
  //                    walks the units with work through these tables
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* qk_go = bars + 2;
  uint64_t* s_full = qk_go + kNS;
  uint64_t* pv_go = s_full + kNS;
  uint64_t* pv_done = pv_go + kPB;
  uint64_t* o_full = pv_done + kPB;
  uint64_t* o_empty = o_full + 2;
  uint64_t* tab_full = o_empty + 2;
  uint64_t* pv_iss = tab_full + 2;    // [4] PV(G) issued (PV issuer), paces the QK issuer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_iss + 4);
  float* c_s = reinterpret_cast<float*>(scratch + 256);  // [unit parity][group][128] column references
  float* alpha_s = c_s + 512;                            // [group][128] rescale factors
  float* l_s = alpha_s + 256;                            // [unit parity][group][128] denominators
  float* f_s = l_s + 512;                                // [group][128] merge factors (incl. 1/l)
  float* red = f_s + 256;                                // [2][CGg][4][CPT] cross-quarter partials
  // Per-unit tables, double-buffered by unit parity and built a unit ahead by the epilogue warpgroup:
  // locality windows [2][32], tile descriptors [2][kInfoCap], key-norm bounds [2][kInfoCap],
  // query-norm bound [2], initial reference [2]
  int* win2 = reinterpret_cast<int*>(red + 2 * Cfg::kCGg * 4 * CPT);
  uint32_t* info2 = reinterpret_cast<uint32_t*>(win2 + 64);
  float* kn2_2 = reinterpret_cast<float*>(info2 + 2 * kInfoCap);
  float* qn2_2 = kn2_2 + 2 * kInfoCap;
  float* c0_2 = qn2_2 + 2;
  float* cmin_s = c0_2 + 2;                                         // [2][CGg][CPT/32] min reference
  int* utab = reinterpret_cast<int*>(cmin_s + 2 * Cfg::kCGg * (CPT / 32));  // [2][8] tiles head qtr qtile nsel
  uint32_t* prog = reinterpret_cast<uint32_t*>(utab + 16);  // [0] QKs, [1] PVs known complete (count)
  float* kmx = reinterpret_cast<float*>(prog + 2);          // [4] table builder's warp maxima

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // named barriers: 1.. softmax column groups, 9/10 softmax groups, 12 epilogue warpgroup,
  // 13/14 (by unit parity) softmax end of unit -> epilogue
  constexpr int kStatBar0 = 13;
  constexpr int kStatCount = 128 + 32 * kGroups * Cfg::kCGg;
  constexpr int kEpiBar = 12;
  const long long n_units = p.unit_end - p.unit_begin;
  const int units_per_head = p.n_trows * g.n_tiles;

  // unit -> (head, q t_row, tile, selection)
  auto decode = [&](long long u, int& head, int& qtr, int& qtile, int& n, const int*& sel) {
    const long long ug = p.unit_begin + u;
    head = (int)(ug / units_per_head);
    const int rem = (int)(ug - (long long)head * units_per_head);
    qtr = p.trow_list[rem / g.n_tiles];
    qtile = rem % g.n_tiles;
    const long long qb = (long long)head * g.bnq + qtr * g.n_tiles + qtile;
    n = min(max(p.sel_count[qb], 0), p.cap);
    sel = p.sel + qb * p.cap;
  };
  auto sel_at = [&](const int* sel, int t) {
    const int kb = sel[t];
    return kb < 0 ? 0 : (kb >= g.bnk ? g.bnk - 1 : kb);
  };
  // descriptor of tile t of the unit in table slot sl (tables hold the first kInfoCap; a unit
  // with more selected blocks than that runs them unpaired, one block per tile)
  auto desc_at = [&](int sl, int t) -> uint32_t {
    if (t < kInfoCap) return info2[sl * kInfoCap + t];
    const int* sel =
        p.sel + ((long long)utab[sl * 8 + 1] * g.bnq + utab[sl * 8 + 2] * g.n_tiles + utab[sl * 8 + 3]) * p.cap;
    return block_desc(g, sel_at(sel, t));
  };

  // ---- setup ----------------------------------------------------------------------------
  if (warp == Cfg::kQkWarp) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  if (threadIdx.x == 0) {
    prog[0] = 0;
    prog[1] = 0;
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < kNS; ++i) { mbar_init(qk_go + i, WG + 1); mbar_init(s_full + i, 1); }
    for (int i = 0; i < kPB; ++i) { mbar_init(pv_go + i, WG + 1); mbar_init(pv_done + i, 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(o_full + i, 1); mbar_init(o_empty + i, 4); }
    for (int i = 0; i < 2; ++i) mbar_init(tab_full + i, 1);
    for (int i = 0; i < 4; ++i) mbar_init(pv_iss + i, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // setup above overlaps the predecessor (top-k) under programmatic dependent launch
  pdl_trigger();
  pdl_wait();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: S buffers [0, NS*NQ), then O^T buffers [group][unit parity]
  const uint32_t tS0 = tmem, tO0 = tmem + kNS * NQ;

  // K or V tile -> stage: half A rows 0-63, half B rows 64-127 of each 64-channel sub-tile
  auto load_kv = [&](const uint8_t* base_ptr, uint8_t* dst, uint32_t desc, long long head_off, uint64_t* bar) {
    const uint32_t hb = desc >> 16;
    const bool two = !half_empty(hb);
    const uint8_t* a = base_ptr + head_off + half_offset<Cfg::kTileBytes>(g, desc & 0xffffu);
    const uint8_t* b = base_ptr + head_off + (two ? half_offset<Cfg::kTileBytes>(g, hb) : 0);
    mbar_arrive_expect_tx(bar, (two ? 2u : 1u) * Cfg::kTileBytes);
#pragma unroll
    for (int s = 0; s < D / 64; ++s) {
      bulk_g2s(dst + s * 16384, a + s * kSubBytes, kSubBytes, bar);
      if (two) bulk_g2s(dst + s * 16384 + kSubBytes, b + s * kSubBytes, kSubBytes, bar);
    }
  };

  // ================================ epilogue warpgroup ====================================
  // Per-unit tables for every other role (slot U & 1), built a whole unit ahead: the tile
  // list (single-frame blocks paired), key-norm bounds, query-norm bound, initial reference,
  // locality windows, and the unit descriptor (tiles < 0 ends the stream).
  auto build_tables = [&](int sl, int n, int head, int qtr, int qtile, const int* sel) {
    const int et = threadIdx.x - Cfg::kEpiWarp * 32;
    uint32_t* info = info2 + sl * kInfoCap;
    float* kn2_s = kn2_2 + sl * kInfoCap;
    if (n <= kInfoCap) {
      if (et < 32) {
        // Pair runs of consecutive single-frame blocks: within a run, entries at even offsets
        // take the next entry as their B half and entries at odd offsets emit nothing.  One
        // warp, 32 entries per step: ballots give the run offsets, a prefix popcount the slot.
        int out = 0, carry = 0;  // carry: parity of the run of singles crossing into this chunk
        for (int base = 0; base < n; base += 32) {
          const int i = base + lane;
          const int kb = i < n ? sel_at(sel, i) : 0;
          const bool single = i < n && block_single(g, kb);
          const uint32_t sm = __ballot_sync(0xffffffffu, single);
          const uint32_t below = (1u << lane) - 1u;
          const uint32_t zeros = ~sm & below;
          const int off = zeros ? lane - (31 - __clz(zeros)) - 1 : lane + carry;
          const bool follower = single && (off & 1);
          const bool emit = i < n && !follower;
          const uint32_t em = __ballot_sync(0xffffffffu, emit);
          if (emit) {
            int kb1 = -1;
            if (single && i + 1 < n) {
              const int nb = sel_at(sel, i + 1);
              if (block_single(g, nb)) kb1 = nb;
            }
            info[out + __popc(em & below)] = kb1 >= 0 ? pair_desc(g, kb, kb1) : block_desc(g, kb);
          }
          out += __popc(em);
          carry = __shfl_sync(0xffffffffu, single ? off + 1 : 0, 31) & 1;
        }
        if (lane == 0) utab[sl * 8] = out;
      }
    } else {
      for (int i = et; i < kInfoCap; i += 128) info[i] = block_desc(g, sel_at(sel, i));
      if (et == 0) utab[sl * 8] = n;
    }
    named_bar_sync(kEpiBar, 128);
    const int nt = utab[sl * 8];
    float kmax = 0.0f;
    uint32_t nfull = 0;
    for (int i = et; i < min(nt, kInfoCap); i += 128) {
      const uint32_t desc = info[i];
      float kn = INFINITY;
      if (p.kn2) {
        const float* kh = p.kn2 + head * p.kn2_head_stride;
        kn = kh[half_offset<1>(g, desc & 0xffffu)];
        if (!half_empty(desc >> 16)) kn = fmaxf(kn, kh[half_offset<1>(g, desc >> 16)]);
      }
      nfull += half_empty(desc >> 16) ? 0u : 1u;
      kn2_s[i] = kn;
      kmax = fmaxf(kmax, kn);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      kmax = fmaxf(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
      nfull += __shfl_xor_sync(0xffffffffu, nfull, o);
    }
    if (lane == 0) {
      kmx[warp & 3] = kmax;
      if (p.tiles && nfull) atomicAdd(p.tiles + 1, (unsigned long long)nfull);
    }
    named_bar_sync(kEpiBar, 128);
    if (et == 0) {
      kmax = fmaxf(fmaxf(kmx[0], kmx[1]), fmaxf(kmx[2], kmx[3]));
      float qn = INFINITY;
      if (p.qn2) {
        qn = 0.0f;
        for (int f = 0; f < g.q_tr_count[qtr]; ++f)
          qn = fmaxf(qn, p.qn2[head * p.qn2_head_stride + (long long)(g.q_tr_first[qtr] + f) * g.n_tiles + qtile]);
      }
      // Fixed-reference mode: when |q||k| bounds every score of the unit by kFixedBound (log2
      // units), the references start at 0 and never move: p = 2^(s*scale*log2e) stays in
      // [2^-kFixedBound, 2^kFixedBound] (no overflow, no underflow), every tile takes the
      // barrier-free fast path and no first tile needs an exact column max.  Otherwise the
      // references start at -inf (exact lazy-rescale path).
      const float b2 = qn * kmax * (p.scale_log2 * p.scale_log2) * 1.0002f;
      const bool fixed = n <= kInfoCap && b2 <= kFixedBound * kFixedBound;
      if (p.tiles) atomicAdd(p.tiles, (unsigned long long)nt);
      utab[sl * 8 + 1] = head;
      utab[sl * 8 + 2] = qtr;
      utab[sl * 8 + 3] = qtile;
      utab[sl * 8 + 4] = n;
      qn2_2[sl] = qn;
      c0_2[sl] = fixed ? 0.0f : -INFINITY;
      mbar_arrive(tab_full + sl);
    }
  };
  // next unit with work at or after item index k (returns the item index, or -1)
  auto next_work = [&](int k, long long& u, int& head, int& qtr, int& qtile, int& n, const int*& sel) -> int {
    for (;; ++k) {
      if ((long long)blockIdx.x + (long long)k * gridDim.x >= n_units) return -1;
      u = blockIdx.x + (long long)k * gridDim.x;
      decode(u, head, qtr, qtile, n, sel);
      if (n > 0) return k;
    }
  };
  // tables of the work unit after item k into slot sl (or the end-of-stream entry)
  auto build_next = [&](int sl, int& k) {
    long long u;
    int head, qtr, qtile, n;
    const int* sel;
    k = k < 0 ? -1 : next_work(k, u, head, qtr, qtile, n, sel);
    if (k >= 0) {
      build_tables(sl, n, head, qtr, qtile, sel);
      ++k;
    } else if (threadIdx.x == Cfg::kEpiWarp * 32) {
      utab[sl * 8] = -1;
      mbar_arrive(tab_full + sl);
    }
  };
  // the unit in table slot U & 1 (every role but the epilogue walks the units with work this way)
  struct UnitTab {
    int nt, head, qtr, qtile;
  };
  auto wait_unit = [&](int U) {
    const int sl = U & 1;
    mbar_wait(tab_full + sl, (uint32_t)(U >> 1) & 1);
    return UnitTab{utab[sl * 8], utab[sl * 8 + 1], utab[sl * 8 + 2], utab[sl * 8 + 3]};
  };

  // Per unit (same order as every role): wait for both groups' references and denominators
  // (named barrier 13 | 14) and all PVs (o_full), merge the groups' O^T accumulators,
  // O = sum_g 2^(c_g - c) O_g / sum_g 2^(c_g - c) l_g, stage bf16 rows and bulk-store them.
  // Runs beside the softmax warps, which move on to the next unit at once.
  auto epilogue_warps = [&]() {
    const int q4 = warp & 3;                   // TMEM lane quarter = channel rows 32*q4..
    const int et = threadIdx.x - Cfg::kEpiWarp * 32;
    const int dj = q4 * 32 + lane;             // output channel of this lane
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    constexpr int kEC = Cfg::kEpiCols;
    uint16_t* stage = reinterpret_cast<uint16_t*>(smem + Cfg::kOffE);  // [kEC][D] bf16
    int kb = 0;  // item index from which the next table is searched (-1: stream ended)
    build_next(0, kb);
    build_next(1, kb);
    int U = 0;
    for (long long u = blockIdx.x; u < n_units; u += gridDim.x) {
      int head, qtr, qtile, n;
      const int* sel;
      decode(u, head, qtr, qtile, n, sel);
      const int qf0 = g.q_tr_first[qtr];
      const int qh0 = 8 * (qtile / g.tiles_w), qw0 = 8 * (qtile % g.tiles_w);
      const int cv = min(8, g.cols - qw0);   // real tokens per tile row
      // first token of tile row r (0-7) of q frame f (0-1) of this unit
      auto row_tok = [&](int f, int r) { return g.q_frame_tok0[qf0 + f] + (long long)(qh0 + r) * g.cols + qw0; };
      if (n == 0) {  // no selected block: the unit's real rows are zero
        constexpr int kChunks = D / 8;
        for (int idx = et; idx < NQ * kChunks; idx += 128) {
          const int col = idx / kChunks, ch = idx % kChunks, qc = col & 63;
          if (qh0 + (qc >> 3) >= g.rows || (qc & 7) >= cv) continue;
          uint16_t* row = p.out_tile_major
                              ? p.out + (u * NQ + col) * D
                              : p.out + head * p.out_head_stride +
                                    (row_tok(col >> 6, qc >> 3) + (qc & 7)) * (p.out_token_stride ? p.out_token_stride : D);
          *reinterpret_cast<uint4*>(row + ch * 8) = make_uint4(0, 0, 0, 0);
        }
        continue;
      }
      const int par = U & 1;
      // hardware barrier, not an mbarrier: the epilogue waits most of a unit here and a parked
      // warp costs no issue slots (ids alternate by unit parity: the softmax cannot run two
      // units ahead, it needs the tables this epilogue releases)
      named_bar_sync(kStatBar0 + par, kStatCount);
      // merge factors per query column: f_g = 2^(c_g - c) / l, l = sum_g l_g 2^(c_g - c);
      // zero for columns outside [row_begin, row_end) (their rows are written as zeros)
      if (et < NQ) {
        float cmax = -INFINITY;
#pragma unroll
        for (int gi = 0; gi < kGroups; ++gi) cmax = fmaxf(cmax, c_s[(par * 2 + gi) * 128 + et]);
        float e[kGroups], l = 0.0f;
#pragma unroll
        for (int gi = 0; gi < kGroups; ++gi) {
          const float lg = l_s[(par * 2 + gi) * 128 + et];
          e[gi] = lg > 0.0f ? ex2(c_s[(par * 2 + gi) * 128 + et] - cmax) : 0.0f;
          l += lg * e[gi];
        }
        const int qc = et & 63;
        bool inr = false;
        if (qh0 + (qc >> 3) < g.rows && (qc & 7) < cv) {
          const long long tq = row_tok(et >> 6, qc >> 3) + (qc & 7);
          inr = tq >= p.row_begin && tq < p.row_end;
          if (inr && !(l > 0.0f)) atomicOr(p.err, kErrDegenerate);
        }
#pragma unroll
        for (int gi = 0; gi < kGroups; ++gi) f_s[gi * 128 + et] = (inr && l > 0.0f) ? e[gi] / l : 0.0f;
      }
      mbar_wait_sleep(o_full + par, (uint32_t)(U >> 1) & 1, 128);
      tc_fence_after();
      named_bar_sync(kEpiBar, 128);  // factors visible
      // O in chunks of kEC query columns: TMEM -> merged bf16 -> staging -> bulk store
#pragma unroll 1
      for (int c0 = 0; c0 < NQ; c0 += kEC) {
        float acc[kEC];
#pragma unroll
        for (int i = 0; i < kEC; ++i) acc[i] = 0.0f;
#pragma unroll
        for (int gi = 0; gi < kGroups; ++gi) {
          uint32_t o[kEC];
          tmem_ld<kEC>(tO0 + (gi * kOB + par) * NQ + c0 + lane_off, o);
          tc_wait_ld();
          const float* fg = f_s + gi * 128 + c0;
#pragma unroll
          for (int i = 0; i < kEC; i += 4) {
            const float4 f4 = *reinterpret_cast<const float4*>(fg + i);
            // a group without tiles in this unit has f = 0 and an undefined accumulator
            if (f4.x != 0.0f) acc[i] = fmaf(__uint_as_float(o[i]), f4.x, acc[i]);
            if (f4.y != 0.0f) acc[i + 1] = fmaf(__uint_as_float(o[i + 1]), f4.y, acc[i + 1]);
            if (f4.z != 0.0f) acc[i + 2] = fmaf(__uint_as_float(o[i + 2]), f4.z, acc[i + 2]);
            if (f4.w != 0.0f) acc[i + 3] = fmaf(__uint_as_float(o[i + 3]), f4.w, acc[i + 3]);
          }
        }
        if (et == 0) bulk_wait_read();  // the previous chunk's stores have read the staging
        named_bar_sync(kEpiBar, 128);
        if (dj < D) {
#pragma unroll
          for (int i = 0; i < kEC; ++i) stage[i * D + dj] = __bfloat16_as_ushort(__float2bfloat16_rn(acc[i]));
        }
        fence_proxy_async_smem();
        named_bar_sync(kEpiBar, 128);
        if (et == 0) {
          if (p.out_tile_major) {
            bulk_s2g(p.out + (u * NQ + c0) * D, stage, kEC * D * 2);
          } else {
            // the chunk's tile rows: cv consecutive tokens each (one copy per row when the
            // tokens are contiguous, else one per token)
            const long long ots = p.out_token_stride ? p.out_token_stride : D;
#pragma unroll 1
            for (int r0 = c0; r0 < c0 + kEC; r0 += 8) {
              const int qc = r0 & 63;
              if (qh0 + (qc >> 3) >= g.rows) continue;
              uint16_t* dst = p.out + head * p.out_head_stride + row_tok(r0 >> 6, qc >> 3) * ots;
              if (ots == D) {
                bulk_s2g(dst, stage + (r0 - c0) * D, cv * D * 2);
              } else {
                for (int w = 0; w < cv; ++w) bulk_s2g(dst + w * ots, stage + (r0 - c0 + w) * D, D * 2);
              }
            }
          }
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty + par);   // O^T buffers of this parity free for unit U + 2
      // slot par (tables, c, l) is free: every role finished unit U; build unit U + 2's tables
      named_bar_sync(kEpiBar, 128);
      build_next(par, kb);
      ++U;
    }
    if (et == 0) bulk_wait_all();
  };

  if (warp >= SW) {
  reg_dealloc<Cfg::kRegOther>();
  if (warp == Cfg::kProducerWarp) {
    // ================================ Q / K producer (warp-wide) =========================
    int T = 0;  // tiles of this CTA so far
    for (int U = 0;; ++U) {
      const UnitTab ut = wait_unit(U);
      if (ut.nt < 0) break;
      const int sl = U & 1;
      if (U >= 1) mbar_wait(q_empty, (U - 1) & 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(q_full, Cfg::kQBytes);
        const int f0 = g.q_tr_first[ut.qtr];
        const uint8_t* qa = p.q + ut.head * p.q_head_stride + ((long long)f0 * g.n_tiles + ut.qtile) * Cfg::kTileBytes;
#pragma unroll
        for (int s = 0; s < D / 64; ++s) {
          bulk_g2s(sQ + s * Cfg::kQSub, qa + s * kSubBytes, kSubBytes, q_full);
          if (NQ == 128)
            bulk_g2s(sQ + s * Cfg::kQSub + kSubBytes, qa + (long long)g.n_tiles * Cfg::kTileBytes + s * kSubBytes,
                     kSubBytes, q_full);
        }
      }
      __syncwarp();
      // the next unit's Q into L2 now if its table is built: its load waits for this unit's
      // last QK and would otherwise pay the full HBM latency between units
      {
        const int nsl = sl ^ 1;
        if (lane < 2 && mbar_test(tab_full + nsl, (uint32_t)((U + 1) >> 1) & 1) && utab[nsl * 8] > 0) {
          const int nqtr = utab[nsl * 8 + 2];
          if (lane < g.q_tr_count[nqtr])
            bulk_prefetch_l2(p.q + utab[nsl * 8 + 1] * p.q_head_stride +
                                 ((long long)(g.q_tr_first[nqtr] + lane) * g.n_tiles + utab[nsl * 8 + 3]) *
                                     Cfg::kTileBytes,
                             Cfg::kTileBytes);
        }
      }
      const long long hoff = ut.head * p.kv_head_stride;
      for (int t = 0; t < ut.nt; ++t, ++T) {
        const uint32_t desc = desc_at(sl, t);
        const int ks = T % kNK;
        // K stage ks is free once QK(T - NK) completed
        if (T >= kNK) {
          mbar_wait(s_full + (T - kNK) % kNS, (uint32_t)((T - kNK) / kNS) & 1);
          if (lane == 0) st_release_shared(prog + 0, (uint32_t)(T - kNK + 1));  // QKs complete
        }
        if (elect_one()) load_kv(p.k, sK + ks * Cfg::kKVBytes, desc, hoff, qk_go + T % kNS);
        __syncwarp();
      }
    }
  } else if (warp == Cfg::kVProducerWarp) {
    // ================================ V producer (warp-wide) =============================
    int T = 0;
    for (int U = 0;; ++U) {
      const UnitTab ut = wait_unit(U);
      if (ut.nt < 0) break;
      const long long hoff = ut.head * p.kv_head_stride;
      for (int t = 0; t < ut.nt; ++t, ++T) {
        const uint32_t desc = desc_at(U & 1, t);
        const int vs = T % kNV;
        // V stage vs is free once PV(T - NV) completed
        if (T >= kNV) {
          mbar_wait(pv_done + (T - kNV) % kPB, (uint32_t)((T - kNV) / kPB) & 1);
          if (lane == 0) st_release_shared(prog + 1, (uint32_t)(T - kNV + 1));  // PVs complete
        }
        if (elect_one()) load_kv(p.v, sV + vs * Cfg::kKVBytes, desc, hoff, pv_go + T % kPB);
        __syncwarp();
      }
    }
  } else if (warp == Cfg::kQkWarp) {
    // ================================ QK^T issuer (warp-wide, elected lane issues) =========
    // S^T(G) = K(G) . Q^T into S buffer G % NS once K(G) landed and the buffer is free
    // (qk_go); runs ahead of the softmax by up to NS tiles, paced by PV issue (kQkLead).
    constexpr uint32_t idesc_qk = umma_idesc_bf16(128, NQ, 0, 0);
    const uint32_t aQ = smem_u32(sQ);
    const uint32_t aK0 = smem_u32(sK);
    int G = 0, sb = 0, ks = 0;
    uint32_t sph = 0;
    for (int U = 0;; ++U) {
      const UnitTab ut = wait_unit(U);
      if (ut.nt < 0) break;
      mbar_wait(q_full, U & 1);
      for (int t = 0; t < ut.nt; ++t, ++G) {
        if (G >= kQkLead) mbar_wait(pv_iss + (G - kQkLead) % 4, (uint32_t)((G - kQkLead) / 4) & 1);
        mbar_wait(qk_go + sb, sph);
        tc_fence_after();
        const uint32_t aK = aK0 + ks * Cfg::kKVBytes;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t da = umma_desc_sw128(aK + (kk >> 2) * 16384 + (kk & 3) * 32, 16u, 1024u);
            const uint64_t db = umma_desc_sw128(aQ + (kk >> 2) * Cfg::kQSub + (kk & 3) * 32, 16u, 1024u);
            tc_mma_f16(tS0 + sb * NQ, da, db, idesc_qk, kk > 0 ? 1u : 0u);
          }
          tc_commit(s_full + sb);
          if (t == ut.nt - 1) tc_commit(q_empty);
        }
        __syncwarp();
        if (++sb == kNS) { sb = 0; sph ^= 1u; }
        if (++ks == kNK) ks = 0;
      }
    }
  } else if (warp == Cfg::kPvWarp) {
    // ================================ PV issuer (warp-wide, elected lane issues) ==========
    // O^T[group(t)] += V(G)^T . P(G)^T once V(G) landed and the softmax wrote P(G) (pv_go).
    constexpr uint32_t idesc_pv = umma_idesc_bf16(128, NQ, 1, 1);
    const uint32_t aV0 = smem_u32(sV), aP0 = smem_u32(sP);
    int G = 0, vs = 0, pb = 0, gb = 0;
    uint32_t gph = 0;
    for (int U = 0;; ++U) {
      const UnitTab ut = wait_unit(U);
      if (ut.nt < 0) break;
      const int ob = U & 1;
      if (U >= 2) mbar_wait(o_empty + ob, ((U >> 1) - 1) & 1);  // epilogue of unit U-2 done
      for (int t = 0; t < ut.nt; ++t, ++G) {
        const bool full = !half_empty(desc_at(U & 1, t) >> 16);  // 128 key rows (else rows 0-63)
        const uint32_t tO = tO0 + ((t % kGroups) * kOB + ob) * NQ;
        mbar_wait(pv_go + gb, gph);
        tc_fence_after();
        const uint32_t aV = aV0 + vs * Cfg::kKVBytes;
        const uint32_t aP = aP0 + pb * Cfg::kPBytes;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            if (kk < 4 || full) {  // a 64-row tile has 4 valid K=16 steps
              const uint64_t da = umma_desc_sw128(aV + kk * 2048, D == 128 ? 16384u : 0u, 1024u);
              const uint64_t db = umma_desc_sw128(aP + kk * 2048, 16384u, 1024u);
              // the first tile of each group in the unit overwrites its O^T buffer
              tc_mma_f16(tO, da, db, idesc_pv, (t >= kGroups || kk > 0) ? 1u : 0u);
            }
          }
          tc_commit(pv_done + gb);
          if (t == ut.nt - 1) tc_commit(o_full + ob);
          mbar_arrive(pv_iss + G % 4);
        }
        __syncwarp();
        if (++gb == kPB) { gb = 0; gph ^= 1u; }
        if (++vs == kNV) vs = 0;
        if (++pb == kNP) pb = 0;
      }
    }
  } else {
    epilogue_warps();
  }
  } else {
    reg_alloc<Cfg::kRegSoftmax>();
    // ===================================== softmax warps ================================
    // Group grp handles the tiles t of a unit with t % kGroups == grp (ping-pong: the two
    // groups' latencies overlap) with its own running references and O^T accumulator.
    const int grp = warp / WG, wl = warp % WG;
    const int quarter = warp & 3, cg = wl >> 2;
    const int j = quarter * 32 + lane;  // key row == TMEM lane
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int col0 = cg * CPT;          // first of this thread's CPT query columns
    const int bar_id = 1 + grp * 4 + cg;  // named barrier of the column group (128 threads)
    const int grp_bar = 9 + grp;          // named barrier of the group
    constexpr int kW = CPT / 32;
    float* cg_a = alpha_s + grp * 128;
    float* cg_red = red + (grp * Cfg::kCGg + cg) * 4 * CPT;
    if (lane == 0)
      for (int i = grp; i < kNS; i += kGroups) mbar_arrive(qk_go + i);  // S buffers start free
    int T = 0;
    // Units with work, from the per-unit tables (slot U & 1); an entry with tiles < 0 ends the
    // stream.  Empty units are the epilogue warps' alone.
    for (int U = 0;; ++U) {
      const int tsl = U & 1;
      const UnitTab ut = wait_unit(U);
      const int n = ut.nt;
      if (n < 0) break;
      const int qtr = ut.qtr, qtile = ut.qtile;
      const int qf0 = g.q_tr_first[qtr];
      const int qh0 = 8 * (qtile / g.tiles_w), qw0 = 8 * (qtile % g.tiles_w);
      const float* kn2_s = kn2_2 + tsl * kInfoCap;
      const float* qn2_s = qn2_2 + tsl;
      // this group's references (and their word minima) start at the unit's initial value;
      // the epilogue of unit U - 2 (same slot) released them with the tables
      float* cg_c = c_s + (tsl * 2 + grp) * 128;
      // references 0 for the whole unit (every tile of it then fits the bound)
      const bool fixed_unit = c0_2[tsl] == 0.0f;
      {
        const float c0v = c0_2[tsl];
        for (int i = wl * 32 + lane; i < NQ; i += WG * 32) cg_c[i] = c0v;
        if (wl == 0 && lane < Cfg::kCGg * kW) cmin_s[grp * Cfg::kCGg * kW + lane] = c0v;
        named_bar_sync(grp_bar, WG * 32);
      }
      // query columns of this thread that are real tokens, as 32-column words: rows of the
      // 8x8 tile below g.rows times columns left of g.cols (both frames of NQ = 128 alike)
      uint32_t qvalid[kW];
      {
        const int rv = min(8, g.rows - qh0), cv = min(8, g.cols - qw0);
        const unsigned long long rowbits = (cv >= 8 ? 0xffull : ((1ull << cv) - 1ull)) * 0x0101010101010101ull;
        const unsigned long long vm = rv >= 8 ? rowbits : (rowbits & ((1ull << (8 * rv)) - 1ull));
#pragma unroll
        for (int w = 0; w < kW; ++w) qvalid[w] = (uint32_t)(vm >> (((col0 + 32 * w) & 63)));
      }
      uint32_t my_pairs = 0;  // <= tiles * CPT per thread per unit
      float lp[CPT];
#pragma unroll
      for (int i = 0; i < CPT; ++i) lp[i] = 0.0f;
      const int ob = U & 1;
      const uint32_t tO = tO0 + (grp * kOB + ob) * NQ;
      // tile t of a unit belongs to group t % kGroups whatever the CTA ran before, so a unit's
      // output is a function of the unit alone (sharded == unsharded, bit for bit)
      const int t_first = grp;
      bool any = false;  // this group processed a tile of the unit (its O^T is defined)

      uint32_t inf_next = t_first < n ? desc_at(tsl, t_first) : 0u;  // prefetched a tile ahead
      // The tile loop, compiled twice: for fixed-reference units (references 0, every tile on
      // the fast path: no vote, no rescale, no reference loads -- a compact hot loop) and for
      // the general case.
      auto tile_loop = [&](auto fixed_tag) {
        constexpr bool kFixed = decltype(fixed_tag)::value;
        for (int t = t_first; t < n; t += kGroups) {
          const int G = T + t;
          const int sb = G % kNS, pb = G % kNP;
          // ---- key row j: validity and allowed-query mask over this thread's columns ----
          const uint32_t inf = inf_next;
          if (t + kGroups < n) inf_next = desc_at(tsl, t + kGroups);
          const uint32_t hd = j < 64 ? (inf & 0xffffu) : (inf >> 16);  // warp-uniform half
          const int kf = (int)((hd >> 11) & 31u);
          const int kh = (int)((hd >> 6) & 31u) * 8 + ((j & 63) >> 3);
          const int kw = (int)(hd & 63u) * 8 + (j & 7);
          const bool kvalid = kf != 31 && kh < g.rows && kw < g.cols;
          uint32_t mk[kW];  // bit i of word w: (key j, column col0 + 32w + i) allowed
#pragma unroll
          for (int w = 0; w < kW; ++w) mk[w] = 0;
          if (kvalid) {
            if (MK == 0) {
#pragma unroll
              for (int w = 0; w < kW; ++w) mk[w] = qvalid[w];
            } else if (MK == 1) {
              // allowed query cols / rows of the 8x8 query tile, closed form (window_bits)
              const uint32_t hb = window_bits(m.mode, kh, qh0, m.extent_h, g.rows);
              const uint32_t wb = window_bits(m.mode, kw, qw0, m.extent_w, g.cols);
              // 64-bit tile mask: byte r (query tile row r) = wb where hb has bit r (bit r of
              // hb spread to byte r, then any nonzero byte widened to 0xff without carries)
              unsigned long long rows64 = ((unsigned long long)(hb & 0xffu) * 0x0101010101010101ull) &
                                          0x8040201008040201ull;
              rows64 = (((rows64 + 0x7f7f7f7f7f7f7f7full) | rows64) & 0x8080808080808080ull) >> 7;
              rows64 *= 0xffull;
              const unsigned long long m64 = rows64 & ((unsigned long long)wb * 0x0101010101010101ull);
#pragma unroll
              for (int w = 0; w < kW; ++w) mk[w] = (uint32_t)(m64 >> ((col0 + 32 * w) & 63)) & qvalid[w];
            } else {
              const long long tk = g.k_frame_tok0[kf] + (long long)kh * g.cols + kw;
#pragma unroll
              for (int w = 0; w < kW; ++w) {
#pragma unroll 4
                for (int i = 0; i < 32; ++i) {
                  if (!((qvalid[w] >> i) & 1u)) continue;
                  const int col = col0 + 32 * w + i, qc = col & 63;
                  const long long tq =
                      g.q_frame_tok0[qf0 + (col >> 6)] + (long long)(qh0 + (qc >> 3)) * g.cols + qw0 + (qc & 7);
                  if ((m.bits[tq * m.words_per_row + (tk >> 6)] >> (tk & 63)) & 1ull) mk[w] |= 1u << i;
                }
              }
            }
          }
#pragma unroll
          for (int w = 0; w < kW; ++w) my_pairs += __popc(mk[w]);
          any = true;

          // MN-major B operand: [NQ/64 groups][128 key rows][128 B], 16-B chunks swizzled by row
          uint8_t* prow = sP + pb * Cfg::kPBytes + j * 128;
          const float sl2 = p.scale_log2;
          // Fast path: |q||k| bounds every score of the tile within kBoundSlack of each word's
          // smallest reference, so no reference can need to move — no vote, no barrier, no
          // memory-clobbering asm between the words, so their loads and math interleave.  The
          // decision uses only shared inputs: all 4 warps of a column group take the same path.
          // (Fixed-reference units: always.)
          bool fast = kFixed || t < kInfoCap;
          if (!kFixed && fast) {
            const float b2 = qn2_s[0] * kn2_s[t] * (sl2 * sl2) * 1.0002f;
#pragma unroll
            for (int w = 0; w < kW; ++w) {
              const float lim = kBoundSlack + cmin_s[(grp * Cfg::kCGg + cg) * kW + w];
              fast = fast && lim > 0.0f && b2 <= lim * lim;
            }
          }
          // S(G) ready: the Q/K producer publishes the QKs it saw complete (it waits on them to
          // recycle K stages, normally well before this tile), else wait on the barrier itself
          if (ld_acquire_shared(prog + 0) <= (uint32_t)G) mbar_wait(s_full + sb, (uint32_t)(G / kNS) & 1);
          tc_fence_after();
          if (fast) {
            // P buffer pb was last read by PV(G - NP) (kNP tiles back: normally long done, and
            // published by the V producer, which waits on PVs to recycle V stages), so each
            // word's P^T is stored as soon as it is computed, under the next word's exps
            // (one P buffer per group, NQ = 128: PV(G - 1) is the previous tile's, so the
            // wait moves behind the exps and the stores follow all words)
            constexpr bool kEarlyP = kNP > kGroups;
            if constexpr (kEarlyP) {
              if (G >= kNP && ld_acquire_shared(prog + 1) <= (uint32_t)(G - kNP))
                mbar_wait(pv_done + (G - kNP) % kPB, (uint32_t)((G - kNP) / kPB) & 1);
            }
            uint32_t pk[CPT / 2];
#pragma unroll
            for (int w = 0; w < kW; ++w) {
              const uint32_t mw = mk[w];
              const float* cw = cg_c + col0 + 32 * w;
              float d[32];
              tmem_ld<32>(tS0 + sb * NQ + col0 + 32 * w + lane_off, reinterpret_cast<uint32_t*>(d));
              tc_wait_ld();
              if (mw == 0u) {
#pragma unroll
                for (int i = 0; i < 16; ++i) pk[16 * w + i] = 0u;
              } else {
                if (kFixed && (MK != 0 || mw == 0xffffffffu)) {
                  // references fixed at 0: d = s * scale * log2(e) in packed pairs; with a token
                  // mask a partially allowed word then sends its masked columns to -inf (exp 0).
                  // (All-allowed units keep the select-in-FFMA form below for edge-tile words:
                  // the hot loop of the headline compiles best that way.)
#pragma unroll
                  for (int i = 0; i < 16; ++i) fmul2(d[2 * i], d[2 * i + 1], sl2);
                  if (MK != 0 && mw != 0xffffffffu) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) d[i] = ((mw >> i) & 1u) ? d[i] : -INFINITY;
                  }
                } else {
#pragma unroll
                  for (int i = 0; i < 32; i += 4) {
                    const float4 c4 = kFixed ? make_float4(0.f, 0.f, 0.f, 0.f)
                                             : *reinterpret_cast<const float4*>(cw + i);
                    d[i] = ((mw >> i) & 1u) ? fmaf(d[i], sl2, -c4.x) : -INFINITY;
                    d[i + 1] = ((mw >> (i + 1)) & 1u) ? fmaf(d[i + 1], sl2, -c4.y) : -INFINITY;
                    d[i + 2] = ((mw >> (i + 2)) & 1u) ? fmaf(d[i + 2], sl2, -c4.z) : -INFINITY;
                    d[i + 3] = ((mw >> (i + 3)) & 1u) ? fmaf(d[i + 3], sl2, -c4.w) : -INFINITY;
                  }
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const float p0 = ex2(d[2 * i]);
                  const float p1 = ex2(d[2 * i + 1]);
                  fadd2(lp[32 * w + 2 * i], lp[32 * w + 2 * i + 1], p0, p1);
                  const __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                  pk[16 * w + i] = *reinterpret_cast<const uint32_t*>(&h2);
                }
              }
              if constexpr (kEarlyP) {
                const int cwi = col0 + 32 * w;
                uint8_t* pw = prow + (cwi >> 6) * 16384;
                const int ch0 = (cwi & 63) >> 3;
#pragma unroll
                for (int c8 = 0; c8 < 4; ++c8)
                  *reinterpret_cast<uint4*>(pw + (((ch0 + c8) ^ (j & 7)) << 4)) =
                      make_uint4(pk[16 * w + 4 * c8], pk[16 * w + 4 * c8 + 1], pk[16 * w + 4 * c8 + 2],
                                 pk[16 * w + 4 * c8 + 3]);
              }
            }
            if constexpr (!kEarlyP) {
              if (G >= kNP && ld_acquire_shared(prog + 1) <= (uint32_t)(G - kNP))
                mbar_wait(pv_done + (G - kNP) % kPB, (uint32_t)((G - kNP) / kPB) & 1);
#pragma unroll
              for (int w = 0; w < kW; ++w) {
                const int cwi = col0 + 32 * w;
                uint8_t* pw = prow + (cwi >> 6) * 16384;
                const int ch0 = (cwi & 63) >> 3;
#pragma unroll
                for (int c8 = 0; c8 < 4; ++c8)
                  *reinterpret_cast<uint4*>(pw + (((ch0 + c8) ^ (j & 7)) << 4)) =
                      make_uint4(pk[16 * w + 4 * c8], pk[16 * w + 4 * c8 + 1], pk[16 * w + 4 * c8 + 2],
                                 pk[16 * w + 4 * c8 + 3]);
              }
            }
          } else {
            // Columns in 32-wide words: each word is loaded, exponentiated and stored on its own
            // (32 live scores per thread); its columns have their own references and vote.
#pragma unroll
            for (int w = 0; w < kW; ++w) {
              const int cw = col0 + 32 * w;                // first column of the word
              const uint32_t tS = tS0 + sb * NQ + cw + lane_off;
              float d[32];  // scores -> exponents -> probabilities
              tmem_ld<32>(tS, reinterpret_cast<uint32_t*>(d));
              tc_wait_ld();
              uint32_t pk[16];
              // d = s*scale*log2(e) - c (one FFMA; c = -inf before a column's first key gives
              // +inf, which forces the exact path); masked entries -> -inf (ex2 -> 0).  The mask
              // word is warp-uniform except on ragged edge tiles: all-allowed / none / mixed.
              const uint32_t mw = mk[w];
              if (mw == 0xffffffffu) {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                  const float4 c4 = *reinterpret_cast<const float4*>(cg_c + cw + i);
                  d[i] = fmaf(d[i], sl2, -c4.x);
                  d[i + 1] = fmaf(d[i + 1], sl2, -c4.y);
                  d[i + 2] = fmaf(d[i + 2], sl2, -c4.z);
                  d[i + 3] = fmaf(d[i + 3], sl2, -c4.w);
                }
              } else if (mw == 0u) {
#pragma unroll
                for (int i = 0; i < 32; ++i) d[i] = -INFINITY;
              } else {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                  const float4 c4 = *reinterpret_cast<const float4*>(cg_c + cw + i);
                  d[i] = ((mw >> i) & 1u) ? fmaf(d[i], sl2, -c4.x) : -INFINITY;
                  d[i + 1] = ((mw >> (i + 1)) & 1u) ? fmaf(d[i + 1], sl2, -c4.y) : -INFINITY;
                  d[i + 2] = ((mw >> (i + 2)) & 1u) ? fmaf(d[i + 2], sl2, -c4.z) : -INFINITY;
                  d[i + 3] = ((mw >> (i + 3)) & 1u) ? fmaf(d[i + 3], sl2, -c4.w) : -INFINITY;
                }
              }
              const bool need = bar_red_or(bar_id, 128, mw != 0u && tree_max<32>(d) > kRescaleThreshold);
              if (need) {
                // exact column max of this tile over the group's 128 key rows, from the raw scores
                tmem_ld<32>(tS, reinterpret_cast<uint32_t*>(d));
                tc_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) d[i] = ((mk[w] >> i) & 1u) ? d[i] * sl2 : -INFINITY;
                warp_colreduce<32, true>(d, lane);
                cg_red[quarter * 32 + lane] = d[0];
                named_bar_sync(bar_id, 128);
                if (quarter == 0) {
                  const float mx = fmaxf(fmaxf(cg_red[lane], cg_red[32 + lane]), fmaxf(cg_red[64 + lane], cg_red[96 + lane]));
                  const float cold = cg_c[cw + lane];
                  const float nw = fmaxf(cold, mx);
                  cg_c[cw + lane] = nw;
                  cg_a[cw + lane] = (nw == -INFINITY) ? 1.0f : ex2(cold - nw);
                  float mn = nw;
#pragma unroll
                  for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                  if (lane == 0) cmin_s[(grp * Cfg::kCGg + cg) * kW + w] = mn;
                }
                named_bar_sync(bar_id, 128);
                tmem_ld<32>(tS, reinterpret_cast<uint32_t*>(d));
                tc_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  lp[32 * w + i] *= cg_a[cw + i];
                  d[i] = ((mk[w] >> i) & 1u) ? fmaf(d[i], sl2, -cg_c[cw + i]) : -INFINITY;
                }
                if (t >= kGroups) {
                  // O^T holds this group's PVs of the unit: wait for its last one, rescale columns
                  const int Gp = G - kGroups;
                  mbar_wait(pv_done + Gp % kPB, (uint32_t)(Gp / kPB) & 1);
                  tc_fence_after();
                  if (j < D) {
                    uint32_t o[32];
                    tmem_ld<32>(tO + cw + lane_off, o);
                    tc_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * cg_a[cw + i]);
                    tmem_st<32>(tO + cw + lane_off, o);
                    tc_wait_st();
                  }
                }
              }
              // ---- P^T row j (bf16) and partial denominators (fp32) -------------------------
              if (mw == 0u) {  // key row j of this tile is padding / masked for every column
#pragma unroll
                for (int i = 0; i < 16; ++i) pk[i] = 0u;
              } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const float p0 = ex2(d[2 * i]);
                  const float p1 = ex2(d[2 * i + 1]);
                  lp[32 * w + 2 * i] += p0;
                  lp[32 * w + 2 * i + 1] += p1;
                  const __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                  pk[i] = *reinterpret_cast<const uint32_t*>(&h2);
                }
              }
              // P buffer pb was last read by PV(G - NP)
              if (w == 0 && G >= kNP) mbar_wait(pv_done + (G - kNP) % kPB, (uint32_t)((G - kNP) / kPB) & 1);
              uint8_t* pw = prow + (cw >> 6) * 16384;
              const int ch0 = (cw & 63) >> 3;
#pragma unroll
              for (int c8 = 0; c8 < 4; ++c8)
                *reinterpret_cast<uint4*>(pw + (((ch0 + c8) ^ (j & 7)) << 4)) =
                    make_uint4(pk[4 * c8], pk[4 * c8 + 1], pk[4 * c8 + 2], pk[4 * c8 + 3]);
            }
          }
          // S buffer free for QK(G + NS); P(G) visible to the tensor core
          tc_fence_before();
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(qk_go + sb);
            mbar_arrive(pv_go + G % kPB);
          }
        }
      };
      if (fixed_unit) tile_loop(std::true_type{}); else tile_loop(std::false_type{});

      // ---- end of unit: this group's denominators -> the epilogue warpgroup -------------
      if (p.pairs) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) my_pairs += __shfl_xor_sync(0xffffffffu, my_pairs, o);
        if (lane == 0 && my_pairs) atomicAdd(p.pairs, (unsigned long long)my_pairs);
      }
      warp_colreduce<CPT, false>(lp, lane);
#pragma unroll
      for (int i = 0; i < CPT / 32; ++i) cg_red[quarter * CPT + colreduce_col(CPT, lane, i)] = lp[i];
      named_bar_sync(bar_id, 128);
      if (quarter == 0) {
        float* lg = l_s + (tsl * 2 + grp) * 128 + col0;
#pragma unroll
        for (int i = 0; i < CPT / 32; ++i) {
          const int cc = lane + 32 * i;
          lg[cc] = any ? (cg_red[cc] + cg_red[CPT + cc]) + (cg_red[2 * CPT + cc] + cg_red[3 * CPT + cc]) : 0.0f;
        }
        named_bar_arrive(kStatBar0 + tsl, kStatCount);  // references (written by quarter 0) and l final
      }
      T += n;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == Cfg::kQkWarp) tmem_dealloc(tmem, Cfg::kTmemCols);
}

}  // namespace fvsr

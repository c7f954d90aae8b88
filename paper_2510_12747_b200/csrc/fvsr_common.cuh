// fvsr_common.cuh — shared device definitions for the sm_100a kernels.
//
// Storage unit: the FRAME-TILE.  The reference tiles tokens into (2,8,8) blocks
// keyed by (frame/2, h/8, w/8) over absolute frame ids (P/src/partition.cpp:38-62,
// P = /root/reference/proj).  A block is therefore one or two 8x8 spatial tiles of
// consecutive frames 2m, 2m+1.  We store every frame's 8x8 tile as a contiguous
// 64-row x d bf16 "frame-tile" (ragged tiles zero-padded), pre-swizzled in HBM in the
// exact UMMA canonical K-major SWIZZLE_128B layout, so one cp.async.bulk moves it into
// shared memory ready for tcgen05.mma:
//     frame-tile = [d/64 sub-tiles][64 rows][64 bf16]   (8 KB per sub-tile)
//     byte(row r, chan c) = (c/64)*8192 + r*128 + (((c%64)/8) ^ (r%8))*16 + (c%8)*2
// Row r of a frame-tile is spatial (8*th + r/8, 8*tw + r%8) of that frame.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda.h>  // CUtensorMap (the driver entry point is resolved at run time)
#include <cuda_runtime.h>

namespace fvsr {

constexpr int kMaxFrames = 32;      // frames per grid in one call
constexpr int kTileRows = 64;       // 8x8 tokens per frame-tile
constexpr int kSubBytes = 64 * 128; // one 64-row x 64-channel bf16 sub-tile

enum : uint32_t {
  kErrShape = 1u << 1,
  kErrConfig = 1u << 2,
  kErrDegenerate = 1u << 3,
  kErrEmptyBlock = 1u << 4,
  kErrInvariant = 1u << 5,
};

// Token-mask descriptor as the kernels see it (fvsr_mask + frame extents).
struct DevMask {
  int kind;      // 0 all, 1 locality, 2 bitmask
  int mode;      // 0 preserved, 1 truncated
  int extent_h, extent_w;
  int frame_h, frame_w;
  const uint64_t* bits;
  long long words_per_row;
};

// Geometry of one (grid_q, grid_k) pair.  Blocks are numbered t_row-major then tile
// (tile = h_tile * tiles_w + w_tile), which is exactly the lexicographic key order of
// partition_blocks because every present t_row covers every spatial tile.
struct DevGeom {
  int rows, cols, tiles_w, tiles_h, n_tiles, d;
  int nqf, nq_trows, bnq;
  int q_tr_first[kMaxFrames];  // first q-frame index of q t_row
  int q_tr_count[kMaxFrames];  // 1 or 2 frames
  int q_tr_diag[kMaxFrames];   // index of the k t_row with the same temporal key, or -1
  int q_frame_tr[kMaxFrames];  // q t_row of q frame i
  int q_frame_tok0[kMaxFrames];// flat token offset of q frame i (i * rows * cols)
  int nkf, nk_trows, bnk;
  int k_tr_first[kMaxFrames];
  int k_tr_count[kMaxFrames];
  int k_slot[kMaxFrames];      // storage slot (ring slot or flat frame index) of k frame i
  int k_frame_tok0[kMaxFrames];// flat token offset of k frame i in grid_k order
};

__host__ __device__ inline int tile_h_count(const DevGeom& g, int tile) {
  const int th = tile / g.tiles_w;
  const int r = g.rows - 8 * th;
  return r < 8 ? r : 8;
}
__host__ __device__ inline int tile_w_count(const DevGeom& g, int tile) {
  const int tw = tile % g.tiles_w;
  const int c = g.cols - 8 * tw;
  return c < 8 ? c : 8;
}

// Locality window [lo, hi) of key coordinates for query coordinate p along an axis of
// length F with extent e (P/src/mask.cpp:128-141).
__host__ __device__ inline void locality_range(int mode, int p, int e, int F, int& lo, int& hi) {
  const int r = e / 2;
  if (mode == 1) {  // boundary_truncated
    lo = p - r;
    hi = p + r + 1;
  } else {          // boundary_preserved
    int a = p - r;
    const int amax = F - e;
    a = a < 0 ? 0 : (a > amax ? amax : a);
    lo = a;
    hi = a + e;
  }
}

// Byte offset of (row, chan) inside a packed frame-tile.
__host__ __device__ inline uint32_t tile_byte_offset(int r, int c) {
  return (uint32_t)((c >> 6) * kSubBytes + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) + ((c & 7) << 1));
}

// ---------------------------------------------------------------------------------------
// PTX wrappers (sm_100a)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Wait for the phase with the given parity to complete.  The suspend-time hint lets the
// hardware park the waiting thread until the phase flips instead of spinning (a spinning
// waiter steals issue slots from the warps doing the work).  A watchdog turns a protocol
// deadlock into a trap instead of a hung device.
// Wait for a phase that is far away (e.g. a whole unit): poll with test_wait and sleep in
// between instead of the try_wait suspend, which wakes on every barrier event of the CTA and
// would steal issue slots from the warps on the critical path.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  const uint32_t addr = smem_u32(bar);
  for (int it = 0;; ++it) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    if (it > (1 << 22)) __trap();
    __nanosleep(ns);
  }
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  for (int it = 0;; ++it) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity), "r"(0x989680u)
        : "memory");
    if (done) return;
    if (it > (1 << 22)) __trap();
  }
}
// 1D bulk copy global -> shared, completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// shared -> global bulk copy (async proxy), tracked by the issuing thread's bulk groups
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
// Tiled tensor copy global -> shared through a tensor map (TMA), 5-D box at the given
// coordinates (innermost first); completion counted on `bar` in bytes (out-of-bounds box
// elements are written as zeros and counted).
__device__ __forceinline__ void tma_load_5d(void* dst, const void* map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
// global -> L2 bulk prefetch (no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// One lane of the (fully active) warp returns true.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_shared(const uint32_t* ptr) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(ptr)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_shared(uint32_t* ptr, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(ptr)), "r"(v) : "memory");
}
// Programmatic dependent launch: a kernel launched with programmatic stream serialization
// may start while its predecessor drains; it must wait (griddepcontrol.wait) before touching
// anything the predecessor writes or reads.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Per-warpgroup register budget (all 4 warps of the warpgroup execute it).
template <int N>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

// ---- tcgen05 ----------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 inputs, fp32 accumulate).
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#define FVSR_R8(i) "=r"(r[i]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3]), "=r"(r[i + 4]), "=r"(r[i + 5]), "=r"(r[i + 6]), "=r"(r[i + 7])
// 32 lanes x 32 bit, 32 consecutive columns: thread t of warp w gets lane 32*(w%4)+t.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : FVSR_R8(0), FVSR_R8(8), FVSR_R8(16), FVSR_R8(24)
      : "r"(taddr));
}
#undef FVSR_R8
#define FVSR_W8(i) "r"(r[i]), "r"(r[i + 1]), "r"(r[i + 2]), "r"(r[i + 3]), "r"(r[i + 4]), "r"(r[i + 5]), "r"(r[i + 6]), "r"(r[i + 7])
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      FVSR_W8(0), FVSR_W8(8), FVSR_W8(16), FVSR_W8(24)
      : "memory");
}
#undef FVSR_W8

// UMMA shared-memory descriptor, SWIZZLE_128B, version 1 (Blackwell).
//   K-major:  LBO unused (1), SBO = 1024 B between 8-row groups.
//   MN-major: LBO = byte stride between 64-element MN groups, SBO = 1024 B between
//             8-deep K groups.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1
  d |= (uint64_t)2 << 61;  // layout = SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16 with bf16 A/B and fp32 D.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                          // D format F32
         | (1u << 7)                        // A format BF16
         | (1u << 10)                       // B format BF16
         | ((uint32_t)a_mn_major << 15)     // A major
         | ((uint32_t)b_mn_major << 16)     // B major
         | ((uint32_t)(N >> 3) << 17)       // N / 8
         | ((uint32_t)(M >> 4) << 24);      // M / 16
}

}  // namespace fvsr

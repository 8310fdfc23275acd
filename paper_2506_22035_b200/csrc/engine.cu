// sm_100a SPIDER stencil engine: strided-swapped 2:4 kernel rows on the
// Blackwell sparse tensor cores (tcgen05.mma.sp), plus the support kernels
// behind the C ABI (include/spider.h).
//
// One launch = one Jacobi step (pipeline.py:247-261 / core.py:176-181) over a
// tile range (or, SPD_RUN_PERSISTENT, all steps in L2-wavefront order).
// Persistent, warp-specialised CTA (one per SM, 16 warps):
//   warps 0-3  epilogue : TMEM -> registers -> fp16 -> xor-butterfly transpose
//                         inside each L-lane group -> 256-bit stores, each
//                         instruction writing whole 128-byte lines
//   warps 4-11 producer : LDS.128 of the TMA-staged natural input rows -> warp
//                         shuffles -> PRMT byte permutes that apply the
//                         reference's input-row involution (transform.py:
//                         130-139) and the 2L-window expansion (pipeline.py:
//                         176-186, 251-252) -> STS.128 straight into the UMMA
//                         K-major B image.  The swap costs no extra pass: it is
//                         folded into the register->smem write.
//   warp 12    MMA      : the converged warp runs a compile-time MMA schedule,
//                         one elected lane issues tcgen05.mma.sp with the
//                         compressed kernel (A) and metadata (E) resident in
//                         TMEM for the whole launch.
//   warp 13    loader   : cp.async.bulk.tensor boxes of the halo-padded block.
//   warps 14-15         : publisher / dependency poller (persistent launches).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <vector>

#include "spider_internal.h"

namespace spd {

// ---------------------------------------------------------------------------
// PTX helpers

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
  return t;
}
// Development builds only (tools/build_variant.sh <name> -DSPD_DEVEL): the
// per-role timeline (SPD_TRACE, event e of tile-iteration it in CTAs 0-7) and
// the role-elimination switches (SPD_DBG bits 1: no output stores, 4: no
// producer work, 8: no MMAs, 16: no epilogue transpose).  The production library compiles
// both to nothing: no runtime debug branch sits in a hot loop, and no switch
// can remove a fence.
#ifdef SPD_DEVEL
#ifndef SPD_NO_TRACE
#define SPD_TRACE(e, it)                                                                                 \
  do {                                                                                                   \
    if (p.trace && blockIdx.x < 8 && (it) < 64) *(volatile unsigned long long*)&p.trace[(blockIdx.x * 16 + (e)) * 64 + (it)] = gtimer(); \
  } while (0)
#else
#define SPD_TRACE(e, it) \
  do {                   \
  } while (0)
#endif
#ifndef SPD_DBG_MASK
#define SPD_DBG_MASK 0xffffffff  // which switches are live (variant builds isolate one site)
#endif
#define SPD_DBG_BIT(b) ((((unsigned)(SPD_DBG_MASK)) & (b)) != 0 && (p.dbg & (b)) != 0)
#else
#define SPD_TRACE(e, it) \
  do {                   \
  } while (0)
#define SPD_DBG_BIT(b) false
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Suspend-time hint for mbarrier waits (ns; 0 = the hardware default): a
// waiting warp sleeps until the phase completes instead of re-polling.
// profiles/r02_power.txt: 1 ms hint B9 73.1 -> 71.9 us at full clock, energy
// per step unchanged.
#ifndef SPD_WAIT_HINT
#define SPD_WAIT_HINT 1000000
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#if SPD_WAIT_HINT > 0
  asm volatile(
      "{\n.reg .pred P1;\nWAIT%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE%=;\nbra WAIT%=;\nDONE%=:\n}" ::"r"(bar),
      "r"(parity), "n"(SPD_WAIT_HINT)
      : "memory");
#else
  asm volatile(
      "{\n.reg .pred P1;\nWAIT%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE%=;\nbra WAIT%=;\nDONE%=:\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
#endif
}

// Non-blocking phase test.
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// Wait for a phase with the warp descheduled between tests: for the roles
// that are off the critical path (publisher, poller), so their waiting does
// not compete for issue slots and the mbarrier unit with the pipeline roles.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  while (!mbar_test(bar, parity)) __nanosleep(128);
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE (verified layout, see
// tools/umma_sp_probe.cu): core matrix = 8 rows x 16 B, LBO = stride between
// K-adjacent core matrices, SBO = stride between 8-row groups.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100)
  return d;
}

// Instruction descriptor for kind::f16 sparse, fp32 accumulate, K-major A/B.
__host__ __device__ constexpr uint32_t idesc_sparse_f16(int m, int n, bool bf16) {
  return (1u << 2)                        // sparse
         | (1u << 4)                      // D = f32
         | ((bf16 ? 1u : 0u) << 7)        // A format
         | ((bf16 ? 1u : 0u) << 10)       // B format
         | ((uint32_t)(n >> 3) << 17)     // N
         | ((uint32_t)(m >> 4) << 24);    // M
}

// D[tmem] (+)= A[tmem] * B[smem desc] with metadata E[tmem]  (ts form)
__device__ __forceinline__ void mma_sp_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t e,
                                          uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(e), "r"(accum), "r"(idesc));
}

// Same, issued by one elected lane of a converged warp.
__device__ __forceinline__ void mma_sp_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t e, uint32_t idesc,
                                                uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|q, 0xffffffff;\n"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(e), "r"(accum), "r"(idesc));
}
__device__ __forceinline__ void tc_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar, uint32_t rank) {
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(bar),
      "r"(rank)
      : "memory");
}
// CTA-pair sparse MMA (issued by the leader CTA only), M = 256
__device__ __forceinline__ void mma_sp_ts_elect_cg2(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t e, uint32_t idesc,
                                                    uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|q, 0xffffffff;\n"
      "@q tcgen05.mma.sp.cta_group::2.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(e), "r"(accum), "r"(idesc));
}
__device__ __forceinline__ void tc_commit_mc_elect(uint32_t bar) {
  asm volatile(
      "{\n.reg .pred q;\n.reg .b16 mask;\nmov.b16 mask, 3;\nelect.sync _|q, 0xffffffff;\n"
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], mask;\n}" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void tmem_st_x1(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v));
}

__device__ __forceinline__ void tmem_ld_x32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

// 16 lanes x 256 bits, four repetitions (32 columns): thread t receives
// {D[l][c], D[l][c+1], D[l+8][c], D[l+8][c+1]} for l = t/4 and columns
// c = 8k + 2(t%4), k = 0..3, in that register order (tools/tmem_layout.cu).
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// 256-bit global store (sm_100): one full 32-B sector group per lane.
__device__ __forceinline__ void stg_v8(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e, uint32_t f,
                                       uint32_t g, uint32_t h) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d), "r"(e),
               "r"(f), "r"(g), "r"(h)
               : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void sts_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

template <typename T>
struct Cvt;
template <>
struct Cvt<__half> {
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};
template <>
struct Cvt<__nv_bfloat16> {
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};

// ---------------------------------------------------------------------------
// Compile-time permutation tables

// input_row_permutation (transform.py:130-139): slot q of the swapped window
// holds window element PI(q).
__host__ __device__ constexpr int perm_slot(int L, int parity, int q) {
  return (q < L) ? (((q % 2) == parity) ? q + L : q) : ((((q - L) % 2) == parity) ? q - L : q);
}

// __byte_perm selector that packs half `ha` of word x (low) and half `hb` of
// word y (high).
__host__ __device__ constexpr uint32_t sel_halves(int ha, int hb) {
  return (uint32_t)((2 * ha) | ((2 * ha + 1) << 4) | ((4 + 2 * hb) << 8) | ((5 + 2 * hb) << 12));
}

// ---------------------------------------------------------------------------
// Kernel parameters

struct StepParams {
  CUtensorMap tmap[2];       // buf[0] / buf[1] as 2D / 3D tensors (tensor-TMA mode)
  Geometry g;
  int use_tmap;              // 1: tensor-TMA boxes, 0: 1D bulk copies per row
  int rowmajor;              // 2D generic radii: ONE 3D-view TMA box per tile lands the block as
                             // contiguous rows [row][nbox*boxw] (no box boundaries inside a row)
  int nbox, boxw, box_slot;  // natural-stage layout: [box][row][boxw] elements
  int nat_bytes;             // bytes per natural stage
  int xoff, yoff, zoff;      // stored coordinates of interior (0, 0, 0)
  void* buf[2];              // step t reads buf[t & 1] and writes buf[(t + 1) & 1]
  int steps;                 // Jacobi steps in this launch (persistent, >= 1)
  unsigned int* band_done;   // [n_bands] completed tiles per band (steps > 1)
  int per_band, n_bands;     // tiles per band; bands (2D: tile rows, 3D: tile planes, 1D: tiles)
  // persistent (steps > 1) work order: sweeps of `sweep` steps; inside a
  // sweep, wavefront w holds (local step s, band w - lag*s) for s ascending,
  // so step s+1 trails step s by `lag` bands and reads what step s wrote a
  // few wavefronts earlier, still resident in L2 (temporal blocking through
  // the 126 MB L2).
  int sweep, lag, total;     // total = pairs * per_band work items
  int stepmajor;             // persistent (steps > 1) in plain step-major order: work item gi is tile
                             // gi % n_tiles of step gi / n_tiles (no order array); every step
                             // traverses its tiles forward
  int use_order;             // steps == 1 with a host-given band order
  int edge_order;            // steps == 1: 1 / 2 = both edge bands first, then the interior forward /
                             // backward (the slab step; computed per tile, no order array)
  int publish;               // steps == 1: publish finished tiles to band_done (system scope) for a
                             // copy engine waiting on them (peer exchange inside one launch)
  int chain;                 // chained one-step launches of a run (SPD_RUN_CHAINED): every tile is
                             // published to band_done (gpu scope); launches after the run's first
                             // one (chain_t >= 1) skip griddepcontrol.wait and instead wait per tile
                             // for the three neighbouring bands of step chain_t - 1, so a step's
                             // first tiles overlap the previous step's last ones
  int chain_t;               // step index of this launch within the chained run
  const int2* order;         // [pairs] (step, band) in execution order (host-built)
  int64_t pitch, plane, origin;
  int64_t nx;                // x extent (interior)
  int64_t row_lo, row_hi;    // valid output rows (2D: y, 3D: z, 1D: unused)
  int64_t ny;                // 3D: y extent (rows beyond it are masked)
  int tiles_x, tiles_y, tiles_z;
  int tile_y0, tile_z0;      // first tile row / plane of the range
  int band_stride;           // tile rows (2D) / planes (3D) between consecutive bands of the range (1, or
                             // last-first for the two-edge launch of a slab's boundary bands)
  int n_tiles;
  int reverse;               // step 0 traverses tiles last-to-first; steps alternate
  int dbg;                   // development switches (SPD_DBG; read only in -DSPD_DEVEL builds)
  int item_fence;            // always 0: a uniform branch per 2D r = 1 producer item (see the producer)
  // Slab step with fused peer stores: output rows (2D) / planes (3D) u < peer_rows are also
  // stored into peer_out[0] at row u + peer_row[0] (the up neighbour's bottom halo), rows
  // u >= row_hi - peer_rows into peer_out[1] at u + peer_row[1] (the down neighbour's top halo)
  void* peer_out[2];
  int64_t peer_row[2];
  int peer_rows;
  unsigned long long* trace; // debug timeline (CTA 0): [event][tile] globaltimer stamps, or null
  const uint16_t* a_img;     // [S][128][16] compressed values (fp16/bf16 bits)
  const uint32_t* e_words;   // [S][128]
};

// Epilogue: kEpiGroups groups of 4 warps (one warp per TMEM lane quadrant);
// group g drains the accumulators of the tiles it == g (mod kEpiGroups), so
// the TMEM -> register -> global path of consecutive tiles overlaps.
#ifndef SPD_3D_NSTAGE
#define SPD_3D_NSTAGE 2
#endif
#ifndef SPD_3D_NNAT
#define SPD_3D_NNAT 4  // 3D natural-row stages (tools/build_variant.sh scans)
#endif
#ifndef SPD_3D_NACC
#define SPD_3D_NACC 4
#endif
// 2D r = 1: one B-image stage and four natural-row (TMA) stages.  The step
// is bound by the memory system (tools/tma_bw.cu: the same TMA loads + 256-bit
// stores with no compute take 82 us with two load stages, 68-70 us with four);
// two B stages + two load stages measured B9 80.7 / W 210.0 us, one + four
// 79.4 / 194.2 us (profiles/r02_stages.txt).
#ifndef SPD_2D_NSTAGE
#define SPD_2D_NSTAGE 1
#endif
#ifndef SPD_2D_NNAT
#define SPD_2D_NNAT 4
#endif
#ifndef SPD_2D_NACC
#define SPD_2D_NACC 3
#endif
#ifndef SPD_EPI_GROUPS
#define SPD_EPI_GROUPS 1
#endif
#ifndef SPD_PROD_WARPS
#define SPD_PROD_WARPS 8
#endif
// Producer warps per geometry (tools/time_cfg.py over builds, profiles/r02_prodwarps.txt):
// 2D r = 1 keeps 8; the 3D two-M-tile geometry runs fastest with 4 (B27
// 140.0 -> 122.3 us; 2: 422, 3: 176, 5: 138), 2D r = 3 with 5 (B49 101.9 ->
// 97.2 us; 4: 115, 6: 99.0, 7: 100.6).
#ifndef SPD_3D_PW
#define SPD_3D_PW 4
#endif
#ifndef SPD_L8_PW
#define SPD_L8_PW 5
#endif
// Producer work items per basic block (0: all of a tile's items in one
// block; see the producer).  profiles/r02_prodsched.txt: 2D r = 1 1 -> 2
// items B9 74.0 -> 73.2 us, 3D 7 items B27 123.6 -> 121.7 us (2: 148), r = 3
// best as one block (2 / 3 / 5 items: 110 / 107 / 101 vs 97.5 us).
#ifndef SPD_2D_ITEMGROUP
#define SPD_2D_ITEMGROUP 2
#endif
#ifndef SPD_3D_ITEMGROUP
#define SPD_3D_ITEMGROUP 7
#endif
#ifndef SPD_L8_ITEMGROUP
#define SPD_L8_ITEMGROUP 0
#endif
#ifndef SPD_L8_NSTAGE
#define SPD_L8_NSTAGE 3
#endif
#ifndef SPD_L8_NNAT
#define SPD_L8_NNAT 4
#endif
#ifndef SPD_L8_NACC
#define SPD_L8_NACC 4
#endif
#ifndef SPD_GEN_PW
#define SPD_GEN_PW 8
#endif
constexpr int kEpiGroups = SPD_EPI_GROUPS;
constexpr int kEpiWarps = 4;                          // warps per epilogue group
constexpr int kEpiAll = kEpiWarps * kEpiGroups;       // warps 0 .. kEpiAll-1
// Producer warps: a per-geometry template parameter (PW below; this is its
// default).  Warp roles of a CTA with PW producers: epilogue 0..kEpiAll-1,
// producers kEpiAll..kEpiAll+PW-1, then MMA, loader, publisher, poller.
// Persistent launches only (idle in one-step launches): the publisher makes
// finished tiles visible and bumps band counters; the poller runs up to kDQ
// tiles ahead of the loader, waiting for each tile's dependencies (so the
// loader never holds an L2 round trip + gpu-scope fence on its path).
constexpr int kProdWarpsDefault = SPD_PROD_WARPS;
template <int PW>
struct Roles {
  static constexpr int kProdWarps = PW;
  static constexpr int kMmaWarp = kEpiAll + PW;
  static constexpr int kLoadWarp = kMmaWarp + 1;
  static constexpr int kPubWarp = kLoadWarp + 1;
  static constexpr int kPollWarp = kPubWarp + 1;
  static constexpr int kThreads = 32 * (kPollWarp + 1);
};
constexpr int kDQ = 8;                   // poller -> loader ring depth
constexpr int kNPub = 8;                 // publish ring depth (max tiles per publish batch)

template <int L, int NTILE, int NSTAGE, int NNAT, int NACC, int RIN, int MT = 1, int MTR = 0, bool CG2 = false,
          int PW = kProdWarpsDefault>
struct Cfg : Roles<PW> {
  // fast paths: L = 4 (r = 1) and L = 8 (r = 3); any other even L up to 16 uses
  // the generic producer / epilogue
  static constexpr bool GEN = !(L == 4 || L == 8);
  static constexpr int KC = (2 * L + 7) / 8 <= 1 ? 1 : ((2 * L + 7) / 8 <= 2 ? 2 : 4);
  static constexpr int CPL = GEN ? 1 : 8 / L;  // chunks per lane
  static constexpr int SEG = 32 * CPL;       // chunks per warp segment (256 points)
  // HALF: tile rows of 32 chunks (128 points, the 3D two-M-tile geometry):
  // a warp item is a row pair, one row per half-warp
  static constexpr bool HALF = !GEN && CPL == 2 && NTILE == 32;
  static constexpr int SEGS = HALF ? 1 : NTILE / SEG;   // segments per tile row
  // natural row segment staged by the bulk copy: [x0 - 8, x0 + NTILE*L + 8)
  static constexpr int ROW_ELEMS = NTILE * L + 16;
  static constexpr int ROW_BYTES = ROW_ELEMS * 2;
  // tensor-TMA split of the natural row into NBOX boxes of BOXW (<= 256) elements
  static constexpr int NBOX = (ROW_ELEMS + 255) / 256;
  static constexpr int BOXW = ((ROW_ELEMS + NBOX - 1) / NBOX + 7) / 8 * 8;
  // generic epilogue staging: rows of 32*L points (64L bytes) with a 16-byte
  // pad: rows stay 16-B aligned for the vector copy-out and successive rows
  // start 4 banks apart
  static constexpr int R_OUT = 128 / L;
  static constexpr int STG_PITCH = 64 * L + 16;
  static constexpr int STG_BYTES = GEN ? 2 * R_OUT * STG_PITCH + 16 * R_OUT + 16 : 0;
  static constexpr int ACC_COL = 0;
  // MT M-tiles per tile (each M = 128): accumulator stage = MT x NTILE columns
  // (CTA pair: each CTA's accumulator holds the pair's 2 x NTILE columns)
  static constexpr int ACC_STAGE = MT * NTILE * (CG2 ? 2 : 1);
  static constexpr int E_COL = NACC * ACC_STAGE;
  // E for MMA s at E_COL + 2s: bit 0 of the metadata TMEM address is the
  // sparse_id2 selector, so each MMA's column must be even (odd -> misaligned).
  static constexpr int S_MMA = (RIN - (MT - 1) * MTR + 4 / KC - 1) / (4 / KC);  // MMAs per M-tile
  static constexpr int A_COL = E_COL + (2 * S_MMA + 7) / 8 * 8;
  static constexpr int TMEM_COLS = 512;  // host checks A_COL + 8*S <= 512
  static_assert(HALF || NTILE % SEG == 0, "tile width must be whole warp segments");
  // producer work items (input row x warp segment, or row pair) per tile
  static constexpr int N_ITEMS = HALF ? RIN / 2 : RIN * SEGS;
  static_assert(!HALF || RIN % 2 == 0, "row pairs");
  // MMA schedule: the first M-tile's input rows; M-tile t uses them shifted
  // by t*MTR rows (same A/E images)
  static constexpr int RIN_MMA = RIN - (MT - 1) * MTR;
  static constexpr int NQ = (N_ITEMS + PW - 1) / PW;
};

// Compile-time twin of aot.cpp assign_mma_halves / lane_of for an
// instantiation: which half of the accumulator lanes MMA s feeds (0: all,
// M = 128; 1 / 2: lanes 0-15 / 16-31 of every quadrant, M = 64).  The choice
// is folded into the issuer's unrolled schedule: reading it per MMA from the
// kernel parameters put constant-bank loads into B27's issue chain (30 N = 32
// MMAs per tile) and cost 11 % per launch (profiles/r02_m64_ct.txt).  The
// launcher checks the table against the plan's.  Tile shapes: MT = 2 -> 3D 8z x 8y
// (a = 8z + y per M-tile, input row b = 10 iz + iy); RIN = R_OUT -> 1D
// segments; else 2D rows (input row b feeds output rows b - 2r .. b).
template <class C, int L, int RIN, int MT>
__host__ __device__ constexpr int ct_lane_of(int a, int i) {
  if (MT == 2) {
    const int z = a / 8, y = a % 8;
    return 32 * (y / 2) + 16 * (z / 2) + 4 * (2 * (z % 2) + (y % 2)) + i;
  }
  if (L == 4) {
    const int j = a / 4;
    return 32 * (j % 4) + 16 * (j / 4) + 2 * (a % 4) + (i >> 1) + 8 * (i & 1);
  }
  if (L == 8) return 32 * ((a % 8) / 2) + 16 * (a / 8) + 8 * (a % 2) + i;
  return L * a + i;
}
template <class C, int L, int RIN, int MT>
__host__ __device__ constexpr bool ct_feeds(int b, int a) {
  if (MT == 2) {
    const int dz = b / 10 - 1 - a / 8, dy = b % 10 - 1 - a % 8;
    return dz >= -1 && dz <= 1 && dy >= -1 && dy <= 1;
  }
  if (RIN == C::R_OUT) return a == b;  // 1D
  return b - a >= 0 && b - a <= L - 2;  // 2D: kernel rows rho = b - a - r, r = (L - 2) / 2
}
template <class C, int L, int RIN, int MT>
__host__ __device__ constexpr int ct_mma_half(int s) {
#ifdef SPD_NO_M64
  return 0 * s;
#else
  constexpr int RPM = 4 / C::KC;
  constexpr int RM = C::RIN_MMA;
  if (s == 0) return 0;
  const int start = s * RPM + RPM <= RM ? s * RPM : RM - RPM;
  bool used0 = false, used1 = false;
  for (int b = s * RPM; b < start + RPM; ++b)
    for (int a = 0; a < C::R_OUT; ++a)
      if (ct_feeds<C, L, RIN, MT>(b, a))
        for (int i = 0; i < L; ++i) {
          if (ct_lane_of<C, L, RIN, MT>(a, i) % 32 >= 16) used1 = true;
          else used0 = true;
        }
  return used0 && used1 ? 0 : (used0 ? 1 : (used1 ? 2 : 0));
#endif
}
// all MMAs of the schedule, 2 bits each (evaluated at compile time)
template <class C, int L, int RIN, int MT>
__host__ __device__ constexpr uint64_t ct_halves_mask() {
  constexpr int RPM = 4 / C::KC;
  constexpr int S = (C::RIN_MMA + RPM - 1) / RPM;
  uint64_t m = 0;
  for (int s = 0; s < S && s < 32; ++s) m |= (uint64_t)ct_mma_half<C, L, RIN, MT>(s) << (2 * s);
  return m;
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// 1D bulk copy global -> shared on the TMA engine, completing on an mbarrier.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// Tensor TMA box loads (tile mode, no swizzle), completing on an mbarrier.
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// Tensor box prefetch into L2 (no smem, no completion): lets the loader run
// further ahead than the natural-row ring allows.
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

__device__ __forceinline__ unsigned int ld_relaxed_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
// Predicated 32-bit shared load: v keeps its value where pred is false (no
// divergent branch around it).
__device__ __forceinline__ void lds_u32_if(uint32_t& v, bool pred, uint32_t addr) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %1, 0;\n@p ld.shared.u32 %0, [%2];\n}" : "+r"(v) : "r"((uint32_t)pred), "r"(addr));
}

// Predicated 128-bit shared load (v keeps its value where pred is false).
__device__ __forceinline__ void lds_v4_if(uint4& v, bool pred, uint32_t addr) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n@p ld.shared.v4.u32 {%0,%1,%2,%3}, [%5];\n}"
               : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
               : "r"((uint32_t)pred), "r"(addr));
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Slab step, fused peer stores (called by the publisher warp, all lanes): the
// tile at (z0, y0, x0)'s rows (2D) / planes (3D) u < peer_rows go to the up
// neighbour's halo (row u + peer_row[0]), u >= row_hi - peer_rows to the down
// neighbour's (u + peer_row[1]).  Only interior x is copied: the neighbours'
// x-halo columns are Dirichlet constants.  16-byte vectors (x = 0 is 32-byte
// aligned), scalar tail.  Inlined or called out of line per geometry: the
// choice moves the whole kernel's code layout, and the two geometries that
// react prefer opposite ones (B27 inlined 123 vs 130 us, B49 out of line 100
// vs 103; profiles/r02_slab_step.txt).
template <typename T>
__device__ __forceinline__ void peer_copy_tile(const StepParams& p, const T* src_base, int64_t z0, int64_t y0,
                                               int64_t x0, int lane) {
  const Geometry& g = p.g;
  const int64_t unit = g.d == 3 ? p.plane : p.pitch;
  const int64_t xw = min((int64_t)g.tile_x, p.nx - x0);
  const int64_t nvec = xw / 8;
  const int rows_y = g.d == 3 ? (int)min((int64_t)g.tile_y, p.ny - y0) : 1;
  const int64_t u0 = g.d == 3 ? z0 : y0;
  const int nu = g.d == 3 ? g.tile_z : g.tile_y;
  for (int k = 0; k < 2; ++k) {
    if (!p.peer_out[k]) continue;
    T* dst_base = static_cast<T*>(p.peer_out[k]);
    for (int du = 0; du < nu; ++du) {
      const int64_t u = u0 + du;
      if (u >= p.row_hi) break;
      if (k == 0 ? u >= p.peer_rows : u < p.row_hi - p.peer_rows) continue;
      for (int ry = 0; ry < rows_y; ++ry) {
        const int64_t off = p.origin + (g.d == 3 ? u * p.plane + (y0 + ry) * p.pitch : u * p.pitch) + x0;
        const T* src = src_base + off;
        T* dst = dst_base + off + p.peer_row[k] * unit;
        for (int64_t v = lane; v < nvec; v += 32)
          reinterpret_cast<uint4*>(dst)[v] = __ldcg(reinterpret_cast<const uint4*>(src) + v);
        for (int64_t e = nvec * 8 + lane; e < xw; e += 32)
          reinterpret_cast<uint16_t*>(dst)[e] = __ldcg(reinterpret_cast<const unsigned short*>(src) + e);
      }
    }
  }
}

template <typename T>
__device__ __noinline__ void peer_copy_tile_call(const StepParams& p, const T* src_base, int64_t z0, int64_t y0,
                                                 int64_t x0, int lane) {
  peer_copy_tile<T>(p, src_base, z0, y0, x0, lane);
}

// ---------------------------------------------------------------------------
// The stencil step kernel.
//
// Pipelines (all mbarrier based):
//   loader --(nat_full: tx bytes)--> producers --(nat_empty)--> loader
//   producers --(b_full)--> MMA --(b_empty: tcgen05.commit)--> producers
//   MMA --(acc_full: tcgen05.commit)--> epilogue --(acc_empty)--> MMA
template <typename T, int L, int PARITY, int NTILE, int NSTAGE, int NNAT, int NACC, int RIN, int MT = 1, int MTR = 0,
          bool CG2 = false, int PW = kProdWarpsDefault, bool EDGE = false>
__global__ void __launch_bounds__(Roles<PW>::kThreads, 1) spider_step_kernel(const __grid_constant__ StepParams p) {
  using C = Cfg<L, NTILE, NSTAGE, NNAT, NACC, RIN, MT, MTR, CG2, PW>;
  constexpr int kProdWarps = C::kProdWarps;
  constexpr int kMmaWarp = C::kMmaWarp;
  constexpr int kLoadWarp = C::kLoadWarp;
  constexpr int kPubWarp = C::kPubWarp;
  constexpr int kPollWarp = C::kPollWarp;
  constexpr int KC = C::KC;
  constexpr int NQ = C::NQ;
  const Geometry& g = p.g;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int sbo = g.b_sbo;
  const int stage_bytes = (NTILE / 8) * sbo;
  uint8_t* bimg = smem;
  uint8_t* nat = smem + NSTAGE * stage_bytes;
  uint8_t* stg = nat + NNAT * p.nat_bytes;  // generic epilogue staging (C::STG_BYTES)
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + C::STG_BYTES);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * NSTAGE + 2 * NACC + 2 * NNAT + 2 * kNPub + 2 * kDQ);
  const uint32_t bimg_s = smem_u32(bimg);
  const uint32_t nat_s = smem_u32(nat);
  const uint32_t bar_full = smem_u32(bars);
  const uint32_t bar_empty = bar_full + 8 * NSTAGE;
  const uint32_t bar_accf = bar_full + 16 * NSTAGE;
  const uint32_t bar_acce = bar_accf + 8 * NACC;
  const uint32_t bar_natf = bar_acce + 8 * NACC;
  const uint32_t bar_nate = bar_natf + 8 * NNAT;
  const uint32_t bar_pubf = bar_nate + 8 * NNAT;  // epilogue -> publisher: tile stores issued
  const uint32_t bar_pube = bar_pubf + 8 * kNPub;  // publisher -> epilogue: slot free
  const uint32_t bar_depf = bar_pube + 8 * kNPub;   // poller -> loader: tile's inputs are final
  const uint32_t bar_depe = bar_depf + 8 * kDQ;     // loader -> poller: slot free

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  // CTA pair (cluster of 2): both CTAs walk the same tiles; rank 0 issues the MMAs
  const uint32_t crank = CG2 ? cluster_ctarank() : 0u;
  const int wid0 = CG2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int wstride = CG2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  if (threadIdx.x == 0) SPD_TRACE(13, 0);
  // let the next step kernel in the stream start its prologue as soon as
  // SMs free up (it still waits for this grid in griddepcontrol.wait)
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(bar_full + 8 * s, kProdWarps * (CG2 ? 2 : 1));  // pair: both CTAs' producers
      mbar_init(bar_empty + 8 * s, 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(bar_accf + 8 * a, 1);
      mbar_init(bar_acce + 8 * a, kEpiWarps * (CG2 ? 2 : 1));  // pair: both CTAs' epilogues
    }
    for (int a = 0; a < NNAT; ++a) {
      mbar_init(bar_natf + 8 * a, 1);
      mbar_init(bar_nate + 8 * a, kProdWarps);
    }
    for (int a = 0; a < kNPub; ++a) {
      mbar_init(bar_pubf + 8 * a, kEpiWarps);
      mbar_init(bar_pube + 8 * a, 1);
    }
    for (int a = 0; a < kDQ; ++a) {
      mbar_init(bar_depf + 8 * a, 1);
      mbar_init(bar_depe + 8 * a, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    if constexpr (CG2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "n"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "n"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  // Resident operands: E words and compressed A into TMEM (loaded once per
  // launch; the stencil kernel is constant — the B200 analogue of keeping the
  // kernel matrix in registers).
  if (warp < kEpiWarps) {
    const int m = warp * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    for (int s = 0; s < g.s; ++s) {
      const size_t si = (size_t)crank * g.s + s;  // pair: rank t's own images
      tmem_st_x1(lane_base + C::E_COL + 2 * s, __ldg(p.e_words + si * 128 + m));
      const uint4* src = reinterpret_cast<const uint4*>(p.a_img + (si * 128 + m) * 16);
      uint4 a0 = __ldg(src), a1 = __ldg(src + 1);
      uint32_t col = lane_base + C::A_COL + 8 * s;
      tmem_st_x1(col + 0, a0.x);
      tmem_st_x1(col + 1, a0.y);
      tmem_st_x1(col + 2, a0.z);
      tmem_st_x1(col + 3, a0.w);
      tmem_st_x1(col + 4, a1.x);
      tmem_st_x1(col + 5, a1.y);
      tmem_st_x1(col + 6, a1.z);
      tmem_st_x1(col + 7, a1.w);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG2) cluster_sync_all();  // the peer's barriers are initialised before any remote arrive
  tc_fence_after();
  // Programmatic dependent launch: everything above (barrier init, TMEM
  // allocation, resident A/E operands) overlaps the previous step kernel's
  // tail; the grids it reads and writes are touched only after the previous
  // grid has completed and its writes are visible.
  if (p.chain_t == 0 || SPD_DBG_BIT(1024)) asm volatile("griddepcontrol.wait;" ::: "memory");

  if (threadIdx.x == 0) SPD_TRACE(14, 0);
  // Work order.  One step (steps == 1): tile t of the step, traversal
  // direction alternating between launches (each step starts on the tiles the
  // previous one wrote last, still in L2).  Persistent (steps > 1): the
  // host-built (step, band) order (sweeps / wavefronts, see StepParams); a
  // tile of step t > 0 first waits (loader) for the three neighbouring bands
  // of step t-1 — dependencies point `lag - 1` >= 1 wavefronts back, i.e. to
  // smaller work indices, so with all CTAs co-resident (cooperative launch)
  // the smallest unfinished tile can always proceed.  Static round-robin
  // over CTAs.
  const bool ordered = p.steps > 1 || p.use_order;
  const bool publishing = p.steps > 1 || p.publish || p.chain;
  // tiles wait (poller -> loader) for their inputs of the previous step
  const bool dep_wait = p.steps > 1 || p.chain_t > 0;
  const int total = ordered ? p.total : p.n_tiles;
  struct TileId {
    int step, band;
    int dep_step;  // step whose bands this tile's inputs come from + 1 (0: no wait)
    int64_t z0, y0, x0;
  };
  // Persistent order entries are fetched one tile ahead (the fetch for the
  // next tile is issued before this tile's work), so the dependent global
  // load never sits on a role's critical path.
  auto fetch = [&](int gi) -> int2 {
    if (!ordered || p.stepmajor || gi >= total) return make_int2(0, 0);
    return __ldg(p.order + gi / p.per_band);
  };
  auto decode_e = [&](int gi, int2 e) {
    TileId id;
    int t;
    if (EDGE) {
      // slab-step instantiation (edge_order set): plain decode, then the band
      // index mapped to the edge-first order -- no extra division
      id.step = 0;
      id.dep_step = 0;
      t = gi;
    } else if (!ordered) {
      id.step = 0;
      id.dep_step = p.chain_t;
      if (p.edge_order) {
        // slab step: both edge bands first, then the interior forward
        // (edge_order 1: 0, nb-1, 1 .. nb-2) or backward (2: nb-1, 0, nb-2 .. 1);
        // arithmetic, so no role waits on a per-tile order lookup
        const int slot = gi / p.per_band;
        const int nb = p.n_bands;
        const int band = p.edge_order == 1 ? (slot == 0 ? 0 : (slot == 1 ? nb - 1 : slot - 1))
                                           : (slot == 0 ? nb - 1 : (slot == 1 ? 0 : nb - slot));
        t = band * p.per_band + (gi - slot * p.per_band);
      } else {
        t = p.reverse ? p.n_tiles - 1 - gi : gi;
      }
    } else if (p.stepmajor) {
      id.step = gi / p.n_tiles;
      id.dep_step = id.step;
      t = gi - id.step * p.n_tiles;
    } else {
      id.step = e.x;
      id.dep_step = e.x;
      t = e.y * p.per_band + gi % p.per_band;
    }
    const int bx = t % p.tiles_x;
    const int rest = t / p.tiles_x;
    int by = rest % p.tiles_y;
    int bz = rest / p.tiles_y;
    if constexpr (EDGE) {  // band at launch position `slot` (see the edge_order branch above)
      int& slot = g.d == 3 ? bz : by;
      const int nb = p.n_bands;
      slot = p.edge_order == 1 ? (slot == 0 ? 0 : (slot == 1 ? nb - 1 : slot - 1))
                               : (slot == 0 ? nb - 1 : (slot == 1 ? 0 : nb - slot));
    }
    id.x0 = (int64_t)bx * g.tile_x;
    id.y0 = (int64_t)(p.tile_y0 + (g.d == 2 ? by * p.band_stride : by)) * g.tile_y;
    id.z0 = (int64_t)(p.tile_z0 + bz * p.band_stride) * g.tile_z;
    id.band = g.d == 3 ? bz : (g.d == 2 ? by : bx);
    return id;
  };


  // Publisher (persistent launches): after all epilogue warps issued a
  // tile's stores (pubf), make them visible at gpu scope and bump the tile's
  // band counter.  Tiles whose stores are already issued are batched behind
  // ONE fence.acq_rel.gpu (cumulative over the epilogue's stores through the
  // CTA-scope mbarrier release/acquire) followed by relaxed increments: the
  // fence waits for the store drain, so one fence per tile cannot keep up
  // with short tiles.
  // single-step publishing (slab step): only the two edge bands' tiles
  auto pub_tile = [&](const TileId& id) {
    return p.steps > 1 || p.chain || id.band == 0 || id.band == p.n_bands - 1;
  };
  // Slab step, fused peer stores: once an edge tile's outputs are stored, the
  // publisher warp copies its edge rows into the neighbours' halos
  // (peer_copy_tile) -- peer-memory stores from inside the step kernel, tile
  // by tile, while the interior is still computing.
  auto peer_copy = [&](const TileId& id) {
    const T* src = static_cast<const T*>(p.buf[(id.step + 1) & 1]);
    if constexpr (L == 8) peer_copy_tile_call<T>(p, src, id.z0, id.y0, id.x0, lane);
    else peer_copy_tile<T>(p, src, id.z0, id.y0, id.x0, lane);
  };
  auto publisher = [&]() {
    if (p.steps == 1 && !p.chain) {  // the whole warp runs this form
      int pit = 0;
      for (int gi = wid0; gi < total; gi += wstride) {
        const TileId id = decode_e(gi, fetch(gi));
        if (!pub_tile(id)) continue;
        mbar_wait_sleep(bar_pubf + 8 * (pit % kNPub), (pit / kNPub) & 1);  // every lane acquires
        if (p.peer_rows) peer_copy(id);
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.acq_rel.sys;" ::: "memory");  // observed by the neighbour / a copy engine
          if (p.band_done)
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.band_done + id.band) : "memory");
          mbar_arrive(bar_pube + 8 * (pit % kNPub));
        }
        __syncwarp();
        ++pit;
      }
      return;
    }
    int it = 0;
    for (int gi = wid0; gi < total;) {
      mbar_wait_sleep(bar_pubf + 8 * (it % kNPub), (it / kNPub) & 1);
      int n = 1;
      while (n < kNPub && gi + n * wstride < total &&
             mbar_test(bar_pubf + 8 * ((it + n) % kNPub), ((it + n) / kNPub) & 1))
        ++n;
      if (!SPD_DBG_BIT(64)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      for (int j = 0; j < n; ++j, ++it, gi += wstride) {
        const TileId id = decode_e(gi, fetch(gi));
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.band_done + id.band) : "memory");
        mbar_arrive(bar_pube + 8 * (it % kNPub));
      }
    }
  };

  if (warp == kLoadWarp) {
    // ===================== loader: TMA copies of the natural input rows ===
    // 2D/3D: the tile's halo-padded input block as nbox tensor boxes
    // (cp.async.bulk.tensor); 1D: one bulk copy per line segment.
    if (lane == 0) {
      const uint32_t box_bytes = (uint32_t)(p.boxw * 2 * g.r_in);
      int it = 0;
      int2 e_nx = fetch(wid0);
      int e_gi = wid0;
      for (int gi = wid0; gi < total; gi += wstride, ++it) {
        const int ns = it % NNAT;
        const uint32_t nphase = (it / NNAT) & 1;
        const int2 e_cur = e_gi == gi ? e_nx : fetch(gi);
        e_nx = fetch(gi + wstride);
        e_gi = gi + wstride;
        const TileId id = decode_e(gi, e_cur);
        const uint32_t dst = nat_s + ns * p.nat_bytes;
        const uint32_t fb = bar_natf + 8 * ns;
        SPD_TRACE(0, it);
        mbar_wait(bar_nate + 8 * ns, nphase ^ 1);
        if (dep_wait && !SPD_DBG_BIT(4096)) {
          // RAW/WAR across steps: the poller has seen the previous step's
          // neighbouring bands complete (gpu-scope acquire) and released this
          // slot; the CTA-scope acquire here extends that to the TMA reads.
          mbar_wait(bar_depf + 8 * (it % kDQ), (it / kDQ) & 1);
          if (!SPD_DBG_BIT(32)) asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> async-proxy reads
        }
        if (p.use_tmap) {
          // select between the two param-space descriptors (a runtime index
          // into the __grid_constant__ array would copy it to local memory,
          // where the TMA unit cannot read it)
          const CUtensorMap* map = (id.step & 1) ? &p.tmap[1] : &p.tmap[0];
          mbar_arrive_expect_tx(fb, box_bytes * p.nbox);
          const int c0 = (int)(p.xoff + id.x0 - 8) + (int)crank * (NTILE * L);  // pair: x-half of this CTA
          const int c1 = (int)(p.yoff + id.y0 - g.r);
          const int c2 = (int)(p.zoff + id.z0 - g.r);
          if (C::GEN && p.rowmajor) {
            tma_load_3d(dst, map, c0, 0, c1, fb);  // view (x, box, row): rows land contiguous
          } else {
            for (int k = 0; k < p.nbox; ++k) {
              if (g.d == 3) tma_load_3d(dst + k * p.box_slot, map, c0 + k * p.boxw, c1, c2, fb);
              else tma_load_2d(dst + k * p.box_slot, map, c0 + k * p.boxw, c1, fb);
            }
          }
        } else {
          mbar_arrive_expect_tx(fb, (uint32_t)(g.r_in * C::ROW_BYTES));
          const T* in = static_cast<const T*>(p.buf[id.step & 1]);
          const T* tbase = in + p.origin + id.z0 * p.plane + id.y0 * p.pitch + id.x0 - 8;
          for (int b = 0; b < g.r_in; ++b) {
            const T* src = tbase + (int64_t)g.in_dz[b] * p.plane + (int64_t)g.in_dy[b] * p.pitch + g.in_dx[b];
            bulk_g2s(dst + b * C::ROW_BYTES, src, C::ROW_BYTES, fb);
          }
        }
        if (dep_wait && !SPD_DBG_BIT(4096)) mbar_arrive(bar_depe + 8 * (it % kDQ));
        SPD_TRACE(1, it);
      }
    }
  } else if (warp >= kEpiAll && warp < kMmaWarp) {
    // ===================== producer: natural rows -> permuted B image =====
    if constexpr (C::GEN) {
      // Generic radius (L = 2r+2 not in {4, 8}): one chunk per lane; the lane
      // reads its 2L-point window as 32-bit words straight from the natural
      // stage and permutes it with compile-time PRMT selectors; window slots
      // past 2L (K-chunk padding) are zero.
      const int pw = warp - kEpiAll;
      constexpr int R = (L - 2) / 2;
      constexpr int n_items = RIN * C::SEGS;
      static_assert((NQ - 1) * kProdWarps < n_items && NQ * kProdWarps >= n_items, "NQ must cover the items");
      constexpr int OFF = R & 1;                  // window-start parity (n*L is even)
      constexpr int NW = (OFF + 2 * L + 1) / 2;  // natural words covering one window
      int it = 0;
      for (int gi = wid0; gi < total; gi += wstride, ++it) {
        const int stage = it % NSTAGE;
        const uint32_t sphase = (it / NSTAGE) & 1;
        const int ns = it % NNAT;
        const uint32_t nphase = (it / NNAT) & 1;
        const uint32_t nbase = nat_s + ns * p.nat_bytes;
        mbar_wait(bar_natf + 8 * ns, nphase);
        mbar_wait(bar_empty + 8 * stage, sphase ^ 1);
        const uint32_t sbase = bimg_s + stage * stage_bytes;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int item = pw + q * kProdWarps;
          if (q == NQ - 1 && item >= n_items) continue;
          const int b = item / C::SEGS, sg = item % C::SEGS;
          const int n = sg * 32 + lane;
          const int s_al = n * L - R + 8 - OFF;
          uint32_t w[NW];
          if (p.rowmajor) {
            // contiguous rows [row][NBOX*BOXW]
            const uint32_t rb = nbase + (uint32_t)(b * C::NBOX * C::BOXW + s_al) * 2;
            if constexpr (L == 16) {
              // window start 16n: 32-B aligned, 128-bit loads (2-way instead
              // of 8-way bank conflicts for 32-bit loads at a 32-B lane stride)
#pragma unroll
              for (int k = 0; k + 4 <= NW; k += 4) {
                const uint4 v = lds_v4(rb + 4 * k);
                w[k] = v.x;
                w[k + 1] = v.y;
                w[k + 2] = v.z;
                w[k + 3] = v.w;
              }
#pragma unroll
              for (int k = NW / 4 * 4; k < NW; ++k) w[k] = lds_u32(rb + 4 * k);
            } else {
#pragma unroll
              for (int k = 0; k < NW; ++k) w[k] = lds_u32(rb + 4 * k);
            }
          } else {
#pragma unroll
            for (int k = 0; k < NW; ++k) {
              const int e = s_al + 2 * k;
              // tensor-TMA stage: [box][row][BOXW]; 1D bulk stage: [row][ROW_ELEMS]
              const int kb = p.use_tmap ? e / C::BOXW : 0;
              const int bw = p.use_tmap ? C::BOXW : C::ROW_ELEMS;
              w[k] = lds_u32(nbase + kb * p.box_slot + (b * bw + e - kb * bw) * 2);
            }
          }
          const uint32_t gbase = sbase + (n / 8) * sbo + (n % 8) * 16 + b * KC * 128;
#pragma unroll
          for (int kc = 0; kc < KC; ++kc) {
            uint32_t wd[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int q0 = 8 * kc + 2 * u;
              if (q0 < 2 * L) {
                const int e0 = OFF + perm_slot(L, PARITY, q0), e1 = OFF + perm_slot(L, PARITY, q0 + 1);
                wd[u] = __byte_perm(w[e0 / 2], w[e1 / 2], sel_halves(e0 % 2, e1 % 2));
              } else {
                wd[u] = 0u;
              }
            }
            sts_v4(gbase + kc * 128, wd[0], wd[1], wd[2], wd[3]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(bar_nate + 8 * ns);
          mbar_arrive(bar_full + 8 * stage);
        }
      }
    } else {
    const int pw = warp - kEpiAll;
    constexpr int n_items = C::N_ITEMS;
    static_assert((NQ - 1) * kProdWarps < n_items && NQ * kProdWarps >= n_items, "NQ must cover the items");
    constexpr int R = (L - 2) / 2;
    // lane position in its row segment (HALF: row pairs, one per half-warp)
    constexpr int SW = C::HALF ? 16 : 32;  // lanes per row segment (shuffle width)
    const int lpos = lane % SW;
    // ext[] words actually referenced by the windows (compile time):
    //   element e of ext is x = 8*lane - 8 + e; windows span
    //   e in [8 - R, 8 + (CPL-1)*L - R + 2L - 1]
    constexpr int kPrevW = (8 - R) / 2;                                     // first prev word used
    constexpr int kNextW = (8 + (C::CPL - 1) * L - R + 2 * L - 1) / 2 - 8;  // last next word used
    // Loop-invariant per-item offsets: natural-stage byte offsets of the lane's
    // 16 B and of its neighbouring groups (edges, lanes 0/31 only), and the
    // B-image byte offset of the lane's first chunk.
    //
    // B-image column order (CPL = 2): chunk n sits at column
    //   sigma(n) = (n & ~15) | ((n & 1) << 3) | ((n >> 1) & 7),
    // i.e. even chunks fill one 8-row core-matrix group and odd chunks the
    // next.  Each STS.128 (all lanes storing their even, then their odd chunk)
    // then covers the 32 banks once per quarter-warp — conflict-free without
    // per-lane selects.  The epilogue undoes sigma when it pairs D columns.
    // producer items per basic block (0: the whole tile in one block)
    constexpr int kItemGroup = C::HALF ? SPD_3D_ITEMGROUP : (L == 4 ? SPD_2D_ITEMGROUP : SPD_L8_ITEMGROUP);
    uint32_t noff[NQ], poff[NQ], xoff_n[NQ], soff[NQ];
    static_assert(kPrevW >= 0 && kPrevW < 4 && kNextW < 4, "edge words must fit one 16-byte block");
    bool valid[NQ];
    // natural stage: element x of row b at box k = x / boxw
    auto nat_addr = [&](int b, int x) -> uint32_t {
      const int k = x / p.boxw;
      return (uint32_t)(k * p.box_slot + (b * p.boxw + (x - k * p.boxw)) * 2);
    };
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int item = pw + q * kProdWarps;
      valid[q] = q < NQ - 1 || item < n_items;  // only the last slot can be empty
      const int b = !valid[q] ? 0 : (C::HALF ? 2 * item + lane / 16 : item / C::SEGS);
      const int sg = (valid[q] && !C::HALF) ? item % C::SEGS : 0;
      const int xl = 8 + sg * 256 + lpos * 8;  // this lane's 8 points (stage-local x)
      noff[q] = nat_addr(b, xl);
      poff[q] = nat_addr(b, xl - 8);  // 16-B block left of the lane's (segment-start lane)
      xoff_n[q] = nat_addr(b, xl + 8);  // 16-B block right of it (segment-end lane)
      const int n0 = sg * C::SEG + lpos * C::CPL;
      const int col = C::CPL == 2 ? ((n0 & ~15) | ((n0 >> 1) & 7)) : n0;
      soff[q] = (uint32_t)(b * KC * 128) + (uint32_t)(col / 8) * sbo + (col % 8) * 16;
    }
    int it = 0;
    for (int gi = wid0; gi < total; gi += wstride, ++it) {
      const int stage = it % NSTAGE;
      const uint32_t sphase = (it / NSTAGE) & 1;
      const int ns = it % NNAT;
      const uint32_t nphase = (it / NNAT) & 1;
      const uint32_t nbase = nat_s + ns * p.nat_bytes;
      mbar_wait(bar_natf + 8 * ns, nphase);
      if (pw == 0 && lane == 0) SPD_TRACE(2, it);
      // phase 1: all shared-memory reads of the tile (ILP across items)
      uint4 cur[NQ];
      uint4 edge[NQ];  // segment-edge lanes: the neighbouring 16-B block (one predicated load)
      const bool l0 = lpos == 0, l31 = lpos == SW - 1;
      // Items are cut into basic blocks of kItemGroup items by a uniform
      // branch on p.item_fence (always 0; the compiler cannot fold it; the
      // test must be written inline in each item's `if` -- a bool computed
      // once is merged into one block).  As one block, ptxas hoisted all
      // neighbour shuffles of a 2D r = 1 tile's 9 items ahead of the first
      // B-image store and the step ran 7 % slower (B9 78.4 -> 73.9 us with
      // one item per block, 73.2 with two); the r = 3 producer is fastest as
      // one block (profiles/r02_prodsched.txt).
#define SPD_ITEM_OK(q) \
  (valid[q] && (kItemGroup == 0 || ((q) % (kItemGroup > 0 ? kItemGroup : 1)) != 0 || p.item_fence == 0))
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (SPD_ITEM_OK(q) && !SPD_DBG_BIT(4)) {
          cur[q] = lds_v4(nbase + noff[q]);
          edge[q] = make_uint4(0, 0, 0, 0);
          lds_v4_if(edge[q], l0 || l31, nbase + (l0 ? poff[q] : xoff_n[q]));
        }
      }
      mbar_wait(bar_empty + 8 * stage, sphase ^ 1);
      if (pw == 0 && lane == 0) SPD_TRACE(3, it);
      const uint32_t sbase = bimg_s + stage * stage_bytes;
      // phase 2: neighbour exchange, permutation, B-image stores
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (SPD_ITEM_OK(q) && !SPD_DBG_BIT(4)) {
          uint32_t ext[12];
          const uint32_t cw[4] = {cur[q].x, cur[q].y, cur[q].z, cur[q].w};
#pragma unroll
          for (int w = 0; w < 4; ++w) ext[4 + w] = cw[w];
          const uint32_t ew[4] = {edge[q].x, edge[q].y, edge[q].z, edge[q].w};
#pragma unroll
          for (int w = kPrevW; w < 4; ++w) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, cw[w], 1, SW);
            ext[w] = l0 ? ew[w] : v;
          }
#pragma unroll
          for (int w = 0; w <= kNextW; ++w) {
            const uint32_t v = __shfl_down_sync(0xffffffffu, cw[w], 1, SW);
            ext[8 + w] = l31 ? ew[w] : v;
          }
          const uint32_t a0 = sbase + soff[q];
#pragma unroll
          for (int c = 0; c < C::CPL; ++c) {
            // CPL = 2: the odd chunk lives in the next core-matrix group
            const uint32_t ac = a0 + (c ? (uint32_t)sbo : 0u);
#pragma unroll
            for (int kc = 0; kc < KC; ++kc) {
              uint32_t wd[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int e0 = 8 + c * L - R + perm_slot(L, PARITY, 8 * kc + 2 * u);
                const int e1 = 8 + c * L - R + perm_slot(L, PARITY, 8 * kc + 2 * u + 1);
                wd[u] = __byte_perm(ext[e0 / 2], ext[e1 / 2], sel_halves(e0 % 2, e1 % 2));
              }
              sts_v4(ac + kc * 128, wd[0], wd[1], wd[2], wd[3]);
            }
          }
        }
      }
#undef SPD_ITEM_OK
      if constexpr (CG2) asm volatile("fence.proxy.async;" ::: "memory");  // the pair's MMA reads this B half
      else fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        // (releasing the natural stage right after phase 1 was measured
        // slower: deeper TMA prefetch only raised load latency)
        mbar_arrive(bar_nate + 8 * ns);
        if (CG2 && crank != 0) mbar_arrive_cluster(bar_full + 8 * stage, 0);  // the leader issues the MMAs
        else mbar_arrive(bar_full + 8 * stage);
        if (pw == 0) SPD_TRACE(4, it);
        if (pw == kProdWarps - 1) SPD_TRACE(5, it);
      }
    }
    }
  } else if (warp == kPubWarp) {
    if (publishing && (lane == 0 || (p.steps == 1 && !p.chain)) && !SPD_DBG_BIT(2048)) publisher();
  } else if (warp == kPollWarp) {
    // ===================== dependency poller (persistent launches) =========
    // Tiles whose dependencies are already met are released in batches of
    // up to kDQ/2 behind ONE acquire fence (a gpu-scope fence per tile cannot
    // keep up with 3D tiles).  A tile that must wait first flushes the batch:
    // its dependencies may be tiles of this very batch.
    if (dep_wait && lane == 0 && p.stepmajor && !SPD_DBG_BIT(4096)) {
      // step-major order: a tile's dependencies lie about one step back and
      // are nearly always met, so the poller's cost is its latency.  Tiles
      // go in batches of kBatch: the loads of all their band counters are
      // issued together (one L2 round trip per batch), then one acquire
      // fence, then the batch is released to the loader.
      constexpr int kBatch = kDQ / 2;
      int it = 0;
      for (int gi = wid0; gi < total;) {
        int n = 0;
        int need[kBatch], b0[kBatch], b1[kBatch], bb[kBatch];
        bool any_dep = false;
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
          need[k] = 0;
          b0[k] = b1[k] = bb[k] = 0;
          const int g = gi + k * wstride;
          if (g < total) {
            const TileId id = decode_e(g, fetch(g));
            mbar_wait_sleep(bar_depe + 8 * ((it + k) % kDQ), (((it + k) / kDQ) & 1) ^ 1);
            if (id.dep_step > 0) {
              need[k] = id.dep_step * p.per_band;
              bb[k] = id.band;
              b0[k] = id.band > 0 ? id.band - 1 : 0;
              b1[k] = id.band + 1 < p.n_bands ? id.band + 1 : p.n_bands - 1;
              any_dep = true;
            }
            n = k + 1;
          }
        }
        auto met = [&](int k) {
          if (need[k] == 0 || SPD_DBG_BIT(128)) return true;
          const unsigned int c0 = ld_relaxed_gpu(p.band_done + b0[k]);
          const unsigned int c1 = ld_relaxed_gpu(p.band_done + bb[k]);
          const unsigned int c2 = ld_relaxed_gpu(p.band_done + b1[k]);
          return min(c0, min(c1, c2)) >= (unsigned int)need[k];
        };
        bool batch_ok = true;
        if (any_dep) {
          // one attempt for the whole batch (the loads go out together)
          bool ok[kBatch];
#pragma unroll
          for (int k = 0; k < kBatch; ++k) ok[k] = k >= n || met(k);
#pragma unroll
          for (int k = 0; k < kBatch; ++k) batch_ok = batch_ok && ok[k];
        }
        if (batch_ok) {
          if (any_dep && !SPD_DBG_BIT(512)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
          for (int k = 0; k < n; ++k) mbar_arrive(bar_depf + 8 * ((it + k) % kDQ));
        } else {
          // slow path, tile by tile: a tile's dependencies may be earlier
          // tiles of this very batch (small grids), which must be released
          // before it is waited for
          for (int k = 0; k < n; ++k) {
            while (!met(k)) __nanosleep(64);
            if (need[k] && !SPD_DBG_BIT(512)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
            mbar_arrive(bar_depf + 8 * ((it + k) % kDQ));
          }
        }
        it += n;
        gi += n * wstride;
      }
    } else if (dep_wait && lane == 0 && !SPD_DBG_BIT(4096)) {
      constexpr int kBatch = kDQ / 2;
      int pending = 0;        // gathered, not yet released (tiles it-pending .. it-1)
      bool pend_dep = false;  // some pending tile has dependencies (needs the fence)
      auto flush = [&](int it_end) {
        if (pending == 0) return;
        if (pend_dep && !SPD_DBG_BIT(512)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int t = it_end - pending; t < it_end; ++t) mbar_arrive(bar_depf + 8 * (t % kDQ));
        pending = 0;
        pend_dep = false;
      };
      int it = 0;
      for (int gi = wid0; gi < total; gi += wstride, ++it) {
        const TileId id = decode_e(gi, fetch(gi));
        mbar_wait_sleep(bar_depe + 8 * (it % kDQ), ((it / kDQ) & 1) ^ 1);
        if (id.dep_step > 0) {
          // a tile of step t reads the three neighbouring bands of step t-1
          // (RAW) and overwrites what step t-1 read (WAR): relaxed polls of
          // the three band counters
          const unsigned int need = (unsigned int)(id.dep_step * p.per_band);
          const int b0 = id.band > 0 ? id.band - 1 : 0;
          const int b1 = id.band + 1 < p.n_bands ? id.band + 1 : p.n_bands - 1;
          bool first = true;
          while (!SPD_DBG_BIT(128)) {
            const unsigned int c0 = ld_relaxed_gpu(p.band_done + b0);
            const unsigned int c1 = ld_relaxed_gpu(p.band_done + id.band);
            const unsigned int c2 = ld_relaxed_gpu(p.band_done + b1);
            if (min(c0, min(c1, c2)) >= need) break;
            if (first) flush(it);
            first = false;
            __nanosleep(32);
          }
          pend_dep = true;
        }
        ++pending;
        if (pending == kBatch) flush(it + 1);
      }
      flush(it);
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer ======================================
    // The whole warp runs the loop (converged, warp-uniform operands in
    // uniform registers) and one elected lane issues: a divergent lane-0
    // issue loop costs ~190 cycles per MMA (per-MMA elect loop + R2UR chain)
    // against ~74 for this form at N = 128 (tools/mma_rate.cu).  The MMA
    // count and start rows are compile-time (start_row(s) = min(s*RPM,
    // RIN-RPM), aot.cpp build_geometry).
    const uint32_t idesc = idesc_sparse_f16(CG2 ? 256 : 128, CG2 ? 2 * NTILE : NTILE,
                                            std::is_same<T, __nv_bfloat16>::value);
    const uint32_t idesc64 = idesc_sparse_f16(64, NTILE, std::is_same<T, __nv_bfloat16>::value);
    constexpr uint64_t kHalves = CG2 ? 0 : ct_halves_mask<C, L, RIN, MT>();
    constexpr int RPM = 4 / KC;
    constexpr int RIN_MMA = C::RIN_MMA;
    constexpr int S_CT = (RIN_MMA + RPM - 1) / RPM;
    int it = 0;
    for (int gi = wid0; gi < total && !(CG2 && crank != 0); gi += wstride, ++it) {
      const int stage = it % NSTAGE;
      const uint32_t sphase = (it / NSTAGE) & 1;
      const int acc = it % NACC;
      const uint32_t aphase = (it / NACC) & 1;
      mbar_wait(bar_acce + 8 * acc, aphase ^ 1);
      if (lane == 0) SPD_TRACE(6, it);
      mbar_wait(bar_full + 8 * stage, sphase);
      tc_fence_after();
      if (lane == 0) SPD_TRACE(7, it);
      const uint32_t sbase = bimg_s + stage * stage_bytes;
      const uint32_t dcol = tmem + C::ACC_COL + acc * C::ACC_STAGE;
      const uint64_t bdesc0 = umma_desc(sbase, 128, sbo);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
        for (int s = 0; s < S_CT; ++s) {
          const int start = (s * RPM + RPM <= RIN_MMA ? s * RPM : RIN_MMA - RPM) + mt * MTR;
          // descriptor start address field is addr >> 4
          const uint64_t bdesc = bdesc0 + (uint64_t)((start * KC * 128) >> 4);
          if (SPD_DBG_BIT(8)) continue;  // role elimination (SPD_DEVEL builds only)
          if constexpr (CG2) {
            mma_sp_ts_elect_cg2(dcol, tmem + C::A_COL + 8 * s, bdesc, tmem + C::E_COL + 2 * s, idesc, s > 0 ? 1u : 0u);
          } else {
            // ct_mma_half (= the plan's g.mma_half, aot.cpp assign_mma_halves): 0 -> M = 128;
            // 1 / 2 -> M = 64 on TMEM lanes 32q + [0, 16) / [16, 32), the same lane offset on D, A, E
            const int half = (int)((kHalves >> (2 * s)) & 3);  // folded: the loop is unrolled
            const uint32_t loff = half == 2 ? (16u << 16) : 0u;
            mma_sp_ts_elect(dcol + mt * NTILE + loff, tmem + C::A_COL + 8 * s + loff, bdesc,
                            tmem + C::E_COL + 2 * s + loff, half ? idesc64 : idesc, s > 0 ? 1u : 0u);
          }
        }
      }
      if constexpr (CG2) {  // both CTAs' B stage and accumulator barriers
        tc_commit_mc_elect(bar_empty + 8 * stage);
        tc_commit_mc_elect(bar_accf + 8 * acc);
      } else {
        tc_commit_elect(bar_empty + 8 * stage);
        tc_commit_elect(bar_accf + 8 * acc);
      }
      __syncwarp();
    }
  } else {
    // ===================== epilogue ========================================
    if constexpr (C::GEN) {
     if (warp < kEpiWarps) {  // one epilogue group (the staging tile is shared)
      // Generic radius: TMEM lane m = L*alpha + i.  Lane pairs (i, i+1) pack
      // their fp16 values through a shuffle, store 32-bit words into a staging
      // tile [alpha][32*L points] (pitch 66L bytes: consecutive lanes hit
      // consecutive banks), and the four epilogue warps then copy the tile out
      // with coalesced 32-bit stores.  Two staging buffers, one named barrier
      // per batch.
      constexpr int NB = NTILE / 32;
      const int quad = warp;
      const int m = quad * 32 + lane;
      const int alpha = m / L;
      const int i = m - alpha * L;
      const bool lead = alpha < C::R_OUT && (i % 2) == 0;
      const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
      const uint32_t stg_s = smem_u32(stg);
      // per-row output offsets relative to the tile origin (loop-invariant),
      // kept in the tail of the staging area: {offset, dy}
      int64_t* rowtab = reinterpret_cast<int64_t*>(stg + 2 * C::R_OUT * C::STG_PITCH);
      if (threadIdx.x < C::R_OUT) {
        const int rr = threadIdx.x;
        rowtab[2 * rr] = (int64_t)g.out_dz[rr] * p.plane + (int64_t)g.out_dy[rr] * p.pitch + g.out_dx[rr];
        rowtab[2 * rr + 1] = ((int64_t)g.out_dy[rr] << 32) | (uint32_t)g.out_dx[rr];
      }
      asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps) : "memory");
      int bt = 0;
      int it = 0;
      int pit = 0;  // published tiles (publish ring index)
      int2 e_nx = fetch(wid0);
      int e_gi = wid0;
      for (int gi = wid0; gi < total; gi += wstride, ++it) {
        const int acc = it % NACC;
        const uint32_t aphase = (it / NACC) & 1;
        const int2 e_cur = e_gi == gi ? e_nx : fetch(gi);
        e_nx = fetch(gi + wstride);
        e_gi = gi + wstride;
        const TileId id = decode_e(gi, e_cur);
        T* out = static_cast<T*>(p.buf[(id.step + 1) & 1]);
        mbar_wait(bar_accf + 8 * acc, aphase);
        tc_fence_after();
        const uint32_t tcol = lane_base + C::ACC_COL + acc * C::ACC_STAGE;
        uint32_t va[32], vb[32];
        tmem_ld_x32(tcol, va);
        tmem_wait_ld();
#pragma unroll
        for (int cb = 0; cb < NB; ++cb, ++bt) {
          uint32_t(&v)[32] = (cb & 1) ? vb : va;
          uint32_t(&vn)[32] = (cb & 1) ? va : vb;
          if (cb + 1 < NB) tmem_ld_x32(tcol + (cb + 1) * 32, vn);
          if (cb == NB - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
            if (CG2 && crank != 0) mbar_arrive_cluster(bar_acce + 8 * acc, 0);
            else mbar_arrive(bar_acce + 8 * acc);
          }
          }
          const uint32_t sb = stg_s + (bt & 1) * (C::R_OUT * C::STG_PITCH);
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const uint32_t mine = Cvt<T>::pack(__uint_as_float(v[2 * jj]), __uint_as_float(v[2 * jj + 1]));
            const uint32_t nb = __shfl_down_sync(0xffffffffu, mine, 1);  // lane (alpha, i+1)
            if (lead) {
              const uint32_t row = sb + alpha * C::STG_PITCH;
              sts_u32(row + ((2 * jj) * L + i) * 2, __byte_perm(mine, nb, 0x5410));
              sts_u32(row + ((2 * jj + 1) * L + i) * 2, __byte_perm(mine, nb, 0x7632));
            }
          }
          asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps) : "memory");
          // coalesced copy-out of R_OUT rows x 4L 16-byte vectors
          constexpr int VPR = 4 * L;
          T* tbase = out + p.origin + id.z0 * p.plane + id.y0 * p.pitch + id.x0 + (int64_t)cb * 32 * L;
          const int64_t xlim = p.nx - id.x0 - (int64_t)cb * 32 * L;
          for (int vi = threadIdx.x; vi < C::R_OUT * VPR; vi += 32 * kEpiWarps) {
            const int row = vi / VPR;
            const int col = vi - row * VPR;
            const int64_t roff = rowtab[2 * row];
            const int64_t rdy = rowtab[2 * row + 1];
            const int dy = (int)(rdy >> 32), dx = (int)(uint32_t)rdy;
            const int64_t y = id.y0 + dy;
            bool ok = true;
            if (g.d == 2) ok = y >= p.row_lo && y < p.row_hi;
            const int64_t x = dx + 8 * col;  // first of the vector's 8 points
            if (ok && x < xlim && !SPD_DBG_BIT(1)) {
              const uint4 val = lds_v4(sb + row * C::STG_PITCH + col * 16);
              T* dst = tbase + roff + 8 * col;
              if (x + 8 <= xlim) {
                *reinterpret_cast<uint4*>(dst) = val;
              } else {  // ragged right edge: whole 32-bit pairs only (nx is even)
                const uint32_t wv[4] = {val.x, val.y, val.z, val.w};
                for (int k = 0; k < 4 && x + 2 * k < xlim; ++k) reinterpret_cast<uint32_t*>(dst)[k] = wv[k];
              }
            }
          }
          if (cb + 1 < NB) tmem_wait_ld();
        }
        if (publishing && pub_tile(id) && !SPD_DBG_BIT(2048)) {
          // hand the tile to the publisher warp (release at CTA scope after
          // the warp's stores); the gpu-scope release happens off this path
          const int ps = pit % kNPub;
          mbar_wait(bar_pube + 8 * ps, ((pit / kNPub) & 1) ^ 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_pubf + 8 * ps);
          ++pit;
        }
      }
     }
    } else if constexpr (C::CPL == 2 && MT == 1 && !CG2) {
    // L = 4, quad-pair lane map (aot.cpp lane_of): accumulator lane
    // 32 (s % 4) + 16 (s / 4) + 2 rho + (i >> 1) + 8 (i & 1) holds output row
    // 4 s + rho, chunk position i.  Warp `quad` drains the 16-lane slabs
    // s = quad + 4 h at lane 32 quad + 16 h (h = 0, 1) with
    // tcgen05.ld.16x256b: thread t gets lanes 32 quad + 16 h + t/4
    // (position 2 hi, hi = bit 2 of t) and + 8 (position 2 hi + 1), i.e. one
    // packed word of two consecutive x per chunk, for columns 8k + 2 (t & 3)
    // + {0, 1}.  Under the sigma column order the four columns of a 16-column
    // block give the thread the four consecutive chunks 4 (t & 3) + 0..3 of
    // that block; thread t ^ 4 holds the other two positions of the same
    // chunks.  One xor-4 shuffle per chunk then leaves each thread all four
    // positions of its four chunks in one block of the 32-column batch (block
    // `hi`): 32 contiguous bytes, one 256-bit store, and each warp store
    // instruction covers whole 128-byte lines.  (The 32x32b read of a linear
    // lane map needed a two-level 4-lane butterfly: ~8.5 instructions per
    // output word against ~3 here.)
    const int quad = warp % 4;
    const int grp = warp / 4;
    const int rho = lane >> 3;             // row within the slab
    const bool hi = ((lane >> 2) & 1) != 0;  // positions 2, 3 (else 0, 1); stores block 1 of a batch
    const int cq = lane & 3;               // column pair within each 8-column group
    // output row of this thread in slab h of M-tile mt (M-tile t holds rows a + t*R_OUT)
    int odz[MT][2], ody[MT][2], odx[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = 4 * (quad + 4 * h) + rho + (mt + (int)crank) * C::R_OUT;  // slab quad + 4 h
        odz[mt][h] = g.out_dz[a];
        ody[mt][h] = g.out_dy[a];
        odx[mt][h] = g.out_dx[a];
      }
    int it = 0;
    int pit = 0;  // published tiles (publish ring index)
    int2 e_nx = fetch(wid0);
    int e_gi = wid0;
    for (int gi = wid0; gi < total; gi += wstride, ++it) {
      if (kEpiGroups > 1 && (it % kEpiGroups) != grp) continue;
      const int acc = it % NACC;
      const uint32_t aphase = (it / NACC) & 1;
      const int2 e_cur = e_gi == gi ? e_nx : fetch(gi);
      e_nx = fetch(gi + wstride);
      e_gi = gi + wstride;
      const TileId id = decode_e(gi, e_cur);
      T* out = static_cast<T*>(p.buf[(id.step + 1) & 1]);
      bool row_ok[MT][2];
      int64_t chunk_lim[MT][2];  // valid chunks in this row
      T* orow[MT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t z = id.z0 + odz[mt][h];
          const int64_t y = id.y0 + ody[mt][h];
          const int64_t xr = id.x0 + odx[mt][h];  // x of chunk 0 of this row
          if (g.d == 3) row_ok[mt][h] = z >= p.row_lo && z < p.row_hi && y < p.ny;
          else if (g.d == 2) row_ok[mt][h] = y >= p.row_lo && y < p.row_hi;
          else row_ok[mt][h] = true;
          chunk_lim[mt][h] = (p.nx - xr) / L;
          orow[mt][h] = out + p.origin + z * p.plane + y * p.pitch + xr;
        }
      if (warp == 0 && lane == 0) SPD_TRACE(12, it);
      mbar_wait(bar_accf + 8 * acc, aphase);
      tc_fence_after();
      if (warp == 0 && lane == 0) SPD_TRACE(8, it);
      constexpr int NB = C::ACC_STAGE / MT / 32;  // 32-column batches per M-tile (pair: both x-halves)
      constexpr int TB = MT * NB;                 // batch bi: M-tile bi / NB, column batch bi % NB
      const uint32_t tcol = tmem + ((uint32_t)(quad * 32) << 16) + C::ACC_COL + acc * C::ACC_STAGE;
      auto load = [&](int bi, uint32_t(&v)[2][16]) {
        tmem_ld_16x256b_x4(tcol + 32 * bi, v[0]);
        tmem_ld_16x256b_x4(tcol + (16u << 16) + 32 * bi, v[1]);
      };
      auto emit = [&](int bi, const uint32_t(&v)[2][16]) {
        const int mt = bi / NB, cb = bi % NB;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          // w[b][j]: block b of the batch, chunk 4 cq + j, positions (2 hi, 2 hi + 1)
          uint32_t w[2][4];
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int k = 2 * b + (j & 1), e = j >> 1;
              w[b][j] = Cvt<T>::pack(__uint_as_float(v[h][4 * k + e]), __uint_as_float(v[h][4 * k + 2 + e]));
            }
          uint32_t o[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t r = __shfl_xor_sync(0xffffffffu, hi ? w[0][j] : w[1][j], 4);
            o[2 * j] = hi ? r : w[0][j];
            o[2 * j + 1] = hi ? w[1][j] : r;
          }
          if (!row_ok[mt][h] || SPD_DBG_BIT(1)) continue;
          const int64_t ch0 = (int64_t)cb * 32 + (hi ? 16 : 0) + 4 * cq;
          T* dst = orow[mt][h] + ch0 * L;
          if (ch0 + 4 <= chunk_lim[mt][h]) {
            stg_v8(dst, o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (ch0 + c < chunk_lim[mt][h]) *reinterpret_cast<uint2*>(dst + c * L) = make_uint2(o[2 * c], o[2 * c + 1]);
          }
        }
      };
      uint32_t va[2][16], vb[2][16];
      load(0, va);
      tmem_wait_ld();
#pragma unroll
      for (int bi = 0; bi < TB; ++bi) {
        uint32_t(&cur)[2][16] = (bi & 1) ? vb : va;
        uint32_t(&nxt)[2][16] = (bi & 1) ? va : vb;
        if (bi + 1 < TB) load(bi + 1, nxt);
        if (bi == TB - 1) {
          // every accumulator column is in registers: free the stage
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG2 && crank != 0) mbar_arrive_cluster(bar_acce + 8 * acc, 0);
            else mbar_arrive(bar_acce + 8 * acc);
          }
        }
        if (warp == 0 && lane == 0 && bi == 0) SPD_TRACE(10, it);
        emit(bi, cur);
        if (bi + 1 < TB) tmem_wait_ld();
      }
      if (warp == 0 && lane == 0) SPD_TRACE(9, it);
      if (publishing && pub_tile(id) && !SPD_DBG_BIT(2048)) {
        const int ps = pit % kNPub;
        mbar_wait(bar_pube + 8 * ps, ((pit / kNPub) & 1) ^ 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_pubf + 8 * ps);
        ++pit;
      }
    }
    } else {
    const int quad = warp % 4;       // TMEM lane quadrant (warp id mod 4)
    const int grp = warp / 4;        // epilogue group: tiles it == grp (mod kEpiGroups)
    const int m = quad * 32 + lane;  // TMEM lane == M row
    // output row of the tile: m / L, or the inverse of the 3D z-split map (aot.cpp lane_of:
    // quadrant y / 2, half z / 2, 4-lane group 2 (z % 2) + y % 2) or of the
    // L = 8 half split: quadrant (a % 8) / 2, half a / 8, 8-lane group a % 2)
    const int alpha = g.lane_map == 2   ? 8 * (2 * ((m % 32) / 16) + (m % 16) / 8) + 2 * quad + (m % 8) / 4
                      : g.lane_map == 3 ? 8 * ((m % 32) / 16) + 2 * quad + (m % 16) / 8
                                        : m / L;
    const int d = lane % L;          // position in the L-lane group
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    // output row of this lane in each M-tile (M-tile t holds rows alpha + t*R_OUT)
    int odz[MT], ody[MT], odx[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      odz[mt] = g.out_dz[alpha + (mt + (int)crank) * C::R_OUT];
      ody[mt] = g.out_dy[alpha + (mt + (int)crank) * C::R_OUT];
      odx[mt] = g.out_dx[alpha + (mt + (int)crank) * C::R_OUT];
    }
    int it = 0;
    int pit = 0;  // published tiles (publish ring index)
    int2 e_nx = fetch(wid0);
    int e_gi = wid0;
    for (int gi = wid0; gi < total; gi += wstride, ++it) {
      if (kEpiGroups > 1 && (it % kEpiGroups) != grp) continue;
      const int acc = it % NACC;
      const uint32_t aphase = (it / NACC) & 1;
      const int2 e_cur = e_gi == gi ? e_nx : fetch(gi);
      e_nx = fetch(gi + wstride);
      e_gi = gi + wstride;
      const TileId id = decode_e(gi, e_cur);
      T* out = static_cast<T*>(p.buf[(id.step + 1) & 1]);
      bool row_ok[MT];
      int64_t chunk_lim[MT];  // whole chunks in this row
      int64_t x_lim[MT];      // valid points of this row from its chunk 0 (a partial last chunk:
                              // an embedded radius-2 grid's width is a multiple of 6, not 8)
      T* orow[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int64_t z = id.z0 + odz[mt];
        const int64_t y = id.y0 + ody[mt];
        const int64_t xr = id.x0 + odx[mt];  // x of chunk 0 of this row
        if (g.d == 3) row_ok[mt] = z >= p.row_lo && z < p.row_hi && y < p.ny;
        else if (g.d == 2) row_ok[mt] = y >= p.row_lo && y < p.row_hi;
        else row_ok[mt] = true;
        x_lim[mt] = p.nx - xr;
        chunk_lim[mt] = x_lim[mt] / L;
        orow[mt] = out + p.origin + z * p.plane + y * p.pitch + xr;
      }
      if (warp == 0 && lane == 0) SPD_TRACE(12, it);
      mbar_wait(bar_accf + 8 * acc, aphase);
      tc_fence_after();
      if (warp == 0 && lane == 0) SPD_TRACE(8, it);
      // Per 32-column batch: pack chunk pairs to 16-bit, xor-butterfly inside
      // the L-lane group so each lane ends up owning 2*PPD consecutive chunks
      // (32 points = 64 B), then two 256-bit full-line stores.  Batches go in
      // pairs: the two butterflies are independent shuffle chains the
      // scheduler interleaves (the epilogue is latency-bound), and the TMEM
      // load of the next batch is in flight while the current one is packed.
      constexpr int NB = C::ACC_STAGE / MT / 32;  // batches per M-tile (pair: both x-halves)
      constexpr int TB = MT * NB;     // batches per tile (batch bi: M-tile bi / NB, column batch bi % NB)
      static_assert(TB % 2 == 0, "epilogue processes batch pairs");
      constexpr int PPD = 16 / L;  // packed words (chunk pairs) per destination lane
      const uint32_t tcol = lane_base + C::ACC_COL + acc * C::ACC_STAGE;  // batch bi at tcol + 32 bi
      // bw[k*L + dd] = chunk pair (2j, 2j+1), j = dd*PPD + k, destined to
      // lane dd of the group.  With the sigma column order (CPL = 2) chunk
      // 2j sits at column (j/8)*16 + j%8 and chunk 2j+1 eight columns later.
      auto pack = [&](const uint32_t(&v)[32], uint32_t(&bw)[16]) {
#pragma unroll
        for (int dd = 0; dd < L; ++dd)
#pragma unroll
          for (int k = 0; k < PPD; ++k) {
            // destination lane dd owns chunk pairs dd*PPD/2 + [0, PPD/2) of
            // each half batch (16 chunks): two 32-byte pieces 16 chunks apart,
            // so each 256-bit store instruction of the warp writes whole
            // 128-byte lines (4 or 8 lanes side by side)
            const int j = (k < PPD / 2 ? 0 : 8) + dd * (PPD / 2) + k % (PPD / 2);
            const int c0 = C::CPL == 2 ? (j / 8) * 16 + (j % 8) : 2 * j;
            const int c1 = C::CPL == 2 ? c0 + 8 : 2 * j + 1;
            bw[k * L + dd] = Cvt<T>::pack(__uint_as_float(v[c0]), __uint_as_float(v[c1]));
          }
      };
      // lane d ends with bw[k*L + s] = source lane s's pair of chunks for
      // its pair index k: PPD consecutive chunks at d*PPD and PPD more at
      // 16 + d*PPD; the 16 output words (x = L*chunk + s, pairs of s), piece
      // by piece in ascending x.
      auto store = [&](int bi, const uint32_t(&bw)[16]) {
        const int mt = bi / NB, cb = bi % NB;
        if (!row_ok[mt] || SPD_DBG_BIT(1)) return;
        uint32_t w[16];
#pragma unroll
        for (int k = 0; k < PPD; ++k)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < L / 2; ++u)
              w[(2 * k + h) * (L / 2) + u] =
                  __byte_perm(bw[k * L + 2 * u], bw[k * L + 2 * u + 1], h ? 0x7632 : 0x5410);
        const int64_t c_lane = (int64_t)cb * 32 + PPD * d;  // first chunk of piece 0; piece 1 at +16
        T* dst = orow[mt] + c_lane * L;
        if (c_lane + 16 + PPD <= chunk_lim[mt]) {
          stg_v8(dst, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7]);
          stg_v8(dst + 16 * L, w[8], w[9], w[10], w[11], w[12], w[13], w[14], w[15]);
        } else {
#pragma unroll
          for (int c = 0; c < 2 * PPD; ++c) {
            const int64_t ch = c_lane + (c / PPD) * 16 + c % PPD;
            if (ch < chunk_lim[mt]) {
              T* dc = orow[mt] + ch * L;
              if (L == 4) *reinterpret_cast<uint2*>(dc) = make_uint2(w[2 * c], w[2 * c + 1]);
              else *reinterpret_cast<uint4*>(dc) = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
            } else if (ch * L < x_lim[mt]) {  // partial last chunk: point by point
              uint16_t* dc = reinterpret_cast<uint16_t*>(orow[mt] + ch * L);
              const int n = (int)(x_lim[mt] - ch * L);
#pragma unroll
              for (int e = 0; e < L; ++e)
                if (e < n) dc[e] = (uint16_t)(w[(L / 2) * c + e / 2] >> (16 * (e & 1)));
            }
          }
        }
      };
      uint32_t va[32], vb[32];
      uint32_t b0[16], b1[16];
      tmem_ld_x32(tcol, va);
      tmem_wait_ld();
#pragma unroll
      for (int pr = 0; pr < TB / 2; ++pr) {
        const int cb0 = 2 * pr, cb1 = 2 * pr + 1;
        tmem_ld_x32(tcol + cb1 * 32, vb);
        if (warp == 0 && lane == 0 && pr == 0) SPD_TRACE(10, it);
        pack(va, b0);
        tmem_wait_ld();
        if (cb1 + 1 < TB) tmem_ld_x32(tcol + (cb1 + 1) * 32, va);
        pack(vb, b1);
        if (pr == TB / 2 - 1) {
          // every accumulator column is in registers: free the stage
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG2 && crank != 0) mbar_arrive_cluster(bar_acce + 8 * acc, 0);
            else mbar_arrive(bar_acce + 8 * acc);
          }
        }
#pragma unroll
        for (int b = 1; b < L; b <<= 1) {
          if (SPD_DBG_BIT(16)) break;
          const bool upper = (d & b) != 0;
#pragma unroll
          for (int k = 0; k < PPD; ++k) {
#pragma unroll
            for (int dd = 0; dd < L; ++dd) {
              if (dd & b) continue;
              const uint32_t s0 = upper ? b0[k * L + dd] : b0[k * L + (dd | b)];
              const uint32_t s1 = upper ? b1[k * L + dd] : b1[k * L + (dd | b)];
              const uint32_t r0 = __shfl_xor_sync(0xffffffffu, s0, b);
              const uint32_t r1 = __shfl_xor_sync(0xffffffffu, s1, b);
              if (upper) {
                b0[k * L + dd] = r0;
                b1[k * L + dd] = r1;
              } else {
                b0[k * L + (dd | b)] = r0;
                b1[k * L + (dd | b)] = r1;
              }
            }
          }
        }
        if (warp == 0 && lane == 0 && pr == 0) SPD_TRACE(11, it);
        store(cb0, b0);
        store(cb1, b1);
        if (cb1 + 1 < TB) tmem_wait_ld();
      }
      if (warp == 0 && lane == 0) SPD_TRACE(9, it);
      if (publishing && pub_tile(id) && !SPD_DBG_BIT(2048)) {
        // hand the tile to the publisher warp (release at CTA scope after
        // the warp's stores); the gpu-scope release happens off this path
        const int ps = pit % kNPub;
        mbar_wait(bar_pube + 8 * ps, ((pit / kNPub) & 1) ^ 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_pubf + 8 * ps);
        ++pit;
      }
    }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) SPD_TRACE(15, 0);
  if constexpr (CG2) cluster_sync_all();  // the peer's MMAs into this TMEM are complete
  if (warp == kMmaWarp) {
    tc_fence_after();
    if constexpr (CG2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Support kernels

template <typename T>
__device__ __forceinline__ T from_f64(double x);
template <>
__device__ __forceinline__ __half from_f64<__half>(double x) { return __double2half(x); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f64<__nv_bfloat16>(double x) { return __double2bfloat16(x); }

struct DenseMap {
  int64_t nzd, nyd, nxd;  // dense extents incl. halo (nzd = 1 for 2D/1D)
  int64_t h;
  int d;
};

// dense natural (halo-padded) fp64 <-> device layout
template <typename T>
__global__ void pack_kernel(DenseMap dm, int64_t pitch, int64_t plane, int64_t origin, const double* dense, T* dev) {
  int64_t n = dm.nzd * dm.nyd * dm.nxd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t xx = i % dm.nxd, rest = i / dm.nxd;
    int64_t yy = rest % dm.nyd, zz = rest / dm.nyd;
    int64_t z = dm.d == 3 ? zz - dm.h : 0;
    int64_t o = origin + z * plane + (yy - dm.h) * pitch + (xx - dm.h);
    dev[o] = from_f64<T>(dense[i]);
  }
}

template <typename T>
__global__ void unpack_kernel(DenseMap dm, int64_t pitch, int64_t plane, int64_t origin, const T* dev, double* dense) {
  int64_t n = dm.nzd * dm.nyd * dm.nxd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t xx = i % dm.nxd, rest = i / dm.nxd;
    int64_t yy = rest % dm.nyd, zz = rest / dm.nyd;
    int64_t z = dm.d == 3 ? zz - dm.h : 0;
    int64_t o = origin + z * plane + (yy - dm.h) * pitch + (xx - dm.h);
    dense[i] = (double)static_cast<float>(dev[o]);
  }
}

// naive_apply on device in fp64 (core.py:151-182): same row-major tap order,
// acc = 0; acc = acc + (w * x) with separate roundings (no FMA contraction).
__global__ void naive_f64_kernel(int d, int r, const double* __restrict__ w, int64_t nz, int64_t ny, int64_t nx,
                                 int64_t h, const double* __restrict__ in, double* __restrict__ out) {
  const int64_t nxd = nx + 2 * h, nyd = (d >= 2) ? ny + 2 * h : ny + 2 * h;
  const int64_t n = nz * ny * nx;
  const int span = 2 * r + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = i % nx, rest = i / nx;
    int64_t y = rest % ny, z = rest / ny;
    double acc = 0.0;
    if (d == 3) {
      int t = 0;
      for (int rz = -r; rz <= r; ++rz)
        for (int ry = -r; ry <= r; ++ry)
          for (int rx = -r; rx <= r; ++rx, ++t) {
            double v = in[((z + h + rz) * nyd + (y + h + ry)) * nxd + (x + h + rx)];
            acc = __dadd_rn(acc, __dmul_rn(w[t], v));
          }
      out[((z + h) * nyd + (y + h)) * nxd + (x + h)] = acc;
    } else if (d == 2) {
      int t = 0;
      for (int ry = -r; ry <= r; ++ry)
        for (int rx = -r; rx <= r; ++rx, ++t) {
          double v = in[(y + h + ry) * nxd + (x + h + rx)];
          acc = __dadd_rn(acc, __dmul_rn(w[t], v));
        }
      out[(y + h) * nxd + (x + h)] = acc;
    } else {
      for (int t = 0; t < span; ++t) {
        double v = in[(y + h) * nxd + (x + h + t - r)];
        acc = __dadd_rn(acc, __dmul_rn(w[t], v));
      }
      out[(y + h) * nxd + (x + h)] = acc;
    }
  }
}

// Halo rows (2D: rows, 3D: planes) <-> contiguous message buffers.
template <typename T>
__global__ void halo_copy_kernel(const T* src, int64_t src_off, T* dst, int64_t dst_off, int64_t count,
                                 int64_t run, int64_t src_stride, int64_t dst_stride) {
  // `count` runs of `run` elements; run i at src_off + i*src_stride.
  int64_t n = count * run;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = k / run, j = k % run;
    dst[dst_off + i * dst_stride + j] = src[src_off + i * src_stride + j];
  }
}

// Single sparse MMA self test: D = decode(A, E) * B, M=128, K=32, N = n.
__global__ void mma_selftest_kernel(const uint16_t* a, const uint8_t* e, const uint16_t* b, int n, float* d) {
  __shared__ __align__(1024) uint8_t sB[256 * 64];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int sbo = 4 * 128;
  for (int idx = threadIdx.x; idx < 32 * n; idx += blockDim.x) {
    int k = idx / n, c = idx % n;
    *reinterpret_cast<uint16_t*>(sB + (c / 8) * sbo + (k / 8) * 128 + (c % 8) * 16 + (k % 8) * 2) = b[k * n + c];
  }
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  const int m = warp * 32 + lane;
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  const int E_COL = 256, A_COL = 264;
  {
    int m0 = m % 8, k1 = (m / 8) % 2, m2 = m / 16;
    uint32_t w = 0;
    for (int m1 = 0; m1 < 2; ++m1)
      for (int c4 = 0; c4 < 4; ++c4) w |= (uint32_t)(e[(m0 + 8 * m1 + 16 * m2) * 8 + 4 * k1 + c4] & 0xF) << (16 * m1 + 4 * c4);
    tmem_st_x1(lane_base + E_COL, w);
    for (int c = 0; c < 8; ++c) tmem_st_x1(lane_base + A_COL + c, (uint32_t)a[m * 16 + 2 * c] | ((uint32_t)a[m * 16 + 2 * c + 1] << 16));
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && lane == 0) {
    mma_sp_ts(tmem, tmem + A_COL, umma_desc(smem_u32(sB), 128, sbo), tmem + E_COL, idesc_sparse_f16(128, n, false), 0u);
    tc_commit(smem_u32(&bar));
  }
  __syncwarp();
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  for (int c0 = 0; c0 < n; c0 += 32) {
    uint32_t v[32];
    tmem_ld_x32(lane_base + c0, v);
    tmem_wait_ld();
    for (int j = 0; j < 32 && c0 + j < n; ++j) d[m * n + c0 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// Host side: plan, dispatch

struct DevInfo {
  int sms = 0;
};

static int cuda_err(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SPD_OK;
  return set_error(SPD_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace spd

struct spd_plan {
  spd::Geometry g;
  int d, r, parity, dtype, device, L, n_rows;
  std::vector<double> coeffs;
  std::vector<double> row_values;  // n_rows x L x L
  std::vector<uint8_t> row_meta;   // n_rows x L x (L/2) x 2
  std::vector<uint16_t> a_img;     // S x 128 x 16
  std::vector<uint32_t> e_words;   // S x 128
  uint16_t* d_a = nullptr;
  uint32_t* d_e = nullptr;
  int sms = 0;
  // persistent work orders (device), keyed by (steps, sweep, lag, n_bands);
  // built on first use under orders_mu, read-only afterwards
  std::map<std::tuple<int, int, int, int>, int2*> orders;
  std::mutex orders_mu;
};

namespace spd {

// Zeroed per-band counters for ONE persistent launch, stream-ordered
// (cudaMallocAsync + memset; freed with cudaFreeAsync after the launch), so
// launches of the same plan on different streams or threads never share them.
static int launch_counters(int n, cudaStream_t st, unsigned int** out) {
  *out = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(out), sizeof(unsigned int) * n, st);
  if (e != cudaSuccess) return cuda_err(e, "counter alloc");
  return cuda_err(cudaMemsetAsync(*out, 0, sizeof(unsigned int) * n, st), "counter reset");
}

template <typename T, int L, int PARITY, int NTILE, int NSTAGE, int NNAT, int NACC, int RIN, int MT = 1, int MTR = 0,
          bool CG2 = false, int PW = kProdWarpsDefault, bool EDGE = false>
static int launch_step(const spd_plan* plan, StepParams& sp, cudaStream_t stream) {
  using C = Cfg<L, NTILE, NSTAGE, NNAT, NACC, RIN, MT, MTR, CG2, PW>;
  if (CG2 != (plan->g.cg2 != 0)) return set_error(SPD_EUNSUPPORTED, "CTA-pair geometry mismatch");
  // the EDGE instantiation (2D fast paths) decodes only edge-first one-step
  // launches; the others take edge_order through their runtime path
  if (EDGE && !(sp.edge_order != 0 && sp.steps == 1 && !sp.use_order))
    return set_error(SPD_EUNSUPPORTED, "edge-first instantiation mismatch");
  auto kern = spider_step_kernel<T, L, PARITY, NTILE, NSTAGE, NNAT, NACC, RIN, MT, MTR, CG2, PW, EDGE>;
  if (plan->g.r_in != RIN) return set_error(SPD_EUNSUPPORTED, "tile geometry mismatch (r_in %d)", plan->g.r_in);
  if ((L == 4 && MT == 1 && !CG2) != (plan->g.lane_map == 1))
    return set_error(SPD_EUNSUPPORTED, "accumulator lane map mismatch (%d)", plan->g.lane_map);
  {  // the MMA issuer's compile-time schedule must be the plan's
    constexpr int RPM = 4 / C::KC;
    constexpr int RM = C::RIN_MMA;
    if (plan->g.s != (RM + RPM - 1) / RPM) return set_error(SPD_EUNSUPPORTED, "MMA count mismatch (%d)", plan->g.s);
    if (plan->g.m_tiles != MT || (MT > 1 && plan->g.mt_rows != MTR))
      return set_error(SPD_EUNSUPPORTED, "M-tile geometry mismatch (%d)", plan->g.m_tiles);
    for (int s = 0; s < plan->g.s; ++s)
      if (!CG2 && plan->g.mma_half[s] != (int)((ct_halves_mask<C, L, RIN, MT>() >> (2 * s)) & 3))
        return set_error(SPD_EUNSUPPORTED, "M = 64 schedule mismatch (MMA %d)", s);
    for (int s = 0; s < plan->g.s; ++s)
      if (plan->g.start_row[s] != (s * RPM + RPM <= RM ? s * RPM : RM - RPM))
        return set_error(SPD_EUNSUPPORTED, "MMA start row mismatch (%d)", s);
  }
  sp.nat_bytes = sp.use_tmap ? sp.nbox * sp.box_slot : plan->g.r_in * C::ROW_BYTES;
  if (sp.rowmajor) sp.nat_bytes = (sp.nbox * sp.boxw * 2 * plan->g.r_in + 127) / 128 * 128;
  if (!sp.use_tmap) {
    sp.nbox = 1;
    sp.boxw = C::ROW_ELEMS;
    sp.box_slot = sp.nat_bytes;
  }
  const size_t smem = (size_t)NSTAGE * (NTILE / 8) * plan->g.b_sbo + (size_t)NNAT * sp.nat_bytes + C::STG_BYTES +
                      8 * (2 * NSTAGE + 2 * NACC + 2 * NNAT + 2 * kNPub + 2 * kDQ) + 16;
  if (smem > 232448) return set_error(SPD_EUNSUPPORTED, "shared memory budget exceeded (%zu B)", smem);
  if (C::A_COL + 8 * plan->g.s > 512) return set_error(SPD_EUNSUPPORTED, "TMEM budget exceeded (S=%d)", plan->g.s);
  // the attribute is per device: remember which devices this thread set it on
  static thread_local uint64_t configured = 0;
  const uint64_t dev_bit = 1ull << (plan->device & 63);
  if (!(configured & dev_bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute");
    configured |= dev_bit;
  }
  if (sp.n_tiles <= 0) return SPD_OK;
  const int64_t work = (int64_t)sp.n_tiles * sp.steps * (CG2 ? 2 : 1);
  int grid = work < plan->sms ? (int)work : plan->sms;
  if (CG2) grid &= ~1;  // whole CTA pairs
  if (CG2 && sp.steps > 1) return set_error(SPD_EUNSUPPORTED, "persistent launch not supported in CTA-pair mode");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  unsigned int nattr = 1;
  if (CG2) {
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    nattr = 2;
  }
  if (sp.steps > 1) {
    attr[0].id = cudaLaunchAttributeCooperative;  // co-residency: cross-step waits need every CTA running
    attr[0].val.cooperative = 1;
  } else {
    static const char* pdl_env = getenv("SPD_NO_PDL");
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_env ? 0 : 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = nattr;
  return cuda_err(cudaLaunchKernelEx(&cfg, kern, sp), "spider_step_kernel launch");
}

template <typename T, int PARITY>
static int dispatch_par(const spd_plan* plan, StepParams& sp, cudaStream_t st) {
  const Geometry& g = plan->g;
  // <T, L, PARITY, NTILE, B-image stages, natural-row stages, accumulator
  //  stages, items per producer warp>; stage counts fill the 227 KB of smem
  // (scan in profiles/r01_tuning.txt).
  if (g.L == 4 && g.n_tile == 128 && g.r_in == 34)
    return sp.edge_order
               ? launch_step<T, 4, PARITY, 128, SPD_2D_NSTAGE, SPD_2D_NNAT, SPD_2D_NACC, 34, 1, 0, false,
                             kProdWarpsDefault, true>(plan, sp, st)
               : launch_step<T, 4, PARITY, 128, SPD_2D_NSTAGE, SPD_2D_NNAT, SPD_2D_NACC, 34>(plan, sp, st);
  if (g.L == 4 && g.n_tile == 128 && g.r_in == 32) return launch_step<T, 4, PARITY, 128, 2, 2, 3, 32>(plan, sp, st);
  if (g.L == 4 && g.n_tile == 32 && g.r_in == 100 && g.m_tiles == 2)
    return launch_step<T, 4, PARITY, 32, SPD_3D_NSTAGE, SPD_3D_NNAT, SPD_3D_NACC, 100, 2, 40, false, SPD_3D_PW>(plan,
                                                                                                              sp, st);
  if (g.L == 4 && g.n_tile == 32 && g.r_in == 100 && g.cg2)
    return launch_step<T, 4, PARITY, 32, 2, SPD_3D_NNAT, 3, 100, 1, 0, true, SPD_3D_PW>(plan, sp, st);
  if (g.L == 8 && g.n_tile == 64 && g.r_in == 22)
    return sp.edge_order
               ? launch_step<T, 8, PARITY, 64, SPD_L8_NSTAGE, SPD_L8_NNAT, SPD_L8_NACC, 22, 1, 0, false, SPD_L8_PW,
                             true>(plan, sp, st)
               : launch_step<T, 8, PARITY, 64, SPD_L8_NSTAGE, SPD_L8_NNAT, SPD_L8_NACC, 22, 1, 0, false, SPD_L8_PW>(
                     plan, sp, st);
  if (g.L == 8 && g.n_tile == 64 && g.r_in == 16)
    return launch_step<T, 8, PARITY, 64, 3, 4, 4, 16, 1, 0, false, SPD_L8_PW>(plan, sp, st);
  // generic radii (2D: r_in = 128/L + 2r; 1D: r_in = 128/L)
  if (g.L == 6 && g.r_in == 25) return launch_step<T, 6, PARITY, 64, 2, 3, 4, 25, 1, 0, false, SPD_GEN_PW>(plan, sp, st);
  if (g.L == 6 && g.r_in == 21) return launch_step<T, 6, PARITY, 64, 2, 3, 4, 21, 1, 0, false, SPD_GEN_PW>(plan, sp, st);
  if (g.L == 10 && g.r_in == 20) return launch_step<T, 10, PARITY, 64, 2, 1, 4, 20, 1, 0, false, SPD_GEN_PW>(plan, sp, st);
  if (g.L == 10 && g.r_in == 12) return launch_step<T, 10, PARITY, 64, 2, 2, 4, 12, 1, 0, false, SPD_GEN_PW>(plan, sp, st);
  if (g.L == 12 && g.r_in == 20) return launch_step<T, 12, PARITY, 64, 2, 1, 4, 20, 1, 0, false, SPD_GEN_PW>(plan, sp, st);
  if (g.L == 12 && g.r_in == 10) return launch_step<T, 12, PARITY, 64, 2, 2, 4, 10, 1, 0, false, SPD_GEN_PW>(plan, sp, st);
  if (g.L == 14 && g.r_in == 21) return launch_step<T, 14, PARITY, 64, 2, 1, 4, 21, 1, 0, false, SPD_GEN_PW>(plan, sp, st);
  if (g.L == 14 && g.r_in == 9) return launch_step<T, 14, PARITY, 64, 2, 2, 4, 9, 1, 0, false, SPD_GEN_PW>(plan, sp, st);
  if (g.L == 16 && g.r_in == 22) return launch_step<T, 16, PARITY, 64, 1, 1, 4, 22, 1, 0, false, SPD_GEN_PW>(plan, sp, st);
  if (g.L == 16 && g.r_in == 8) return launch_step<T, 16, PARITY, 64, 2, 2, 4, 8, 1, 0, false, SPD_GEN_PW>(plan, sp, st);
  return set_error(SPD_EUNSUPPORTED, "no kernel instantiation for L=%d n_tile=%d", g.L, g.n_tile);
}

static int dispatch(const spd_plan* plan, StepParams& sp, cudaStream_t st) {
  {  // launches go to the current device: it must be the one holding the plan's operands
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != plan->device)
      return set_error(SPD_EINVAL, "plan lives on device %d but device %d is current", plan->device, cur);
  }
  if (plan->dtype == SPD_DTYPE_F16)
    return plan->parity == 0 ? dispatch_par<__half, 0>(plan, sp, st) : dispatch_par<__half, 1>(plan, sp, st);
  return plan->parity == 0 ? dispatch_par<__nv_bfloat16, 0>(plan, sp, st)
                           : dispatch_par<__nv_bfloat16, 1>(plan, sp, st);
}

static int64_t roundup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

#ifdef SPD_DEVEL
static unsigned long long* g_trace = nullptr;       // debug timeline buffer (SPD_TRACE), device view
#endif
static unsigned long long* g_trace_host = nullptr;  // mapped pinned host view (readable during a hang)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// Tensor map of an input buffer for the loader warp: the stored grid as a
// [planes][rows][pitch] (3D) or [rows][pitch] (2D) tensor of 16-bit elements;
// one box = nbox-th of the tile's halo-padded input block.
static int make_tensor_map(const spd_plan* plan, const spd_grid_desc* gd, const void* buf, StepParams& sp,
                           CUtensorMap* map) {
  const Geometry& g = plan->g;
  // same split as Cfg::NBOX / Cfg::BOXW: <= 256-element boxes, widths a
  // multiple of 8 (boxes may overrun the row; TMA zero-fills out of bounds)
  const int row_elems = g.n_tile * g.L + 16;
  sp.nbox = (row_elems + 255) / 256;
  sp.boxw = ((row_elems + sp.nbox - 1) / sp.nbox + 7) / 8 * 8;
  sp.box_slot = (int)roundup((int64_t)sp.boxw * 2 * g.r_in, 128);
  // (The producer quarter-warp straddling a box boundary reads with a 2-way
  // bank conflict -- ncu: 5 wavefronts instead of 4 per LDS.128 on B9.
  // Skewing the box slots to continue the row's bank pattern is illegal:
  // tensor-TMA shared destinations must be 128-byte aligned (misaligned
  // address fault, r02).)
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return set_error(SPD_ECUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  const int64_t rows = gd->plane / gd->pitch;
  if (g.d == 2 && g.L != 4 && g.L != 8) {
    // generic radii: one box per tile through the view (x, box, row) with
    // box stride boxw elements, so the rows land contiguous in shared memory
    cuuint64_t vdims[3] = {(cuuint64_t)gd->pitch, (cuuint64_t)sp.nbox, (cuuint64_t)rows};
    cuuint64_t vstrides[2] = {(cuuint64_t)sp.boxw * 2, (cuuint64_t)gd->pitch * 2};
    cuuint32_t vbox[3] = {(cuuint32_t)sp.boxw, (cuuint32_t)sp.nbox, (cuuint32_t)g.r_in};
    cuuint32_t vestr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(buf), vdims, vstrides, vbox, vestr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(SPD_ECUDA, "cuTensorMapEncodeTiled (row view) failed (%d)", (int)r);
    sp.use_tmap = 1;
    sp.rowmajor = 1;
    return SPD_OK;
  }
  cuuint64_t dims[3] = {(cuuint64_t)gd->pitch, (cuuint64_t)rows, (cuuint64_t)(gd->alloc_elems / gd->plane)};
  cuuint64_t strides[2] = {(cuuint64_t)gd->pitch * 2, (cuuint64_t)gd->plane * 2};
  cuuint32_t box[3] = {(cuuint32_t)sp.boxw, (cuuint32_t)(g.tile_y + 2 * g.r), (cuuint32_t)(g.tile_z + 2 * g.r)};
  cuuint32_t estr[3] = {1, 1, 1};
  const cuuint32_t rank = g.d == 3 ? 3 : 2;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, rank, const_cast<void*>(buf), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SPD_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  sp.use_tmap = 1;
  return SPD_OK;
}

// buf0 holds the input of the launch's first step; steps > 1 alternate buffers
// inside the (persistent) launch.
// A host thread that has made no runtime call yet has no current context, and
// the driver-API calls below (cuTensorMapEncodeTiled) then fail with
// CUDA_ERROR_INVALID_CONTEXT: bind the current device's primary context once
// per thread and device (cudaSetDevice of the device that is already current).
static void bind_context() {
  static thread_local uint64_t bound = 0;
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return;
  const uint64_t bit = 1ull << (cur & 63);
  if (!(bound & bit)) {
    cudaSetDevice(cur);
    bound |= bit;
  }
}

static int fill_step_params(const spd_plan* plan, const spd_grid_desc* gd, const void* buf0, void* buf1, int64_t lo,
                            int64_t hi, int steps, StepParams& sp) {
  const Geometry& g = plan->g;
  bind_context();
  std::memset(&sp, 0, sizeof(sp));
  sp.g = g;
  sp.buf[0] = const_cast<void*>(buf0);
  sp.buf[1] = buf1;
  sp.steps = steps;
  sp.pitch = gd->pitch;
  sp.plane = gd->plane;
  sp.origin = gd->origin;
  sp.nx = gd->nx;
  sp.ny = gd->ny;
  sp.a_img = plan->d_a;
  sp.e_words = plan->d_e;
  sp.tiles_x = (int)((gd->nx + g.tile_x - 1) / g.tile_x);
  if (g.d == 3) {
    lo = lo < 0 ? 0 : lo;
    hi = hi > gd->nz ? gd->nz : hi;
    sp.row_lo = lo;
    sp.row_hi = hi;
    sp.tiles_y = (int)((gd->ny + g.tile_y - 1) / g.tile_y);
    sp.tile_y0 = 0;
    sp.tile_z0 = (int)(lo / g.tile_z);
    sp.tiles_z = hi > lo ? (int)((hi + g.tile_z - 1) / g.tile_z - sp.tile_z0) : 0;
  } else if (g.d == 2) {
    lo = lo < 0 ? 0 : lo;
    hi = hi > gd->ny ? gd->ny : hi;
    sp.row_lo = lo;
    sp.row_hi = hi;
    sp.tiles_z = 1;
    sp.tile_z0 = 0;
    sp.tile_y0 = (int)(lo / g.tile_y);
    sp.tiles_y = hi > lo ? (int)((hi + g.tile_y - 1) / g.tile_y - sp.tile_y0) : 0;
  } else {
    sp.row_lo = 0;
    sp.row_hi = 1;
    sp.tiles_y = sp.tiles_z = 1;
  }
  sp.band_stride = 1;
  sp.n_tiles = sp.tiles_x * sp.tiles_y * sp.tiles_z;
  if (g.d == 3) {
    sp.n_bands = sp.tiles_z;
    sp.per_band = sp.tiles_x * sp.tiles_y;
  } else if (g.d == 2) {
    sp.n_bands = sp.tiles_y;
    sp.per_band = sp.tiles_x;
  } else {
    sp.n_bands = sp.tiles_x;
    sp.per_band = 1;
  }
  sp.trace = nullptr;
#ifdef SPD_DEVEL
  const char* dbg_env = getenv("SPD_DBG");
  sp.dbg = dbg_env ? atoi(dbg_env) : 0;
  if (getenv("SPD_TRACE")) {
    if (!g_trace_host) {
      cudaHostAlloc(&g_trace_host, 8 * 16 * 64 * sizeof(unsigned long long), cudaHostAllocMapped);
      std::memset(g_trace_host, 0, 8 * 16 * 64 * sizeof(unsigned long long));
      cudaHostGetDevicePointer(&g_trace, g_trace_host, 0);
    }
    sp.trace = g_trace;
  }
#endif
  sp.zoff = (int)(gd->origin / gd->plane);
  sp.yoff = (int)((gd->origin % gd->plane) / gd->pitch);
  sp.xoff = (int)(gd->origin % gd->pitch);
  sp.use_tmap = 0;
  if (g.d >= 2) {
    int rc = make_tensor_map(plan, gd, buf0, sp, &sp.tmap[0]);
    if (rc) return rc;
    return make_tensor_map(plan, gd, buf1, sp, &sp.tmap[1]);
  }
  return SPD_OK;
}

// Persistent work order: sweeps of S steps, step s+1 lagging step s by `lag`
// bands.  The data step s writes is re-read by step s+1 about `lag`
// wavefronts later; S is sized so that everything in flight between the
// leading and trailing steps of a sweep (~ 2 buffers x lag x S bands) stays
// well inside the 126 MB L2.  SPD_SWEEP / SPD_LAG override (tuning).
static int wavefront_order(const spd_plan* cplan, const spd_grid_desc* gd, StepParams& sp) {
  spd_plan* plan = const_cast<spd_plan*>(cplan);
  const Geometry& g = plan->g;
  const int64_t band_bytes =
      2 * (g.d == 3 ? (int64_t)g.tile_z * gd->plane : (g.d == 2 ? (int64_t)g.tile_y * gd->pitch : (int64_t)g.tile_x));
  const char* lag_env = getenv("SPD_LAG");
  const char* sweep_env = getenv("SPD_SWEEP");
  int lag = lag_env ? atoi(lag_env) : 3;
  if (lag < 2) lag = 2;
  int64_t S = (int64_t)40 << 20;
  S /= 2 * lag * (band_bytes > 0 ? band_bytes : 1);
  if (sweep_env) S = atoi(sweep_env);
  if (S < 1) S = 1;
  if (S > 64) S = 64;
  if (S > sp.steps) S = sp.steps;
  sp.sweep = (int)S;
  sp.lag = lag;
  const int64_t pairs = (int64_t)sp.steps * sp.n_bands;
  if (pairs * sp.per_band >= ((int64_t)1 << 31))
    return set_error(SPD_EINVAL, "persistent launch too large (%lld work items)", (long long)(pairs * sp.per_band));
  sp.total = (int)(pairs * sp.per_band);
  const auto key = std::make_tuple(sp.steps, sp.sweep, sp.lag, sp.n_bands);
  std::lock_guard<std::mutex> lock(plan->orders_mu);
  auto it = plan->orders.find(key);
  if (it == plan->orders.end()) {
    // built once per key (synchronous upload: warm up outside graph capture)
    std::vector<int2> order;
    order.reserve((size_t)pairs);
    for (int k0 = 0; k0 < sp.steps; k0 += sp.sweep) {
      const int sk = sp.steps - k0 < sp.sweep ? sp.steps - k0 : sp.sweep;
      for (int w = 0; w < lag * (sk - 1) + sp.n_bands; ++w)
        for (int s = 0; s < sk; ++s) {
          const int band = w - lag * s;
          if (band >= 0 && band < sp.n_bands) order.push_back(make_int2(k0 + s, band));
        }
    }
    int2* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(int2) * order.size());
    if (e != cudaSuccess) return cuda_err(e, "order alloc");
    e = cudaMemcpy(d, order.data(), sizeof(int2) * order.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_err(e, "order upload");
    it = plan->orders.emplace(key, d).first;
  }
  sp.order = it->second;
  return SPD_OK;
}

static int check_desc(const spd_plan* plan, const spd_grid_desc* gd) {
  if (!plan || !gd) return set_error(SPD_EINVAL, "null plan or grid descriptor");
  if (gd->nx % plan->L != 0)
    return set_error(SPD_EINVAL, "grid width %lld must be a multiple of the x-chunk size L=%d", (long long)gd->nx,
                     plan->L);
  if (gd->halo < plan->r)
    return set_error(SPD_EINVAL, "grid halo %d too small for stencil radius %d", gd->halo, plan->r);
  return SPD_OK;
}

}  // namespace spd

// ---------------------------------------------------------------------------
// C ABI (device part)
extern "C" {

int spd_plan_create(int d, int r, int parity, const double* coeffs, int dtype, int device, spd_plan** out) {
  return spd_plan_create_ex(d, r, parity, coeffs, dtype, device, 0, out);
}

int spd_plan_create_ex(int d, int r, int parity, const double* coeffs, int dtype, int device, int flags,
                       spd_plan** out) {
  using namespace spd;
  if (!out) return set_error(SPD_EINVAL, "null output pointer");
  if (flags & ~(SPD_PLAN_CTA_PAIR | SPD_PLAN_NO_EMBED)) return set_error(SPD_EINVAL, "unknown plan flags 0x%x", flags);
  if ((flags & SPD_PLAN_CTA_PAIR) && d != 3) return set_error(SPD_EUNSUPPORTED, "CTA-pair plans are 3D only");
  *out = nullptr;
  if (d < 1 || d > 3) return set_error(SPD_EINVAL, "unsupported dimensionality %d", d);
  if (parity != 0 && parity != 1) return set_error(SPD_EINVAL, "bad parity code %d", parity);
  if (dtype != SPD_DTYPE_F16 && dtype != SPD_DTYPE_BF16) return set_error(SPD_EINVAL, "bad dtype code %d", dtype);
  int L = band_rows(r);
  if (L < 0) return L;
  spd_plan* p = new spd_plan();
  p->d = d;
  p->r = r;
  p->parity = parity;
  p->dtype = dtype;
  p->device = device;
  p->L = L;
  int span = 2 * r + 1;
  int ncoef = d == 1 ? span : (d == 2 ? span * span : span * span * span);
  p->coeffs.assign(coeffs, coeffs + ncoef);
  // Radius 2 in 1D / 2D runs as radius 3 with the coefficients embedded in a
  // zero ring: the L = 8 fast path (profiles/r02_embed.txt: B25 154 -> ~97
  // us) instead of the generic L = 6 one.  The grid keeps its own halo and
  // width rule (multiple of 6); the zero ring's reads land in the zero
  // padding or the TMA's zero fill, and the epilogue masks the last partial
  // 8-point chunk.  SPD_PLAN_NO_EMBED keeps the L = 6 path.
  int r_dev = r;
  std::vector<double> dev_coeffs(coeffs, coeffs + ncoef);
  if (r == 2 && d <= 2 && !(flags & SPD_PLAN_NO_EMBED)) {
    r_dev = 3;
    const int sp7 = 7;
    dev_coeffs.assign(d == 1 ? sp7 : sp7 * sp7, 0.0);
    for (int i = 0; i < (d == 1 ? 1 : span); ++i)
      for (int j = 0; j < span; ++j)
        dev_coeffs[(size_t)(d == 1 ? 0 : i + 1) * sp7 + j + 1] = coeffs[(size_t)(d == 1 ? 0 : i) * span + j];
  }
  const int L_dev = band_rows(r_dev);
  const int span_dev = 2 * r_dev + 1;
  p->n_rows = (int)dev_coeffs.size() / span_dev;
  p->row_values.resize((size_t)p->n_rows * L_dev * L_dev);
  p->row_meta.resize((size_t)p->n_rows * L_dev * (L_dev / 2) * 2);
  for (int k = 0; k < p->n_rows; ++k) {
    int rc = transform_row(r_dev, parity, dev_coeffs.data() + (size_t)k * span_dev,
                           p->row_values.data() + (size_t)k * L_dev * L_dev,
                           p->row_meta.data() + (size_t)k * L_dev * L_dev);
    if (rc) {
      delete p;
      return rc;
    }
  }
  int rc = build_geometry(d, r_dev, flags & ~SPD_PLAN_NO_EMBED, &p->g);
  if (rc) {
    delete p;
    return rc;
  }
  rc = pack_operands(p->g, p->n_rows, p->row_values.data(), p->row_meta.data(), dtype, p->a_img, p->e_words);
  if (rc) {
    delete p;
    return rc;
  }
  if (device >= 0) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_a, p->a_img.size() * sizeof(uint16_t));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_e, p->e_words.size() * sizeof(uint32_t));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_a, p->a_img.data(), p->a_img.size() * sizeof(uint16_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_e, p->e_words.data(), p->e_words.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
    cudaSetDevice(cur);
    if (e != cudaSuccess) {
      int code = cuda_err(e, "plan upload");
      spd_plan_destroy(p);
      return code;
    }
  }
  *out = p;
  return SPD_OK;
}

int spd_plan_destroy(spd_plan* plan) {
  if (!plan) return SPD_OK;
  if (plan->d_a) cudaFree(plan->d_a);
  if (plan->d_e) cudaFree(plan->d_e);
  for (auto& kv : plan->orders) cudaFree(kv.second);
  delete plan;
  return SPD_OK;
}

int spd_plan_info(const spd_plan* plan, int32_t* info) {
  if (!plan || !info) return spd::set_error(SPD_EINVAL, "null argument");
  const spd::Geometry& g = plan->g;
  info[0] = g.L;
  info[1] = g.r_in;
  info[2] = g.r_out;
  info[3] = g.s;
  info[4] = g.n_tile;
  info[5] = g.tile_z;
  info[6] = g.tile_y;
  info[7] = g.kc;
  info[8] = g.m_tiles;
  info[9] = g.mt_rows;
  info[10] = g.cg2;
  info[11] = g.r;  // device radius (3 for an embedded radius-2 stencil)
  return SPD_OK;
}

int spd_plan_operands(const spd_plan* plan, uint16_t* a_img, uint32_t* e_words, int32_t* start_rows) {
  if (!plan) return spd::set_error(SPD_EINVAL, "null plan");
  if (a_img) std::memcpy(a_img, plan->a_img.data(), plan->a_img.size() * sizeof(uint16_t));
  if (e_words) std::memcpy(e_words, plan->e_words.data(), plan->e_words.size() * sizeof(uint32_t));
  if (start_rows)
    for (int s = 0; s < plan->g.s; ++s) start_rows[s] = plan->g.start_row[s];
  return SPD_OK;
}

int spd_plan_lane_map(const spd_plan* plan, int32_t* lane) {
  if (!plan || !lane) return spd::set_error(SPD_EINVAL, "null argument");
  const spd::Geometry& g = plan->g;
  for (int a = 0; a < g.r_out; ++a)
    for (int i = 0; i < g.L; ++i) lane[g.L * a + i] = spd::lane_of(g, a, i);
  return SPD_OK;
}

int spd_plan_mma_halves(const spd_plan* plan, int32_t* half) {
  if (!plan || !half) return spd::set_error(SPD_EINVAL, "null argument");
  for (int s = 0; s < plan->g.s; ++s) half[s] = plan->g.mma_half[s];
  return SPD_OK;
}

int spd_plan_geometry(const spd_plan* plan, int32_t* in_off, int32_t* out_off) {
  if (!plan) return spd::set_error(SPD_EINVAL, "null plan");
  const spd::Geometry& g = plan->g;
  for (int b = 0; in_off && b < g.r_in; ++b) {
    in_off[3 * b] = g.in_dz[b];
    in_off[3 * b + 1] = g.in_dy[b];
    in_off[3 * b + 2] = g.in_dx[b];
  }
  for (int a = 0; out_off && a < g.r_out * (g.cg2 ? 2 : g.m_tiles); ++a) {
    out_off[3 * a] = g.out_dz[a];
    out_off[3 * a + 1] = g.out_dy[a];
    out_off[3 * a + 2] = g.out_dx[a];
  }
  return SPD_OK;
}

int spd_grid_layout(const spd_plan* plan, int64_t nz, int64_t ny, int64_t nx, int halo, spd_grid_desc* out) {
  using namespace spd;
  if (!plan || !out) return set_error(SPD_EINVAL, "null argument");
  if (halo < plan->r) return set_error(SPD_EINVAL, "grid halo %d too small for stencil radius %d", halo, plan->r);
  if (nx < 1 || ny < 1 || nz < 1) return set_error(SPD_EINVAL, "grid extent too small for its halo");
  if (nx % plan->L != 0)
    return set_error(SPD_EINVAL, "grid width %lld must be a multiple of the x-chunk size L=%d", (long long)nx,
                     plan->L);
  const Geometry& g = plan->g;
  if (plan->d == 2 && nz != 1) return set_error(SPD_EINVAL, "2D grid must have nz = 1");
  if (plan->d == 1 && (nz != 1 || ny != 1)) return set_error(SPD_EINVAL, "1D grid must have nz = ny = 1");
  // x = 0 sits 32-B aligned (256-bit epilogue stores); >= 8 elements of left
  // margin for the 16-B groups left of the first chunk window
  const int64_t xoff = roundup(halo > 8 ? halo : 8, 16);
  const int64_t nx_pad = roundup(nx, g.tile_x);
  int64_t need_x = nx_pad + 8 > nx + halo ? nx_pad + 8 : nx + halo;
  const int64_t pitch = roundup(xoff + need_x, 64);
  int64_t rows, planes, yoff, zoff;
  if (plan->d == 1) {
    rows = 2 * halo + 1;
    yoff = halo;
    planes = 1;
    zoff = 0;
  } else {
    const int64_t ny_pad = roundup(ny, g.tile_y);
    yoff = halo;
    rows = halo + (ny_pad + plan->r > ny + halo ? ny_pad + plan->r : ny + halo);
    if (plan->d == 3) {
      const int64_t nz_pad = roundup(nz, g.tile_z);
      zoff = halo;
      planes = halo + (nz_pad + plan->r > nz + halo ? nz_pad + plan->r : nz + halo);
    } else {
      zoff = 0;
      planes = 1;
    }
  }
  out->nz = nz;
  out->ny = ny;
  out->nx = nx;
  out->halo = halo;
  out->dims = plan->d;
  out->pitch = pitch;
  out->plane = rows * pitch;
  out->origin = zoff * out->plane + yoff * pitch + xoff;
  // + slack: the generic-radius row view may read a few elements past the
  // last padded row (boxes are rounded up to 8 elements)
  out->alloc_elems = planes * out->plane + (plan->d == 2 && plan->g.L != 4 && plan->g.L != 8 ? 4096 : 0);
  return SPD_OK;
}

int spd_step_range(const spd_plan* plan, const spd_grid_desc* gd, const void* in, void* out, int64_t lo, int64_t hi,
                   void* stream) {
  using namespace spd;
  int rc = check_desc(plan, gd);
  if (rc) return rc;
  StepParams sp;
  rc = fill_step_params(plan, gd, in, out, lo, hi, 1, sp);
  if (rc) return rc;
  return dispatch(plan, sp, (cudaStream_t)stream);
}

int spd_step_edges(const spd_plan* plan, const spd_grid_desc* gd, const void* in, void* out, void* stream) {
  return spd::step_edges_ex(plan, gd, in, out, nullptr, stream);
}

}  // extern "C"

namespace spd {

static void set_peer_stores(StepParams& sp, const PeerStores* ps) {
  if (!ps) return;
  sp.peer_out[0] = ps->out[0];
  sp.peer_out[1] = ps->out[1];
  sp.peer_row[0] = ps->row[0];
  sp.peer_row[1] = ps->row[1];
  sp.peer_rows = ps->rows;
}

bool plan_peer_stores(const spd_plan* plan) { return plan && !plan->g.cg2; }

int step_edges_ex(const spd_plan* plan, const spd_grid_desc* gd, const void* in, void* out, const PeerStores* ps,
                  void* stream) {
  int rc = check_desc(plan, gd);
  if (rc) return rc;
  if (plan->d == 1) return set_error(SPD_EINVAL, "edge bands are defined for 2D / 3D grids");
  const int64_t extent = plan->d == 3 ? gd->nz : gd->ny;
  StepParams sp;
  rc = fill_step_params(plan, gd, in, out, 0, extent, 1, sp);
  if (rc) return rc;
  int& nb = plan->d == 3 ? sp.tiles_z : sp.tiles_y;
  if (nb > 2) {  // first and last tile band only, one launch
    sp.band_stride = nb - 1;
    nb = 2;
    sp.n_tiles = sp.tiles_x * sp.tiles_y * sp.tiles_z;
    sp.n_bands = 2;
  }
  if (ps && !plan_peer_stores(plan)) return set_error(SPD_EUNSUPPORTED, "no fused peer stores for this geometry");
  set_peer_stores(sp, ps);
  if (ps) sp.publish = 1;  // the publisher warp makes the peer stores (no band counters)
  return dispatch(plan, sp, (cudaStream_t)stream);
}

int step_edge_first_ex(const spd_plan* plan, const spd_grid_desc* gd, const void* in, void* out, int dir,
                       unsigned int* band_done, int publish, const PeerStores* ps, void* stream) {
  int rc = check_desc(plan, gd);
  if (rc) return rc;
  if (plan->d == 1) return set_error(SPD_EINVAL, "band orders are defined for 2D / 3D grids");
  if (plan->g.cg2) return set_error(SPD_EUNSUPPORTED, "edge-first launch not supported in CTA-pair mode");
  if (dir != 0 && dir != 1) return set_error(SPD_EINVAL, "interior direction must be 0 or 1, got %d", dir);
  if (publish && !band_done) return set_error(SPD_EINVAL, "publishing needs band counters");
  if (ps && !plan_peer_stores(plan)) return set_error(SPD_EUNSUPPORTED, "no fused peer stores for this geometry");
  const int64_t extent = plan->d == 3 ? gd->nz : gd->ny;
  StepParams sp;
  rc = fill_step_params(plan, gd, in, out, 0, extent, 1, sp);
  if (rc) return rc;
  sp.edge_order = dir + 1;
  sp.publish = (publish || ps) ? 1 : 0;
  sp.band_done = publish ? band_done : nullptr;
  set_peer_stores(sp, ps);
  return dispatch(plan, sp, (cudaStream_t)stream);
}

}  // namespace spd

extern "C" {

int spd_step_ordered(const spd_plan* plan, const spd_grid_desc* gd, const void* in, void* out, const void* order,
                     int n_pairs, unsigned int* band_done, int publish, void* stream) {
  using namespace spd;
  int rc = check_desc(plan, gd);
  if (rc) return rc;
  if (plan->d == 1) return set_error(SPD_EINVAL, "band orders are defined for 2D / 3D grids");
  if (plan->g.cg2) return set_error(SPD_EUNSUPPORTED, "ordered launch not supported in CTA-pair mode");
  const int64_t extent = plan->d == 3 ? gd->nz : gd->ny;
  StepParams sp;
  rc = fill_step_params(plan, gd, in, out, 0, extent, 1, sp);
  if (rc) return rc;
  if (!order || n_pairs < 1 || n_pairs > sp.n_bands) return set_error(SPD_EINVAL, "bad band order (%d pairs)", n_pairs);
  if (publish && !band_done) return set_error(SPD_EINVAL, "publishing needs band counters");
  sp.use_order = 1;
  sp.order = (const int2*)order;
  sp.total = n_pairs * sp.per_band;
  sp.publish = publish ? 1 : 0;
  sp.band_done = band_done;
  return dispatch(plan, sp, (cudaStream_t)stream);
}

int spd_step_edge_first(const spd_plan* plan, const spd_grid_desc* gd, const void* in, void* out, int dir,
                        unsigned int* band_done, int publish, void* stream) {
  return spd::step_edge_first_ex(plan, gd, in, out, dir, band_done, publish, nullptr, stream);
}

int spd_run(const spd_plan* plan, const spd_grid_desc* gd, void* buf0, void* buf1, int steps, void* stream) {
  static const char* persist_env = getenv("SPD_PERSISTENT");
  const int flags = (persist_env && atoi(persist_env) != 0) ? SPD_RUN_PERSISTENT : 0;
  return spd_run_ex(plan, gd, buf0, buf1, steps, flags, stream);
}

int spd_run_ex(const spd_plan* plan, const spd_grid_desc* gd, void* buf0, void* buf1, int steps, int flags,
               void* stream) {
  using namespace spd;
  int rc = check_desc(plan, gd);
  if (rc) return rc;
  if (steps < 1) return set_error(SPD_EINVAL, "step count must be >= 1, got %d", steps);
  // Default: one launch per step (alternating traversal for L2 reuse).
  // SPD_RUN_PERSISTENT: one cooperative launch for all steps, in sweep /
  // wavefront order (temporal blocking through L2), ordered by per-band
  // completion counters; bit-identical to the per-step launches.
  const bool persistent = (flags & SPD_RUN_PERSISTENT) != 0;
  // SPD_RUN_CHAINED: one launch per step, but launches 1.. of the run wait per
  // tile for the previous step's neighbouring bands (published counters)
  // instead of for the whole previous grid
  const bool chained = !persistent && (flags & SPD_RUN_CHAINED) != 0 && steps > 1 && plan->d >= 2 && !plan->g.cg2;
  const bool forward = (flags & SPD_RUN_FORWARD) != 0;
  const int64_t extent = plan->d == 3 ? gd->nz : (plan->d == 2 ? gd->ny : 1);
  if (!persistent && !chained) {
    // Plain per-step launches: the parameters of even and odd steps (buffer
    // roles and tensor maps) are built once, so the host cost per launch is
    // the launch itself (small grids are otherwise host-bound: encoding two
    // tensor maps per step cost more than a 512^2 step).
    StepParams sp2[2];
    for (int k = 0; k < 2 && k < steps; ++k) {
      rc = fill_step_params(plan, gd, k ? buf1 : buf0, k ? buf0 : buf1, 0, extent, 1, sp2[k]);
      if (rc) return rc;
    }
    for (int done = 0; done < steps; ++done) {
      StepParams& sp = sp2[done & 1];
      sp.reverse = forward ? 0 : (done & 1);
      rc = dispatch(plan, sp, (cudaStream_t)stream);
      if (rc) return rc;
    }
    return SPD_OK;
  }
  unsigned int* chain_counters = nullptr;
  int done = 0;
  while (done < steps) {
    int chunk = persistent ? steps - done : 1;
    StepParams sp;
    rc = fill_step_params(plan, gd, done % 2 ? buf1 : buf0, done % 2 ? buf0 : buf1, 0, extent, chunk, sp);
    if (rc) return rc;
    if (chained) {
      if (!chain_counters) {
        rc = launch_counters(sp.n_bands, (cudaStream_t)stream, &chain_counters);
        if (rc) return rc;
      }
      sp.chain = 1;
      sp.chain_t = done;
      sp.band_done = chain_counters;
      sp.reverse = forward ? 0 : (done & 1);
      rc = dispatch(plan, sp, (cudaStream_t)stream);
      if (rc) {
        cudaFreeAsync(chain_counters, (cudaStream_t)stream);
        return rc;
      }
      done += 1;
      continue;
    }
    if (chunk > 1) {
      // keep the work count in int range
      const int64_t cap = ((int64_t)1 << 30) / ((int64_t)sp.n_bands * sp.per_band);
      if (chunk > cap) {
        chunk = (int)cap;
        sp.steps = chunk;
      }
      if (flags & SPD_RUN_STEPMAJOR) {
        sp.stepmajor = 1;
        sp.total = sp.steps * sp.n_tiles;
      } else {
        rc = wavefront_order(plan, gd, sp);
        if (rc) return rc;
      }
      rc = launch_counters(sp.n_bands, (cudaStream_t)stream, &sp.band_done);
      if (rc) return rc;
    }
    sp.reverse = (persistent || forward) ? 0 : (done & 1);
    rc = dispatch(plan, sp, (cudaStream_t)stream);
    if (sp.band_done) cudaFreeAsync(sp.band_done, (cudaStream_t)stream);
    if (rc) return rc;
    done += chunk;
  }
  if (chain_counters) cudaFreeAsync(chain_counters, (cudaStream_t)stream);
  return SPD_OK;
}

static spd::DenseMap dense_map(const spd_grid_desc* g, int d) {
  spd::DenseMap dm;
  dm.h = g->halo;
  dm.d = d;
  dm.nxd = g->nx + 2 * g->halo;
  dm.nyd = g->ny + 2 * g->halo;
  dm.nzd = d == 3 ? g->nz + 2 * g->halo : 1;
  return dm;
}

int spd_pack_grid(const spd_grid_desc* g, int dtype, const double* dense, void* dev, void* stream) {
  if (!g) return spd::set_error(SPD_EINVAL, "null grid descriptor");
  spd::DenseMap dm = dense_map(g, g->dims);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SPD_DTYPE_F16)
    spd::pack_kernel<__half><<<1184, 256, 0, st>>>(dm, g->pitch, g->plane, g->origin, dense, (__half*)dev);
  else
    spd::pack_kernel<__nv_bfloat16><<<1184, 256, 0, st>>>(dm, g->pitch, g->plane, g->origin, dense,
                                                          (__nv_bfloat16*)dev);
  return spd::cuda_err(cudaGetLastError(), "pack_kernel");
}

int spd_unpack_grid(const spd_grid_desc* g, int dtype, const void* dev, double* dense, void* stream) {
  if (!g) return spd::set_error(SPD_EINVAL, "null grid descriptor");
  spd::DenseMap dm = dense_map(g, g->dims);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SPD_DTYPE_F16)
    spd::unpack_kernel<__half><<<1184, 256, 0, st>>>(dm, g->pitch, g->plane, g->origin, (const __half*)dev, dense);
  else
    spd::unpack_kernel<__nv_bfloat16><<<1184, 256, 0, st>>>(dm, g->pitch, g->plane, g->origin,
                                                            (const __nv_bfloat16*)dev, dense);
  return spd::cuda_err(cudaGetLastError(), "unpack_kernel");
}

static cudaMemcpy3DParms copy_parms(const spd_grid_desc* g, void* dev, void* host, bool h2d) {
  cudaMemcpy3DParms p;
  std::memset(&p, 0, sizeof(p));
  const int64_t h = g->halo;
  const int64_t nxd = g->nx + 2 * h, nyd = g->ny + 2 * h;
  const int64_t nzd = g->dims == 3 ? g->nz + 2 * h : 1;
  const int64_t z0 = g->dims == 3 ? h : 0;
  const int64_t rows_alloc = g->plane / g->pitch;
  char* corner = (char*)dev + 2 * (g->origin - z0 * g->plane - h * g->pitch - h);
  cudaPitchedPtr dp = make_cudaPitchedPtr(corner, (size_t)g->pitch * 2, (size_t)nxd * 2, (size_t)rows_alloc);
  cudaPitchedPtr hp = make_cudaPitchedPtr(host, (size_t)nxd * 2, (size_t)nxd * 2, (size_t)nyd);
  p.extent = make_cudaExtent((size_t)nxd * 2, (size_t)nyd, (size_t)nzd);
  if (h2d) {
    p.srcPtr = hp;
    p.dstPtr = dp;
    p.kind = cudaMemcpyHostToDevice;
  } else {
    p.srcPtr = dp;
    p.dstPtr = hp;
    p.kind = cudaMemcpyDeviceToHost;
  }
  return p;
}

int spd_upload(const spd_grid_desc* g, const void* host_dense, void* dev, void* stream) {
  if (!g || !host_dense || !dev) return spd::set_error(SPD_EINVAL, "null argument");
  cudaMemcpy3DParms p = copy_parms(g, dev, const_cast<void*>(host_dense), true);
  return spd::cuda_err(cudaMemcpy3DAsync(&p, (cudaStream_t)stream), "spd_upload");
}

int spd_download(const spd_grid_desc* g, const void* dev, void* host_dense, void* stream) {
  if (!g || !host_dense || !dev) return spd::set_error(SPD_EINVAL, "null argument");
  cudaMemcpy3DParms p = copy_parms(g, const_cast<void*>(dev), host_dense, false);
  return spd::cuda_err(cudaMemcpy3DAsync(&p, (cudaStream_t)stream), "spd_download");
}

// Dense rows (2D) / planes (3D) [lo, hi) of the grid into the same rows of
// the host dense array (the whole grid's array; only those rows are written):
// a streamed execute downloads each window's finished slab this way.
int spd_download_rows(const spd_grid_desc* g, const void* dev, void* host_dense, int64_t lo, int64_t hi,
                      void* stream) {
  if (!g || !host_dense || !dev) return spd::set_error(SPD_EINVAL, "null argument");
  const int64_t h = g->halo;
  const int64_t nxd = g->nx + 2 * h, nyd = g->ny + 2 * h;
  const int64_t units = g->dims == 3 ? g->nz + 2 * h : nyd;
  if (g->dims == 1) return spd::set_error(SPD_EINVAL, "row ranges are defined for 2D / 3D grids");
  if (lo < 0 || hi > units || lo >= hi) return spd::set_error(SPD_EINVAL, "bad row range [%lld, %lld) of %lld",
                                                              (long long)lo, (long long)hi, (long long)units);
  cudaMemcpy3DParms p = copy_parms(g, const_cast<void*>(dev), host_dense, false);
  if (g->dims == 3) {
    p.srcPtr.ptr = (char*)p.srcPtr.ptr + 2 * lo * g->plane;
    p.dstPtr.ptr = (char*)p.dstPtr.ptr + 2 * lo * nyd * nxd;
    p.extent.depth = (size_t)(hi - lo);
  } else {
    p.srcPtr.ptr = (char*)p.srcPtr.ptr + 2 * lo * g->pitch;
    p.dstPtr.ptr = (char*)p.dstPtr.ptr + 2 * lo * nxd;
    p.extent.height = (size_t)(hi - lo);
    p.dstPtr.ysize = (size_t)(hi - lo);
  }
  return spd::cuda_err(cudaMemcpy3DAsync(&p, (cudaStream_t)stream), "spd_download_rows");
}

// Staged transfers: one linear DMA between the host dense array and a
// device staging buffer of the same (dense) layout at full PCIe rate, plus a
// row-wise repack kernel on the device.  A strided cudaMemcpy3D moves one
// (nx+2h)-element row per DMA descriptor, which for the 3D grids' ~1 KB rows
// runs at a fraction of the link rate.
namespace spd {
__global__ void repack_rows_kernel(DenseMap dm, int64_t pitch, int64_t plane, int64_t origin, const uint16_t* src,
                                   uint16_t* dst, bool to_dev) {
  const int64_t rows = dm.nzd * dm.nyd;
  const int64_t z0 = dm.d == 3 ? dm.h : 0;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t zz = row / dm.nyd, yy = row - zz * dm.nyd;
    const int64_t dense0 = row * dm.nxd;
    const int64_t dev0 = origin + (zz - z0) * plane + (yy - dm.h) * pitch - dm.h;
    if (to_dev)
      for (int64_t x = threadIdx.x; x < dm.nxd; x += blockDim.x) dst[dev0 + x] = src[dense0 + x];
    else
      for (int64_t x = threadIdx.x; x < dm.nxd; x += blockDim.x) dst[dense0 + x] = src[dev0 + x];
  }
}
}  // namespace spd

namespace spd {
// Dirichlet ring of a halo-padded grid (everything of the dense region that
// is not interior) from one device buffer to the other: one warp per stored
// dense row; halo rows / planes are copied whole, interior rows only their
// h left and h right elements.
__global__ void halo_ring_kernel(DenseMap dm, int64_t pitch, int64_t plane, int64_t origin, const uint16_t* src,
                                 uint16_t* dst) {
  const int64_t rows = dm.nzd * dm.nyd;
  const int64_t z0 = dm.d == 3 ? dm.h : 0;
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; row < rows; row += warps) {
    const int64_t zz = row / dm.nyd, yy = row - zz * dm.nyd;
    const int64_t dev0 = origin + (zz - z0) * plane + (yy - dm.h) * pitch - dm.h;
    const bool halo_row = yy < dm.h || yy >= dm.nyd - dm.h || (dm.d == 3 && (zz < dm.h || zz >= dm.nzd - dm.h));
    if (halo_row) {
      for (int64_t x = lane; x < dm.nxd; x += 32) dst[dev0 + x] = src[dev0 + x];
    } else {
      for (int64_t k = lane; k < 2 * dm.h; k += 32) {
        const int64_t x = k < dm.h ? k : dm.nxd - 2 * dm.h + k;
        dst[dev0 + x] = src[dev0 + x];
      }
    }
  }
}
}  // namespace spd

int spd_copy_halo(const spd_grid_desc* g, const void* src, void* dst, void* stream) {
  if (!g || !src || !dst) return spd::set_error(SPD_EINVAL, "null argument");
  if (g->halo < 1) return SPD_OK;
  spd::halo_ring_kernel<<<148 * 4, 256, 0, (cudaStream_t)stream>>>(dense_map(g, g->dims), g->pitch, g->plane,
                                                                   g->origin, (const uint16_t*)src, (uint16_t*)dst);
  return spd::cuda_err(cudaGetLastError(), "halo_ring_kernel");
}

static int64_t dense_elems(const spd_grid_desc* g) {
  const int64_t h = g->halo;
  return (g->dims == 3 ? g->nz + 2 * h : 1) * (g->ny + 2 * h) * (g->nx + 2 * h);
}

int spd_upload_staged(const spd_grid_desc* g, const void* host_dense, void* dev, void* staging, void* stream) {
  if (!g || !host_dense || !dev || !staging) return spd::set_error(SPD_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(staging, host_dense, (size_t)dense_elems(g) * 2, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return spd::cuda_err(e, "spd_upload_staged copy");
  spd::repack_rows_kernel<<<148 * 8, 256, 0, st>>>(dense_map(g, g->dims), g->pitch, g->plane, g->origin,
                                                   (const uint16_t*)staging, (uint16_t*)dev, true);
  return spd::cuda_err(cudaGetLastError(), "repack_rows_kernel");
}

int spd_download_staged(const spd_grid_desc* g, const void* dev, void* host_dense, void* staging, void* stream) {
  if (!g || !host_dense || !dev || !staging) return spd::set_error(SPD_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  spd::repack_rows_kernel<<<148 * 8, 256, 0, st>>>(dense_map(g, g->dims), g->pitch, g->plane, g->origin,
                                                   (const uint16_t*)dev, (uint16_t*)staging, false);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(host_dense, staging, (size_t)dense_elems(g) * 2, cudaMemcpyDeviceToHost, st);
  return spd::cuda_err(e, "spd_download_staged");
}

int spd_naive_apply_f64(int d, int r, const double* coeffs, int64_t nz, int64_t ny, int64_t nx, int halo,
                        const double* in, double* out, double* scratch, int steps, void* stream) {
  using namespace spd;
  if (steps < 1) return set_error(SPD_EINVAL, "step count must be >= 1, got %d", steps);
  if (halo < r) return set_error(SPD_EINVAL, "grid halo %d too small for stencil radius %d", halo, r);
  if (d < 1 || d > 3) return set_error(SPD_EINVAL, "dimensionality must be 1, 2 or 3, got %d", d);
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nzd = d == 3 ? nz + 2 * halo : 1;
  int64_t total = nzd * (ny + 2 * halo) * (nx + 2 * halo);
  // cur/nxt double buffer: both start as copies of the input (halo included)
  cudaError_t e = cudaMemcpyAsync(out, in, total * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(scratch, in, total * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_err(e, "naive copy");
  double* w = nullptr;
  int span = 2 * r + 1, ncoef = d == 1 ? span : (d == 2 ? span * span : span * span * span);
  e = cudaMallocAsync(&w, ncoef * sizeof(double), st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(w, coeffs, ncoef * sizeof(double), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_err(e, "naive coeffs");
  // steps alternate scratch <-> out so the result lands in `out`
  double* bufs[2] = {out, scratch};
  int cur = steps % 2 == 0 ? 0 : 1;  // start so that the last step writes `out`
  int64_t n = nz * ny * nx;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  for (int s = 0; s < steps; ++s) {
    naive_f64_kernel<<<blocks, 256, 0, st>>>(d, r, w, d == 3 ? nz : 1, ny, nx, halo, bufs[cur], bufs[1 - cur]);
    cur = 1 - cur;
  }
  cudaFreeAsync(w, st);
  return cuda_err(cudaGetLastError(), "naive_f64_kernel");
}

// Debug: copy the CTA-0 timeline of the last traced launch (16 x 64 stamps).
extern "C" int spd_debug_trace(unsigned long long* host) {
  if (!spd::g_trace_host) return spd::set_error(SPD_EINVAL, "no trace (set SPD_TRACE and run a step)");
  std::memcpy(host, spd::g_trace_host, 8 * 16 * 64 * 8);  // mapped memory: readable while a kernel runs
  return SPD_OK;
}

int spd_mma_selftest(const uint16_t* a, const uint8_t* e, const uint16_t* b, int n, float* d, void* stream) {
  using namespace spd;
  if (n < 8 || n > 256 || n % 8) return set_error(SPD_EINVAL, "N must be a multiple of 8 in [8, 256], got %d", n);
  mma_selftest_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(a, e, b, n, d);
  return cuda_err(cudaGetLastError(), "mma_selftest_kernel");
}

// Whole stored rows (2D) or planes (3D) including the x halo, so corner
// cells travel with the rows they belong to.
static int64_t halo_unit(const spd_grid_desc* g) { return g->dims == 3 ? g->plane : g->pitch; }
static int64_t halo_unit_start(const spd_grid_desc* g, int64_t i) {
  // element offset of stored row / plane holding interior index i
  int64_t u = halo_unit(g);
  return g->origin - (g->origin % u) + i * u;
}

int spd_halo_pack(const spd_grid_desc* g, const void* buf, int rows, int dir, void* msg, void* stream) {
  using namespace spd;
  if (!g) return set_error(SPD_EINVAL, "null grid descriptor");
  if (g->dims == 1) return set_error(SPD_EINVAL, "1D grids have no slab halo");
  int64_t extent = g->dims == 3 ? g->nz : g->ny;
  if (rows < 1 || rows > extent) return set_error(SPD_EINVAL, "bad halo row count %d", rows);
  int64_t u = halo_unit(g);
  int64_t first = dir == 0 ? 0 : extent - rows;
  halo_copy_kernel<uint16_t><<<592, 256, 0, (cudaStream_t)stream>>>(
      (const uint16_t*)buf, halo_unit_start(g, first), (uint16_t*)msg, 0, rows, u, u, u);
  return cuda_err(cudaGetLastError(), "halo_pack");
}

int spd_halo_unpack(const spd_grid_desc* g, void* buf, int rows, int dir, const void* msg, void* stream) {
  using namespace spd;
  if (!g) return set_error(SPD_EINVAL, "null grid descriptor");
  if (g->dims == 1) return set_error(SPD_EINVAL, "1D grids have no slab halo");
  int64_t extent = g->dims == 3 ? g->nz : g->ny;
  if (rows < 1 || rows > g->halo) return set_error(SPD_EINVAL, "bad halo row count %d", rows);
  int64_t u = halo_unit(g);
  int64_t first = dir == 0 ? -rows : extent;
  halo_copy_kernel<uint16_t><<<592, 256, 0, (cudaStream_t)stream>>>(
      (const uint16_t*)msg, 0, (uint16_t*)buf, halo_unit_start(g, first), rows, u, u, u);
  return cuda_err(cudaGetLastError(), "halo_unpack");
}

}  // extern "C"

/*
 * spider.h — C ABI of the B200-native SPIDER stencil engine (libspider.so).
 *
 * The reference (arxiv/paper_2506_22035, /root/reference/pkg) is a pure-Python
 * package with no FFI; its hot path sits behind the Python functions
 * `transform_stencil` (pipeline.py:128-144), `execute` (pipeline.py:189-262)
 * and `naive_apply` (core.py:151-182).  Every entry point below replaces one
 * reference function or one step of those call stacks; the citation is given
 * per function.  Plain pointers and sizes only: no torch / CUDA-runtime types
 * except `void* stream` (a cudaStream_t, may be NULL for the legacy stream).
 *
 * Conventions
 *   - return 0 on success; SPD_EINVAL (-1) for a configuration error (the
 *     Python mirror raises ValueError with the reference's message
 *     substrings); SPD_ECUDA (-2) for a CUDA failure (RuntimeError);
 *     SPD_EUNSUPPORTED (-3) for a valid stencil the device path does not
 *     implement (ValueError "unsupported").
 *   - spd_last_error() returns a thread-local message for the last failure.
 *   - Device pointers are owned by the caller (torch tensors); a plan owns only
 *     the packed A (compressed kernel) images and E (metadata) words.
 *   - One plan per device, stream-ordered.  Per-step launches (spd_step,
 *     spd_step_range, spd_run without SPD_RUN_PERSISTENT), copies and
 *     naive_apply only read the plan, so several host threads may use one
 *     plan at once on their own streams.  Persistent and ordered launches
 *     (SPD_RUN_PERSISTENT, spd_step_ordered, spd_slab_step) use the plan's
 *     completion counters: at most one of those in flight per plan.
 */
#ifndef SPIDER_H
#define SPIDER_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPD_OK 0
#define SPD_EINVAL (-1)
#define SPD_ECUDA (-2)
#define SPD_EUNSUPPORTED (-3)

#define SPD_PARITY_EVEN 0 /* transform.py:280-288 Parity.EVEN, start 0 */
#define SPD_PARITY_ODD 1  /* Parity.ODD, start 1 */

#define SPD_DTYPE_F16 0
#define SPD_DTYPE_BF16 1

/* ---------------------------------------------------------------------------
 * Library / diagnostics
 */
const char* spd_last_error(void);
/* ABI version; bumps when a signature changes. */
int spd_abi_version(void);

/* ---------------------------------------------------------------------------
 * AOT transform (host, exact twin of transform.py).  Pure functions, no GPU.
 */

/* band_rows: L = 2r+2 (transform.py:37-41). Returns L or SPD_EINVAL. */
int spd_band_rows(int r);

/* input_row_permutation (transform.py:130-139): mapping[2L] (int64). */
int spd_row_permutation(int L, int parity, int64_t* mapping);

/* build_kernel_matrix (transform.py:118-127): row[2r+1] -> out[L x 2L]. */
int spd_build_kernel_matrix(int r, const double* row, double* out);

/* swap_columns (transform.py:142-147): out[rows x 2L] = values[:, perm]. */
int spd_swap_columns(const double* values, int rows, int width, int parity,
                     double* out);

/* check_2to4 (transform.py:163-180).  Writes up to max_viol (row, segment)
 * pairs into viol[2*k]; returns the number of violations (>= 0). */
int spd_check_2to4(const double* values, int rows, int width, int32_t* viol,
                   int max_viol);

/* encode_segment (transform.py:183-205): seg[4] -> vals[2], pos[2]. */
int spd_encode_segment(const double* seg, double* vals, uint8_t* pos);

/* encode (transform.py:208-223): swapped[rows x width] ->
 * values[rows x width/2], metadata[rows x width/4 x 2]. */
int spd_encode(const double* swapped, int rows, int width, double* values,
               uint8_t* metadata);

/* validate_metadata + decode (transform.py:226-246). */
int spd_decode(const double* values, const uint8_t* metadata, int rows,
               int segments, double* out);

/* metadata_to_bytes (transform.py:253-257): one nibble-pair byte per segment. */
int spd_metadata_to_bytes(const uint8_t* metadata, int n_segments,
                          uint8_t* out);

/* transform_stencil for one kernel row (pipeline.py:135-137):
 * row[2r+1] -> values[L x L], metadata[L x L/2 x 2]. */
int spd_transform_row(int r, int parity, const double* row, double* values,
                      uint8_t* metadata);

/* ---------------------------------------------------------------------------
 * Device plan: packs the transformed kernel rows into the tcgen05.mma.sp
 * operand images (A = compressed fp16 values in UMMA K-major smem layout,
 * E = 2-bit ascending-pair metadata in the TMEM lane/bit layout) and fixes the
 * tile geometry.  Replaces pipeline.py:225-234 (operand staging / packing).
 *
 * d in {1,2,3}; coeffs has (2r+1)^d entries in row-major (ρz, ρy, δ) order
 * (core.py:63-89 for d<=2; the 3D extension follows the same convention).
 */
typedef struct spd_plan spd_plan;

int spd_plan_create(int d, int r, int parity, const double* coeffs, int dtype,
                    int device, spd_plan** out);
/* spd_plan_create with geometry flags.  SPD_PLAN_CTA_PAIR (3D only): one
 * M = 256 tcgen05.mma.sp.cta_group::2 per K-block on a cluster of two CTAs
 * (measured slower than the default two-M-tile CTA; kept for experiments).
 * The geometry depends only on (d, r, flags), never on the environment. */
#define SPD_PLAN_CTA_PAIR 1
/* SPD_PLAN_NO_EMBED: keep a radius-2 1D / 2D stencil on the generic L = 6
 * path (by default it runs as radius 3 with a zero ring, on the L = 8 fast
 * path). */
#define SPD_PLAN_NO_EMBED 2
int spd_plan_create_ex(int d, int r, int parity, const double* coeffs, int dtype,
                       int device, int flags, spd_plan** out);
int spd_plan_destroy(spd_plan* plan);

/* Introspection of the packed operands (for the exact-layout tests).
 * info[0..11] = {L, R_in, R_out (per M-tile), S, n_tile, tile_z, tile_y, kchunks,
 * m_tiles, mt_rows, cg2, r_dev} (L and r_dev are the device geometry's: an
 * embedded radius-2 stencil reports L = 8, r_dev = 3).  The tile has m_tiles M = 128 tiles; M-tile t reuses
 * the MMA schedule with the B rows shifted by t * mt_rows.  cg2 = 1: a CTA pair
 * runs one M = 256 MMA per K-block; rank t has its own A/E images (operands
 * then hold 2 * S records, rank-major) for output rows t * R_out .. and stages
 * x-half t of the B columns (n_tile per CTA). */
int spd_plan_info(const spd_plan* plan, int32_t* info);
/* Host copies of the packed images: a_img[S * 128 * 16] (fp16 bits, logical
 * (s, m, k') order, not the smem swizzle), e_words[S * 128], start_rows[S]. */
int spd_plan_operands(const spd_plan* plan, uint16_t* a_img, uint32_t* e_words,
                      int32_t* start_rows);

/* Tile geometry tables: in_off[3*R_in] = (dz, dy, dx) of each input image row
 * relative to the tile origin, out_off[3*R_out*max(m_tiles, 2*cg2)] likewise for output rows. */
int spd_plan_geometry(const spd_plan* plan, int32_t* in_off, int32_t* out_off);
/* MMA row / accumulator TMEM lane of each logical kernel-matrix row
 * m = L*a + i (output row a of the M-tile, position i in the x-chunk);
 * lane[m] for m < r_out*L.  2D / 1D r = 1 plans use the quad-pair order read
 * back by the epilogue's tcgen05.ld.16x256b (16-lane slab j of rows
 * 4j..4j+3 at lane 32 (j % 4) + 16 (j / 4)); 3D and other radii the
 * identity. */
int spd_plan_lane_map(const spd_plan* plan, int32_t* lane);
/* Accumulator lanes each MMA of the tile schedule feeds (half[s], s <
 * mmas_per_tile): 0 all 128 lanes (an M = 128 MMA); 1 / 2 only lanes 0-15 /
 * 16-31 of each 32-lane quadrant (an M = 64 MMA at that TMEM lane offset;
 * every coefficient of MMA s on the other lanes is zero).  All zero in
 * CTA-pair plans. */
int spd_plan_mma_halves(const spd_plan* plan, int32_t* half);

/* ---------------------------------------------------------------------------
 * Device grid layout.  Interior (z, y, x) lives at element
 *   origin + z*plane + y*pitch + x
 * of a zero-initialised buffer of `alloc_elems` elements; the Dirichlet halo
 * of width `halo` surrounds it (core.py:92-127: the halo is never written).
 * Rows are 16-byte aligned at x = 0 and padded to whole tiles.
 */
typedef struct {
  int64_t nz, ny, nx; /* interior extents (nz = 1 for 2D, ny = 1 for 1D) */
  int32_t halo;
  int32_t dims;   /* d of the plan that laid it out (1, 2 or 3) */
  int64_t pitch;  /* elements per stored row */
  int64_t plane;  /* elements per stored plane */
  int64_t origin; /* element offset of interior (0,0,0) */
  int64_t alloc_elems;
} spd_grid_desc;

int spd_grid_layout(const spd_plan* plan, int64_t nz, int64_t ny, int64_t nx,
                    int halo, spd_grid_desc* out);

/* Run `steps` Jacobi steps (pipeline.py:247-261 / core.py:176-181):
 * buf0 holds step 0; the result is in buf[steps % 2].  Both buffers must hold
 * the same halo.  stream = cudaStream_t or NULL. */
int spd_run(const spd_plan* plan, const spd_grid_desc* g, void* buf0,
            void* buf1, int steps, void* stream);

/* spd_run with flags: SPD_RUN_PERSISTENT runs all steps in one cooperative
 * launch ordered by per-band completion counters instead of one launch per
 * step (same results bit for bit). */
#define SPD_RUN_PERSISTENT 1
/* SPD_RUN_CHAINED: one launch per step, but every launch after the first
 * skips the whole-grid dependency on its predecessor: each tile waits only for
 * the previous step's three neighbouring tile bands (per-band completion
 * counters published at gpu scope), so consecutive steps overlap at the
 * launch boundary.  SPD_RUN_FORWARD: traverse every step's tiles in the same
 * direction (default: alternate, for L2 reuse).  Same results bit for bit. */
#define SPD_RUN_CHAINED 2
#define SPD_RUN_FORWARD 4
/* with SPD_RUN_PERSISTENT: plain step-major work order (every step's tiles
 * forward, round-robin over the resident CTAs, no L2 sweeps); a tile still
 * waits for the previous step's three neighbouring bands. */
#define SPD_RUN_STEPMAJOR 8
int spd_run_ex(const spd_plan* plan, const spd_grid_desc* g, void* buf0,
               void* buf1, int steps, int flags, void* stream);

/* One step over the first and the last tile band (2D: tile rows, 3D: tile
 * planes) of the grid in a single launch: a slab's boundary bands, computed
 * before its halo exchange (replaces two spd_step_range calls; the rest is
 * spd_step_range over the interior bands).  2D / 3D only. */
int spd_step_edges(const spd_plan* plan, const spd_grid_desc* g, const void* in,
                   void* out, void* stream);

/* One step over the tile bands listed in `order` (n_pairs int2 entries
 * {0, band}, in execution order).  publish != 0: every finished tile bumps
 * band_done[band] after a system-scope release, so a copy engine waiting on
 * the counters (cuStreamWaitValue32) can move a band's rows while the rest of
 * the step is still running.  2D / 3D only. */
int spd_step_ordered(const spd_plan* plan, const spd_grid_desc* g, const void* in,
                     void* out, const void* order, int n_pairs,
                     unsigned int* band_done, int publish, void* stream);

/* One step with both edge bands (first and last tile row / plane) first, then
 * the interior forward (dir 0) or backward (dir 1); with publish, every edge
 * tile bumps band_done[band] (system scope) when its stores are visible.
 * The slab step's launch (spd_slab_step): the order is computed per tile,
 * so it costs no more than a plain step. */
int spd_step_edge_first(const spd_plan* plan, const spd_grid_desc* g,
                        const void* in, void* out, int dir,
                        unsigned int* band_done, int publish, void* stream);

/* One step restricted to output rows [y_begin, y_end) (2D) or planes
 * [z_begin, z_end) (3D) — used by the slab driver to compute the boundary
 * bands before the halo exchange and the interior after. */
int spd_step_range(const spd_plan* plan, const spd_grid_desc* g,
                   const void* in, void* out, int64_t lo, int64_t hi,
                   void* stream);

/* Dense host array (natural (A+2h) x (B+2h) layout, or (nz+2h)(ny+2h)(nx+2h)
 * for 3D, double) <-> device layout conversion kernels (fp64 <-> fp16/bf16,
 * round-to-nearest).  `src`/`dst` dense pointers are device pointers. */
int spd_pack_grid(const spd_grid_desc* g, int dtype, const double* dense,
                  void* dev, void* stream);
int spd_unpack_grid(const spd_grid_desc* g, int dtype, const void* dev,
                    double* dense, void* stream);

/* Host 16-bit dense array (natural halo-padded layout, element type = the
 * plan's dtype) <-> device layout, via strided DMA (cudaMemcpy2D/3DAsync);
 * the host buffer should be pinned for the copy to be asynchronous. */
int spd_upload(const spd_grid_desc* g, const void* host_dense, void* dev,
               void* stream);
int spd_download(const spd_grid_desc* g, const void* dev, void* host_dense,
                 void* stream);
/* Dense rows (2D) / planes (3D) [lo, hi) (dense coordinates: 0 is the first
 * halo row) of the grid into the same rows of host_dense, the whole grid's
 * dense host array; nothing else is written (streamed execute). */
int spd_download_rows(const spd_grid_desc* g, const void* dev, void* host_dense,
                      int64_t lo, int64_t hi, void* stream);

/* Same transfers through a caller-owned device staging buffer of the dense
 * size ((nz+2h)(ny+2h)(nx+2h) 16-bit elements): one linear DMA plus a
 * device repack kernel, stream-ordered.  Faster than the strided DMA when
 * rows are short (3D grids: ~1 KB rows). */
int spd_upload_staged(const spd_grid_desc* g, const void* host_dense,
                      void* dev, void* staging, void* stream);
int spd_download_staged(const spd_grid_desc* g, const void* dev,
                        void* host_dense, void* staging, void* stream);

/* Copy the Dirichlet ring (halo rows, planes and columns of the dense
 * region; not the interior) of a grid from one device buffer to another of
 * the same layout: after a host upload into one ping-pong buffer, the other
 * needs the same halo before the second step reads it.  16-bit elements. */
int spd_copy_halo(const spd_grid_desc* g, const void* src, void* dst, void* stream);

/* Device fp64 brute-force executor: naive_apply (core.py:151-182) on the
 * natural dense layout, same row-major tap order, separate multiply and add
 * roundings (bit-identical to the numpy oracle).  d in {1,2,3}. */
int spd_naive_apply_f64(int d, int r, const double* coeffs, int64_t nz,
                        int64_t ny, int64_t nx, int halo, const double* in,
                        double* out, double* scratch, int steps, void* stream);

/* Single sparse-MMA self test (tests/test_sptc.py:60-70 analogue on the
 * hardware): D[128 x n] = decode(A,E) * B via one tcgen05.mma.sp.
 * a: 128 x 16 fp16 bits (compressed, logical order); e: 128 x 8 metadata
 * nibbles (ascending pairs, transform.py:253 packing, one byte per segment);
 * b: 32 x n fp16 bits (row-major K x N); d: 128 x n float.  Device pointers. */
int spd_mma_selftest(const uint16_t* a, const uint8_t* e, const uint16_t* b,
                     int n, float* d, void* stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU slab exchange helpers (the driver runs on torch.distributed; these
 * pack/unpack the r boundary rows so one contiguous message per neighbour is
 * sent).  rows = r (or r*T_f).  dir = 0: top boundary, 1: bottom boundary. */
int spd_halo_pack(const spd_grid_desc* g, const void* buf, int rows, int dir,
                  void* msg, void* stream);
int spd_halo_unpack(const spd_grid_desc* g, void* buf, int rows, int dir,
                    const void* msg, void* stream);

/* ---------------------------------------------------------------------------
 * Peer-memory slab exchange (one process per GPU, CUDA IPC).
 * spd_ipc_export: 64-byte IPC handle of the allocation holding ptr and ptr's
 * byte offset in it; spd_ipc_open maps a handle exported by another process
 * (returns the pointer and the mapping base for spd_ipc_close).
 * spd_slab_create: buf0/buf1 this rank's ping-pong grids, my_flags a zeroed
 * device uint32[2] ([0] written by the up neighbour, [1] by the down one);
 * the up_ / dn_ arguments are the neighbours' mapped buffers, layouts and flag
 * words (NULL buffers at the global boundary).
 * spd_slab_step(t): waits (stream memory op) for the neighbours' step t-1
 * halos, computes the two boundary tile bands first (the kernel's publisher
 * warp copies each finished edge tile's r outermost rows into the neighbours'
 * halo rows over peer memory; SPD_SLAB_COPY=1: a copy-engine copy on
 * comm_stream instead), bumps the neighbours' flags on comm_stream once the
 * edge bands are done, and computes the interior bands on compute_stream.
 * The result of step t is in buf[(t+1) % 2]. */
int spd_ipc_export(const void* ptr, void* handle64, int64_t* offset);
int spd_ipc_open(const void* handle64, int64_t offset, void** ptr, void** base);
int spd_ipc_close(void* base);
typedef struct spd_slab spd_slab;
int spd_slab_create(const spd_plan* plan, const spd_grid_desc* g, void* buf0, void* buf1,
                    void* my_flags, void* up_buf0, void* up_buf1,
                    const spd_grid_desc* up_g, void* up_flags, void* dn_buf0,
                    void* dn_buf1, const spd_grid_desc* dn_g, void* dn_flags,
                    spd_slab** out);
int spd_slab_step(spd_slab* s, int t, void* compute_stream, void* comm_stream);
int spd_slab_destroy(spd_slab* s);
/* spd_slab_run: steps t0 .. t0+steps-1 of spd_slab_step in one call. */
int spd_slab_run(spd_slab* s, int t0, int steps, void* compute_stream, void* comm_stream);
/* spd_peer_enable: direct access from `device` to `peer` memory (one process
 * driving several devices: execute(..., DeviceConfig(devices=...)) passes the
 * neighbours' buffers straight to spd_slab_create).  No-op when equal;
 * SPD_EUNSUPPORTED when the pair has no peer path. */
int spd_peer_enable(int device, int peer);

#ifdef __cplusplus
}
#endif

#endif /* SPIDER_H */

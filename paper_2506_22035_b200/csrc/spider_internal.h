// Internal declarations shared by the host AOT code (aot.cpp) and the device
// engine (engine.cu).  Not part of the public ABI (include/spider.h is).
#pragma once

#include <stdint.h>

#include <vector>

#include "../../include/spider.h"

#define SPD_ABI_VERSION 1
#define SPD_MAX_RIN 128
#define SPD_MAX_ROUT 64
#define SPD_MAX_S 32

namespace spd {

int set_error(int code, const char* fmt, ...);
const char* last_error();

int band_rows(int r);
int row_permutation(int L, int parity, int64_t* mapping);
int build_kernel_matrix(int r, const double* row, double* out);
int swap_columns(const double* values, int rows, int width, int parity, double* out);
int check_2to4(const double* values, int rows, int width, int32_t* viol, int max_viol);
int encode_segment(const double* seg, double* vals, uint8_t* pos);
int encode(const double* swapped, int rows, int width, double* values, uint8_t* metadata);
int decode(const double* values, const uint8_t* metadata, int rows, int segments, double* out);
int metadata_to_bytes(const uint8_t* metadata, int n_segments, uint8_t* out);
int transform_row(int r, int parity, const double* row, double* values, uint8_t* metadata);

uint16_t f64_to_f16_bits(double x);
uint16_t f64_to_bf16_bits(double x);

// Tile geometry of the sm_100a stencil kernel (see aot.cpp build_geometry).
// Passed to the kernel by value.
struct Geometry {
  int d, r, L;
  int kc;            // 16-byte K-chunks per input-row window (2L/8 rounded up to 1, 2 or 4)
  int rows_per_mma;  // input rows per K=32 MMA (4/kc)
  int r_out;         // output rows per M-tile (128/L)
  int m_tiles;       // M = 128 tiles per tile (3D: 2, sharing one input block)
  int mt_rows;       // input-row offset between consecutive M-tiles
  int cg2;           // 3D CTA-pair mode: one M = 256 tcgen05.mma.sp.cta_group::2 per K-block;
                     // CTA rank t holds output rows t*r_out.. (its own A/E images) and x-half t of B
  int lane_map;      // MMA row (TMEM lane) of output row a, chunk position i: 0 linear (m = L*a + i);
                     // 1 quad pair (L = 4, one M-tile): m = 16*(a/4) + 2*(a%4) + (i>>1) + 8*(i&1), read back
                     // with tcgen05.ld.16x256b (lanes m and m+8 land in one thread: phases i, i+1);
                     // 2 z-split (3D, two M-tiles): m = 32*(y/2) + 16*(z/2) + 4*(2*(z%2) + y%2) + i
                     // 3 half split (L = 8): m = 32*((a%8)/2) + 16*(a/8) + 8*(a%2) + i
  int r_in;          // input image rows per tile
  int s;             // MMAs per tile
  int n_tile;        // x-chunks per tile (MMA N)
  int tile_z, tile_y, tile_x;  // tile extent in output points (x in points)
  int b_sbo;         // bytes between 8-chunk core-matrix groups of the B image
  int start_row[SPD_MAX_S];
  int first_owned[SPD_MAX_S];
  int mma_half[SPD_MAX_S];  // accumulator lanes MMA s feeds: 0 all 128 (M = 128); 1 / 2 only lanes
                            // 32q + [0, 16) / 32q + [16, 32) of each quadrant q: issued as an M = 64
                            // MMA at TMEM lane offset 0 / 16 (D, A and E alike; tools/umma_m64_probe.cu)
  int in_dz[SPD_MAX_RIN], in_dy[SPD_MAX_RIN], in_dx[SPD_MAX_RIN];
  int out_dz[SPD_MAX_ROUT], out_dy[SPD_MAX_ROUT], out_dx[SPD_MAX_ROUT];
};

// Fused peer stores of a slab step (peer.cu): output rows (2D) / planes (3D)
// u < rows also go to out[0] at u + row[0], rows u >= extent - rows to
// out[1] at u + row[1] (the neighbours' halo rows, same layout).
struct PeerStores {
  void* out[2];
  int64_t row[2];
  int rows;
};
bool plan_peer_stores(const spd_plan* plan);  // the plan's epilogue supports them
int step_edge_first_ex(const spd_plan* plan, const spd_grid_desc* g, const void* in, void* out, int dir,
                       unsigned int* band_done, int publish, const PeerStores* ps, void* stream);
int step_edges_ex(const spd_plan* plan, const spd_grid_desc* g, const void* in, void* out, const PeerStores* ps,
                  void* stream);

int build_geometry(int d, int r, int flags, Geometry* g);
int lane_of(const Geometry& g, int a, int i);
int pack_operands(const Geometry& g, int n_rows, const double* row_values,
                  const uint8_t* row_meta, int dtype, std::vector<uint16_t>& a_img,
                  std::vector<uint32_t>& e_words);

}  // namespace spd

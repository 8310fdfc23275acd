// Host-side AOT transform (bit-exact twin of the reference transform.py) and
// the device operand packer that lays the compressed kernel rows out for
// tcgen05.mma.sp.  No CUDA code in this file: it is pure C++ so the CPU test
// tier can exercise it through the C ABI.
//
// Reference citations are /root/reference/pkg/src/sparsestencil/<file>:<line>.
#include "spider_internal.h"

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace spd {

static thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

const char* last_error() { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// transform.py twins

// band_rows, transform.py:37-41
int band_rows(int r) {
  if (r < 1) return set_error(SPD_EINVAL, "radius must be >= 1, got %d", r);
  return 2 * r + 2;
}

// input_row_permutation, transform.py:130-139
int row_permutation(int L, int parity, int64_t* mapping) {
  if (L % 2 != 0) return set_error(SPD_EINVAL, "L must be even, got %d", L);
  if (parity != SPD_PARITY_EVEN && parity != SPD_PARITY_ODD)
    return set_error(SPD_EINVAL, "bad parity code %d", parity);
  for (int j = 0; j < 2 * L; ++j) mapping[j] = j;
  for (int j = parity; j < L; j += 2) {
    mapping[j] = j + L;
    mapping[j + L] = j;
  }
  return SPD_OK;
}

// build_kernel_matrix, transform.py:118-127
int build_kernel_matrix(int r, const double* row, double* out) {
  int L = band_rows(r);
  if (L < 0) return L;
  std::memset(out, 0, sizeof(double) * L * 2 * L);
  for (int i = 0; i < L; ++i)
    for (int t = 0; t < 2 * r + 1; ++t) out[i * 2 * L + i + t] = row[t];
  return SPD_OK;
}

// swap_columns, transform.py:142-147
int swap_columns(const double* values, int rows, int width, int parity, double* out) {
  if (width % 2 != 0) return set_error(SPD_EINVAL, "width %d must be even", width);
  int L = width / 2;
  std::vector<int64_t> perm(2 * L);
  int rc = row_permutation(L, parity, perm.data());
  if (rc) return rc;
  for (int i = 0; i < rows; ++i)
    for (int q = 0; q < width; ++q) out[i * width + q] = values[i * width + perm[q]];
  return SPD_OK;
}

// check_2to4, transform.py:163-180
int check_2to4(const double* values, int rows, int width, int32_t* viol, int max_viol) {
  if (width % 4 != 0) return set_error(SPD_EINVAL, "width %d not divisible by 4", width);
  int n = 0;
  for (int i = 0; i < rows; ++i)
    for (int s = 0; s < width / 4; ++s) {
      int cnt = 0;
      for (int t = 0; t < 4; ++t) cnt += values[i * width + 4 * s + t] != 0.0;
      if (cnt > 2) {
        if (viol && n < max_viol) {
          viol[2 * n] = i;
          viol[2 * n + 1] = s;
        }
        ++n;
      }
    }
  return n;
}

// encode_segment, transform.py:183-205: placeholder after the value except at
// position 3, where it precedes; an empty segment is (0, 0) at (0, 1).
int encode_segment(const double* seg, double* vals, uint8_t* pos) {
  int nz[4], cnt = 0;
  for (int t = 0; t < 4; ++t)
    if (seg[t] != 0.0) nz[cnt++] = t;
  if (cnt > 2)
    return set_error(SPD_EINVAL, "segment [%g, %g, %g, %g] has %d nonzeros; 2:4 violated",
                     seg[0], seg[1], seg[2], seg[3], cnt);
  if (cnt == 2) {
    vals[0] = seg[nz[0]];
    vals[1] = seg[nz[1]];
    pos[0] = (uint8_t)nz[0];
    pos[1] = (uint8_t)nz[1];
  } else if (cnt == 1) {
    int p = nz[0];
    if (p < 3) {
      vals[0] = seg[p];
      vals[1] = 0.0;
      pos[0] = (uint8_t)p;
      pos[1] = (uint8_t)(p + 1);
    } else {
      vals[0] = 0.0;
      vals[1] = seg[3];
      pos[0] = 2;
      pos[1] = 3;
    }
  } else {
    vals[0] = vals[1] = 0.0;
    pos[0] = 0;
    pos[1] = 1;
  }
  return SPD_OK;
}

// encode, transform.py:208-223 (row-major loops, segment-major output)
int encode(const double* swapped, int rows, int width, double* values, uint8_t* metadata) {
  if (width % 4 != 0) return set_error(SPD_EINVAL, "width %d not divisible by 4", width);
  int segs = width / 4;
  for (int i = 0; i < rows; ++i)
    for (int s = 0; s < segs; ++s) {
      int rc = encode_segment(swapped + i * width + 4 * s, values + i * 2 * segs + 2 * s,
                              metadata + (i * segs + s) * 2);
      if (rc) return rc;
    }
  return SPD_OK;
}

// validate_metadata, transform.py:226-233
static int validate_metadata(const uint8_t* meta, int n_pairs) {
  for (int k = 0; k < n_pairs; ++k) {
    if (meta[2 * k] > 3 || meta[2 * k + 1] > 3)
      return set_error(SPD_EINVAL, "metadata positions must lie in {0,1,2,3}");
    if (meta[2 * k] >= meta[2 * k + 1])
      return set_error(SPD_EINVAL, "metadata position pairs must be strictly ascending");
  }
  return SPD_OK;
}

// decode, transform.py:236-246
int decode(const double* values, const uint8_t* metadata, int rows, int segments, double* out) {
  int rc = validate_metadata(metadata, rows * segments);
  if (rc) return rc;
  int width = 4 * segments;
  std::memset(out, 0, sizeof(double) * rows * width);
  for (int i = 0; i < rows; ++i)
    for (int s = 0; s < segments; ++s)
      for (int t = 0; t < 2; ++t)
        out[i * width + 4 * s + metadata[(i * segments + s) * 2 + t]] =
            values[i * 2 * segments + 2 * s + t];
  return SPD_OK;
}

// metadata_to_bytes, transform.py:253-257
int metadata_to_bytes(const uint8_t* metadata, int n_segments, uint8_t* out) {
  for (int k = 0; k < n_segments; ++k)
    out[k] = (uint8_t)((metadata[2 * k] & 3) | ((metadata[2 * k + 1] & 3) << 2));
  return SPD_OK;
}

// One kernel row of transform_stencil (pipeline.py:135-137):
// encode(strided_swap(build_kernel_matrix(row, r), parity)).
int transform_row(int r, int parity, const double* row, double* values, uint8_t* metadata) {
  int L = band_rows(r);
  if (L < 0) return L;
  std::vector<double> band(L * 2 * L), sw(L * 2 * L);
  int rc = build_kernel_matrix(r, row, band.data());
  if (rc) return rc;
  rc = swap_columns(band.data(), L, 2 * L, parity, sw.data());
  if (rc) return rc;
  return encode(sw.data(), L, 2 * L, values, metadata);
}

// ---------------------------------------------------------------------------
// Tile geometry + operand packing for the sm_100a kernel.
//
// The MMA is D[m, n] += A[m, k] * B[k, n] with
//   n  = x-chunk of L output points (N dimension, n_tile chunks per tile),
//   m  = L*alpha + i: output row alpha of the tile, position i in the chunk,
//   k  = (input image row c within the MMA, window slot q): each input row
//        contributes one 2L-slot window (KC = 2L/8 K-chunks of 8 slots).
// A K=32 MMA therefore spans 32/(2L) input rows; the MMAs of a tile walk the
// input image rows from top to bottom (start_rows[]) so every input row is
// consumed by exactly one MMA, and partial sums over kernel rows accumulate in
// the same TMEM accumulator (the reference accumulates kernel rows in
// ascending order, pipeline.py:249-253; here the order is fixed by the MMA
// sequence and fp32 accumulation).
static void assign_mma_halves(Geometry* g);

int build_geometry(int d, int r, int flags, Geometry* g) {
  std::memset(g, 0, sizeof(*g));
  int L = band_rows(r);
  if (L < 0) return L;
  if (L > 16)
    return set_error(SPD_EUNSUPPORTED,
                     "unsupported radius %d for the device path (supported: 1 <= r <= 7)", r);
  if (d == 3 && L != 4)
    return set_error(SPD_EUNSUPPORTED, "unsupported radius %d for 3D on the device (r = 1 only)", r);
  g->d = d;
  g->r = r;
  g->L = L;
  // window of 2L slots in 16-byte K-chunks; a K=32 MMA holds 4 chunks, so the
  // per-row chunk count is padded to a divisor of 4 (pad slots carry zero
  // coefficients with (0,1) metadata)
  {
    const int need = (2 * L + 7) / 8;
    g->kc = need <= 1 ? 1 : (need <= 2 ? 2 : 4);
  }
  g->rows_per_mma = 4 / g->kc;
  g->r_out = 128 / L;
  g->m_tiles = 1;
  g->mt_rows = 0;
  int rin = 0;
  if (d == 2) {
    // (Stacking M-tiles to share the input block, as 3D does, was measured
    // slower for r = 3: 4 M-tiles x N = 32 113 -> 142 us, 2 x 32 -> 119 us.)
    g->tile_z = 1;
    g->tile_y = g->r_out * g->m_tiles;
    g->n_tile = (L == 4) ? 128 : 64;
    g->tile_x = g->n_tile * L;
    for (int a = 0; a < g->r_out * g->m_tiles; ++a) {
      g->out_dz[a] = 0;
      g->out_dy[a] = a;
      g->out_dx[a] = 0;
    }
    for (int b = 0; b < g->tile_y + 2 * r; ++b) {
      g->in_dz[rin] = 0;
      g->in_dy[rin] = b - r;
      g->in_dx[rin] = 0;
      ++rin;
    }
  } else if (d == 3) {
    // Two M = 128 tiles (4 z-planes x 8 rows each) share one 8z x 8y input
    // block: 100 input rows for 64 output rows (1.56x) instead of 60 per 32
    // (1.875x).  M-tile 1 uses M-tile 0's MMA schedule and A/E images with
    // the B rows shifted by 4 planes (40 rows).  N = 32 chunks keeps two B
    // stages and four natural-row stages in shared memory.
    g->m_tiles = 2;
    g->tile_z = 8;
    g->tile_y = 8;
    g->n_tile = 32;
    g->tile_x = g->n_tile * L;
    g->mt_rows = (g->tile_z / g->m_tiles) * (g->tile_y + 2 * r);
    // CTA-pair mode (SPD_PLAN_CTA_PAIR): the same 8z x 8y block, but one
    // cta_group::2 MMA (M = 256: rank t's TMEM holds M-tile t) per K-block of
    // all 100 input rows, each CTA staging the B columns of its x-half
    // (n_tile = 32 chunks per CTA, 64 per pair).
    if (flags & SPD_PLAN_CTA_PAIR) {
      g->cg2 = 1;
      g->m_tiles = 1;
      g->tile_x = 2 * g->n_tile * L;
    }
    for (int a = 0; a < g->r_out * 2; ++a) {  // two M-tiles (or the two CTAs of a pair)
      g->out_dz[a] = a / g->tile_y;
      g->out_dy[a] = a % g->tile_y;
      g->out_dx[a] = 0;
    }
    for (int iz = 0; iz < g->tile_z + 2 * r; ++iz)
      for (int iy = 0; iy < g->tile_y + 2 * r; ++iy) {
        g->in_dz[rin] = iz - r;
        g->in_dy[rin] = iy - r;
        g->in_dx[rin] = 0;
        ++rin;
      }
  } else if (d == 1) {
    // 1D: the line is cut into r_out consecutive segments of seg = n_tile*L
    // points; each segment is one "row" of the tile (windows cross segment
    // boundaries through contiguous memory).
    g->tile_z = 1;
    g->tile_y = 1;
    g->n_tile = (L == 4) ? 128 : 64;
    int seg = g->n_tile * L;
    g->tile_x = seg * g->r_out;
    for (int a = 0; a < g->r_out; ++a) {
      g->out_dz[a] = 0;
      g->out_dy[a] = 0;
      g->out_dx[a] = a * seg;
      g->in_dz[rin] = 0;
      g->in_dy[rin] = 0;
      g->in_dx[rin] = a * seg;
      ++rin;
    }
  } else {
    return set_error(SPD_EINVAL, "dimensionality must be 1, 2 or 3, got %d", d);
  }
  g->r_in = rin;
  // L = 4, one M-tile (2D, 1D): quad-pair lane map (see Geometry::lane_map
  // and the epilogue).  The 3D two-M-tile geometry keeps the linear map: its
  // quad-pair epilogue measured 123.8 -> 141.9 us per B27 step, while 2D r = 1
  // gains ~1 % (B9 79.3 -> 78.4 us; profiles/r02_epilogue.txt).
  // (The same layout for L = 8 -- 16x256b reads plus a two-level butterfly
  // over lanes ^4, ^8 -- measured B49 97.4 -> 108.0 us: not used.)
  g->lane_map = (L == 4 && g->m_tiles == 1 && !g->cg2) ? 1 : 0;
  // 3D two-M-tile geometry: z-split lane map (lane_of), so the K-blocks of
  // the first / last two input planes are M = 64 MMAs (9 of 15 instead of 5
  // with the linear map's y split).
  if (d == 3 && g->m_tiles == 2 && !g->cg2) g->lane_map = 2;
  // L = 8 (r = 3 and embedded r = 2; 2D and 1D): rows 0-7 on lanes 0-15 and
  // rows 8-15 on lanes 16-31 of the quadrants (B49: 7 of 11 MMAs at M = 64)
  if (L == 8 && d != 3) g->lane_map = 3;
  // B image: core matrices (8 chunks x 16 B) of consecutive window K-chunks
  // are adjacent (LBO = 128 B); 8-chunk groups are SBO apart.  UMMA needs the
  // core matrices 128-B aligned, so SBO is a multiple of 128.
  g->b_sbo = rin * g->kc * 128;
  if (rin > SPD_MAX_RIN) return set_error(SPD_EINVAL, "tile needs %d input rows (max %d)", rin, SPD_MAX_RIN);
  // MMA start rows: consecutive groups of rows_per_mma; a ragged tail reuses
  // an overlapping window whose leading rows carry zero coefficients.
  int rpm = g->rows_per_mma;
  int s = 0;
  const int rin_mma = g->cg2 ? rin : rin - (g->m_tiles - 1) * g->mt_rows;  // M-tile 0's input rows (pair: all)
  for (int b0 = 0; b0 < rin_mma; b0 += rpm) {
    int start = b0 + rpm <= rin_mma ? b0 : rin_mma - rpm;
    g->start_row[s] = start;
    g->first_owned[s] = b0;  // rows [first_owned, start+rpm) belong to MMA s
    ++s;
  }
  g->s = s;
  if (s > SPD_MAX_S) return set_error(SPD_EINVAL, "tile needs %d MMAs (max %d)", s, SPD_MAX_S);
#ifndef SPD_NO_M64  // comparison builds (tools/build_variant.sh -DSPD_NO_M64): every MMA at M = 128
  if (!g->cg2) assign_mma_halves(g);
#endif
  return SPD_OK;
}

// MMA row (= accumulator TMEM lane) holding output row a, chunk position i.
int lane_of(const Geometry& g, int a, int i) {
  if (g.lane_map == 1) {
    // 16-lane slabs of 16/L rows; lanes m, m+8 hold positions i, i+1.  Slab
    // j sits at lane 32 (j % 4) + 16 (j / 4): the top half of the tile's rows
    // on lanes 0-15 of the four quadrants, the bottom half on lanes 16-31, so
    // a K-block feeding only one half of the rows is an M = 64 MMA
    // (assign_mma_halves).
    const int rows16 = 16 / g.L;
    const int j = a / rows16;
    return 32 * (j % 4) + 16 * (j / 4) + (g.L / 2) * (a % rows16) + (i >> 1) + 8 * (i & 1);
  }
  if (g.lane_map == 2) {
    // 3D M-tile of 4 z-planes x 8 rows (a = 8 z + y), L = 4: quadrant y / 2,
    // z-planes 0-1 on lanes 0-15 and 2-3 on lanes 16-31 of the quadrant,
    // 4-lane group 2 (z % 2) + y % 2 inside the half (the epilogue inverts it)
    const int z = a / 8, y = a % 8;
    return 32 * (y / 2) + 16 * (z / 2) + 4 * (2 * (z % 2) + (y % 2)) + i;
  }
  if (g.lane_map == 3)  // L = 8: quadrant (a % 8) / 2, half a / 8, 8-lane group a % 2
    return 32 * ((a % 8) / 2) + 16 * (a / 8) + 8 * (a % 2) + i;
  return g.L * a + i;
}

// Kernel-row index for an (input row, output row) pair, or -1 if the input row
// does not feed that output row.  Kernel rows are ordered like
// StencilKernel.row_offsets (core.py:46-50): rho ascending; for 3D (rho_z,
// rho_y) row-major.
static int kernel_row_index(const Geometry& g, int b, int a) {
  int r = g.r;
  if (g.in_dx[b] != g.out_dx[a]) return -1;
  int rz = g.in_dz[b] - g.out_dz[a];
  int ry = g.in_dy[b] - g.out_dy[a];
  if (g.d == 1) return (rz == 0 && ry == 0) ? 0 : -1;
  if (rz < -r || rz > r || ry < -r || ry > r) return -1;
  if (g.d == 2) return rz == 0 ? ry + r : -1;
  return (rz + r) * (2 * r + 1) + (ry + r);
}

// Which half of the accumulator lanes each MMA feeds (Geometry::mma_half).
// An M = 64 tcgen05.mma.sp at TMEM lane offset h (D, A and E addresses)
// computes the rows on lanes 32q + h + [0, 16) of every quadrant q from the
// same A/E images as the M = 128 form (tools/umma_m64_probe.cu), so an MMA
// whose input rows feed only output rows on one half can skip the other half:
// the skipped rows have zero coefficients for those input rows.  MMA 0 stays
// M = 128: it initialises every accumulator lane (accumulate = 0).
static void assign_mma_halves(Geometry* g) {
  const int ranks_rows = g->r_out;  // M-tile 0; the other M-tiles reuse its schedule and images
  for (int s = 0; s < g->s; ++s) {
    int used[2] = {0, 0};
    for (int c = 0; c < g->rows_per_mma; ++c) {
      const int b = g->start_row[s] + c;
      if (b < g->first_owned[s]) continue;
      for (int a = 0; a < ranks_rows; ++a) {
        if (kernel_row_index(*g, b, a) < 0) continue;
        for (int i = 0; i < g->L; ++i) used[(lane_of(*g, a, i) % 32) >= 16] = 1;
      }
    }
    g->mma_half[s] = (s == 0 || (used[0] && used[1])) ? 0 : (used[0] ? 1 : (used[1] ? 2 : 0));
  }
}

// Packs A (compressed values, logical (s, m, k') order, fp16 or bf16 bits) and
// E (one 32-bit TMEM word per (s, lane)).  E layout (verified on B200 by
// tools/umma_sp_probe.cu, variant 1; matches CUTLASS tmem_e_frg for 16-bit A):
//   row m = m0 + 8*m1 + 16*m2, K=32 segment seg = 4*k1 + c (c in 0..3)
//   -> TMEM lane m0 + 8*k1 + 16*m2, bits 16*m1 + 4*c, nibble idx0 | idx1 << 2.
int pack_operands(const Geometry& g, int n_rows, const double* row_values,
                  const uint8_t* row_meta, int dtype, std::vector<uint16_t>& a_img,
                  std::vector<uint32_t>& e_words) {
  const int L = g.L;
  const int segs_per_row = L / 2;  // 4-wide segments in one 2L window
  const int ranks = g.cg2 ? 2 : 1;  // CTA pair: rank t's images map output rows t*r_out..
  a_img.assign((size_t)ranks * g.s * 128 * 16, 0);
  e_words.assign((size_t)ranks * g.s * 128, 0);
  std::vector<uint8_t> nib((size_t)128 * 8);
  for (int rk = 0; rk < ranks; ++rk)
  for (int s = 0; s < g.s; ++s) {
    const size_t si = (size_t)rk * g.s + s;
    std::fill(nib.begin(), nib.end(), (uint8_t)(0 | (1 << 2)));  // empty segment: (0, 1)
    for (int c = 0; c < g.rows_per_mma; ++c) {
      int b = g.start_row[s] + c;
      if (b < g.first_owned[s]) continue;  // owned by the previous MMA
      for (int a = 0; a < g.r_out; ++a) {
        int kr = kernel_row_index(g, b, a + rk * g.r_out);
        if (kr < 0) continue;
        if (kr >= n_rows) return set_error(SPD_EINVAL, "kernel row %d out of range", kr);
        const double* vals = row_values + (size_t)kr * L * L;
        const uint8_t* meta = row_meta + (size_t)kr * L * segs_per_row * 2;
        for (int i = 0; i < L; ++i) {
          int m = lane_of(g, a, i);
          for (int sg = 0; sg < segs_per_row; ++sg) {
            int kseg = c * 2 * g.kc + sg;  // segment within K=32 (rows padded to kc chunks)
            for (int t = 0; t < 2; ++t) {
              double v = vals[i * L + 2 * sg + t];
              a_img[(si * 128 + m) * 16 + 2 * kseg + t] =
                  dtype == SPD_DTYPE_BF16 ? f64_to_bf16_bits(v) : f64_to_f16_bits(v);
            }
            const uint8_t* p = meta + (i * segs_per_row + sg) * 2;
            nib[m * 8 + kseg] = (uint8_t)(p[0] | (p[1] << 2));
          }
        }
      }
    }
    for (int lane = 0; lane < 128; ++lane) {
      int m0 = lane % 8, k1 = (lane / 8) % 2, m2 = lane / 16;
      uint32_t w = 0;
      for (int m1 = 0; m1 < 2; ++m1)
        for (int c4 = 0; c4 < 4; ++c4) {
          int m = m0 + 8 * m1 + 16 * m2;
          w |= (uint32_t)nib[m * 8 + 4 * k1 + c4] << (16 * m1 + 4 * c4);
        }
      e_words[si * 128 + lane] = w;
    }
  }
  return SPD_OK;
}

// Round-to-nearest-even double -> binary16 / bfloat16 bit patterns (host).
uint16_t f64_to_f16_bits(double x) {
  // Go through float first is not exact (double rounding); do it directly.
  uint64_t u;
  std::memcpy(&u, &x, 8);
  uint16_t sign = (uint16_t)((u >> 48) & 0x8000);
  uint64_t mag = u & 0x7FFFFFFFFFFFFFFFull;
  if (mag >= 0x7FF0000000000000ull) {  // inf / nan
    if (mag > 0x7FF0000000000000ull) return sign | 0x7E00;
    return sign | 0x7C00;
  }
  int exp = (int)(mag >> 52) - 1023;
  uint64_t mant = mag & 0xFFFFFFFFFFFFFull;
  if (exp > 15) return sign | 0x7C00;  // overflow (rounding handled below)
  if (exp >= -14) {
    // normal half: 10 mantissa bits, drop 42
    uint64_t full = mant | (1ull << 52);
    uint64_t keep = full >> 42;  // 11 bits incl implicit
    uint64_t rem = full & ((1ull << 42) - 1);
    uint64_t half = 1ull << 41;
    if (rem > half || (rem == half && (keep & 1))) ++keep;
    int e = exp + 15;
    if (keep >> 11) {  // mantissa overflow
      keep >>= 1;
      ++e;
    }
    if (e >= 31) return sign | 0x7C00;
    return (uint16_t)(sign | (e << 10) | (keep & 0x3FF));
  }
  // subnormal: value = m * 2^-24
  if (exp < -25) return sign;  // rounds to zero (|x| < 2^-25)
  uint64_t full = mant | (1ull << 52);
  int shift = 52 - (exp + 24);  // bits to drop so that unit = 2^-24
  uint64_t keep = full >> shift;
  uint64_t rem = full & ((1ull << shift) - 1);
  uint64_t half = 1ull << (shift - 1);
  if (rem > half || (rem == half && (keep & 1))) ++keep;
  return (uint16_t)(sign | keep);  // keep may carry into the exponent: correct
}

uint16_t f64_to_bf16_bits(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  uint16_t sign = (uint16_t)((u >> 48) & 0x8000);
  uint64_t mag = u & 0x7FFFFFFFFFFFFFFFull;
  if (mag >= 0x7FF0000000000000ull) return mag > 0x7FF0000000000000ull ? (sign | 0x7FC0) : (sign | 0x7F80);
  int exp = (int)(mag >> 52) - 1023;
  uint64_t mant = mag & 0xFFFFFFFFFFFFFull;
  if (exp >= -126) {
    uint64_t full = mant | (1ull << 52);
    uint64_t keep = full >> 45;  // 8 bits incl implicit
    uint64_t rem = full & ((1ull << 45) - 1);
    uint64_t half = 1ull << 44;
    if (rem > half || (rem == half && (keep & 1))) ++keep;
    int e = exp + 127;
    if (keep >> 8) {
      keep >>= 1;
      ++e;
    }
    if (e >= 255) return sign | 0x7F80;
    return (uint16_t)(sign | (e << 7) | (keep & 0x7F));
  }
  if (exp < -134) return sign;
  uint64_t full = mant | (1ull << 52);
  int shift = 52 - (exp + 133);
  uint64_t keep = full >> shift;
  uint64_t rem = full & ((1ull << shift) - 1);
  uint64_t half = 1ull << (shift - 1);
  if (rem > half || (rem == half && (keep & 1))) ++keep;
  return (uint16_t)(sign | keep);
}

}  // namespace spd

// ---------------------------------------------------------------------------
// C ABI (host part)
extern "C" {

const char* spd_last_error(void) { return spd::last_error(); }
int spd_abi_version(void) { return SPD_ABI_VERSION; }
int spd_band_rows(int r) { return spd::band_rows(r); }
int spd_row_permutation(int L, int parity, int64_t* mapping) {
  return spd::row_permutation(L, parity, mapping);
}
int spd_build_kernel_matrix(int r, const double* row, double* out) {
  return spd::build_kernel_matrix(r, row, out);
}
int spd_swap_columns(const double* values, int rows, int width, int parity, double* out) {
  return spd::swap_columns(values, rows, width, parity, out);
}
int spd_check_2to4(const double* values, int rows, int width, int32_t* viol, int max_viol) {
  return spd::check_2to4(values, rows, width, viol, max_viol);
}
int spd_encode_segment(const double* seg, double* vals, uint8_t* pos) {
  return spd::encode_segment(seg, vals, pos);
}
int spd_encode(const double* swapped, int rows, int width, double* values, uint8_t* metadata) {
  return spd::encode(swapped, rows, width, values, metadata);
}
int spd_decode(const double* values, const uint8_t* metadata, int rows, int segments, double* out) {
  return spd::decode(values, metadata, rows, segments, out);
}
int spd_metadata_to_bytes(const uint8_t* metadata, int n_segments, uint8_t* out) {
  return spd::metadata_to_bytes(metadata, n_segments, out);
}
int spd_transform_row(int r, int parity, const double* row, double* values, uint8_t* metadata) {
  return spd::transform_row(r, parity, row, values, metadata);
}

}  // extern "C"

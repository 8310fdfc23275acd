// Memory-system micro-benchmark for the B9 step's access pattern (one GPU):
// how fast can 148 persistent CTAs (a) TMA-load the halo-padded input blocks
// of the 6400 tiles of a 10240^2 fp16 grid, (b) store the 32 x 512 output
// tiles with 256-bit full-line stores, (c) both at once -- with no compute.
// Bounds the step kernel's achievable DRAM rate (tools/tma_bw.cu; not part of
// the library).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tma_bw tools/tma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE%=;\nbra WAIT%=;\nDONE%=:\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, uint32_t s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(s), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t s, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(s), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void stg_v8(void* p, uint32_t a) {
  asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
}

struct P {
  CUtensorMap map;
  CUtensorMap omap;  // output tensor map (TMA stores), box 256 x 32
  int nbox, boxw, box_rows, stage_bytes, nnat, box_slot;
  int tiles_x, n_tiles, tile_x, tile_y;
  int64_t pitch, origin;
  uint16_t* out;
  int mode;  // 1 load, 2 store, 3 both; +4: stores by TMA (1D bulk rows), +8: stores by tensor TMA
  int ostage;  // smem bytes of the output staging area (TMA stores)
  int store_warps;
};

// warp 0 lane 0: loader; warps 1..store_warps: "epilogue" stores (and the
// consumers of the loads: wait full, arrive empty)
__global__ void __launch_bounds__(256, 1) bw_kernel(const __grid_constant__ P p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.nnat * p.stage_bytes);  // 1 KB, then the output staging
  const uint32_t bfull = smem_u32(bars), bempty = bfull + 8 * 16;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nnat; ++s) {
      mbar_init(bfull + 8 * s, 1);
      mbar_init(bempty + 8 * s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const bool loads = p.mode & 1, stores = p.mode & 2;
  if (warp == 0) {
    if (lane == 0 && loads) {
      int it = 0;
      for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++it) {
        const int s = it % p.nnat;
        mbar_wait(bempty + 8 * s, ((it / p.nnat) & 1) ^ 1);
        const int bx = t % p.tiles_x, by = t / p.tiles_x;
        mbar_expect(bfull + 8 * s, p.nbox * p.boxw * 2 * p.box_rows);
        for (int k = 0; k < p.nbox; ++k)
          tma_2d(smem_u32(smem + s * p.stage_bytes + k * p.box_slot), &p.map,
                 (int)(p.origin % p.pitch) + bx * p.tile_x - 8 + k * p.boxw, (int)(p.origin / p.pitch) + by * p.tile_y - 1,
                 bfull + 8 * s);
      }
    }
  } else if (warp <= p.store_warps) {
    const int sw = warp - 1;
    int it = 0;
    for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++it) {
      const int s = it % p.nnat;
      if (loads) mbar_wait(bfull + 8 * s, (it / p.nnat) & 1);
      if (stores && (p.mode & 12)) {
        // one elected thread per tile stores the tile from smem (content is
        // whatever is in the staging area) with the TMA engine
        const int bx = t % p.tiles_x, by = t / p.tiles_x;
        const uint32_t st = smem_u32(smem + p.nnat * p.stage_bytes + 1024);
        if (sw == 0 && lane == 0) {
          bulk_wait_read<1>();  // staging half from two tiles ago was read
          if (p.mode & 4) {
            for (int row = 0; row < p.tile_y; ++row)
              bulk_s2g(p.out + p.origin + (int64_t)(by * p.tile_y + row) * p.pitch + bx * p.tile_x, st, p.tile_x * 2);
          } else {
            for (int k = 0; k < p.tile_x / 256; ++k)
              tma_store_2d(&p.omap, st, (int)(p.origin % p.pitch) + bx * p.tile_x + 256 * k,
                           (int)(p.origin / p.pitch) + by * p.tile_y);
          }
          bulk_commit();
        }
      } else if (stores) {
        const int bx = t % p.tiles_x, by = t / p.tiles_x;
        // tile rows split over the store warps; each row = tile_x fp16 =
        // tile_x/16 lanes x 32 B
        const int lanes_per_row = p.tile_x / 16;
        const int rows_per_pass = 32 / lanes_per_row;
        for (int r0 = sw * rows_per_pass; r0 < p.tile_y; r0 += p.store_warps * rows_per_pass) {
          const int row = r0 + lane / lanes_per_row;
          if (row < p.tile_y) {
            uint16_t* dst = p.out + p.origin + (int64_t)(by * p.tile_y + row) * p.pitch + bx * p.tile_x +
                            (lane % lanes_per_row) * 16;
            stg_v8(dst, (uint32_t)t);
          }
        }
      }
      __syncwarp();
      if (loads && sw == 0 && lane == 0) mbar_arrive(bempty + 8 * s);
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int N = 10240;
  const int64_t pitch = 10240 + 64, rows = N + 2 * 32;
  const int64_t origin = 16 * pitch + 16;
  size_t elems = (size_t)rows * pitch + 4096;
  uint16_t *in, *out;
  CK(cudaMalloc(&in, elems * 2));
  CK(cudaMalloc(&out, elems * 2));
  CK(cudaMemset(in, 0, elems * 2));
  CK(cudaMemset(out, 0, elems * 2));
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fnp;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
  struct V {
    const char* name;
    int tile_x, boxw, nbox, nnat, mode, store_warps;
  } vs[] = {
      {"load  3x176 nnat2", 512, 176, 3, 2, 1, 4},  {"load  3x176 nnat3", 512, 176, 3, 3, 1, 4},
      {"load  3x176 nnat4", 512, 176, 3, 4, 1, 4},  {"load  3x176 nnat6", 512, 176, 3, 6, 1, 4},
      {"load  4x136 nnat4", 512, 136, 4, 4, 1, 4},  {"load 5x216 w1024 nnat3", 1024, 216, 5, 3, 1, 4},
      {"store 512 4w", 512, 176, 3, 2, 2, 4},       {"store 512 8w", 512, 176, 3, 2, 2, 7},
      {"both  3x176 nnat2 4w", 512, 176, 3, 2, 3, 4}, {"both  3x176 nnat4 4w", 512, 176, 3, 4, 3, 4},
      {"both  3x176 nnat6 7w", 512, 176, 3, 6, 3, 7},
      {"store bulk rows", 512, 176, 3, 2, 2 | 4, 4}, {"store tensor 256x32", 512, 176, 3, 2, 2 | 8, 4},
      {"both  nnat3 bulk rows", 512, 176, 3, 3, 3 | 4, 4}, {"both  nnat3 tensor", 512, 176, 3, 3, 3 | 8, 4},
      {"both  nnat4 tensor", 512, 176, 3, 4, 3 | 8, 4},
  };
  for (auto& v : vs) {
    P p;
    std::memset(&p, 0, sizeof(p));
    p.tile_x = v.tile_x;
    p.tile_y = 32;
    p.boxw = v.boxw;
    p.nbox = v.nbox;
    p.box_rows = 34;
    p.box_slot = (v.boxw * 2 * 34 + 127) / 128 * 128;
    p.stage_bytes = (p.box_slot * v.nbox + 1023) / 1024 * 1024;
    p.nnat = v.nnat;
    p.tiles_x = N / v.tile_x;
    p.n_tiles = p.tiles_x * (N / 32);
    p.pitch = pitch;
    p.origin = origin;
    p.out = out;
    p.mode = v.mode;
    p.store_warps = v.store_warps;
    cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)pitch * 2};
    cuuint32_t box[2] = {(cuuint32_t)v.boxw, 34};
    cuuint32_t es[2] = {1, 1};
    if (enc(&p.map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
    cuuint32_t obox[2] = {256, 32};
    if (enc(&p.omap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, out, dims, strides, obox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode (out) failed\n");
      return 1;
    }
    size_t smem = (size_t)p.nnat * p.stage_bytes + 1024 + ((v.mode & 12) ? 32768 : 0);
    if (smem > 232448) {
      printf("%-26s smem %zu too big\n", v.name, smem);
      continue;
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int w = 0; w < 3; ++w) bw_kernel<<<sms, 256, smem>>>(p);
    CK(cudaEventRecord(e0));
    const int reps = 20;
    for (int w = 0; w < reps; ++w) bw_kernel<<<sms, 256, smem>>>(p);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us = ms * 1e3 / reps;
    const double rd = (v.mode & 1) ? (double)p.n_tiles * p.nbox * p.boxw * 2 * 34 : 0;
    const double wr = (v.mode & 2) ? (double)N * N * 2 : 0;
    printf("%-26s %8.1f us  read %6.0f MB (%5.2f TB/s)  write %6.0f MB (%5.2f TB/s)  total %5.2f TB/s\n", v.name, us,
           rd / 1e6, rd / us / 1e6, wr / 1e6, wr / us / 1e6, (rd + wr) / us / 1e6);
  }
  return 0;
}

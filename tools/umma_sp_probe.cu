// Probe for the tcgen05.mma.sp kind::f16 operand layouts on sm_100a.
// Not product code: a one-off hardware experiment that pins the metadata (E)
// TMEM layout, the sparse-A / dense-B K-major smem descriptors and the
// instruction-descriptor fields that the stencil kernel relies on.
//
//   usage: umma_sp_probe <variant>
//     variant 0: dense kind::f16 M=128 N=64 K=16 (descriptor sanity)
//     variant 1: sparse, E layout H1 (CUTLASS tmem_e_frg: lane=m0+8k1+16m2, bit=16m1+4c)
//     variant 2: sparse, E layout H2 (lane=m, bit=4*seg)
//     variant 3: sparse H1 but nibble = idx1 | idx0<<2
//     variant 4: sparse H1, A from TMEM (ts form)
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x) do { cudaError_t ce_ = (x); if (ce_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(ce_)); exit(3);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm100)
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nWAIT%=:\n"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
               "@P1 bra DONE%=;\nbra WAIT%=;\nDONE%=:\n}" :: "r"(smem_u32(b)), "r"(par));
}

// a: dense-or-compressed A (128 x KA fp16, logical), b: K x 64 fp16 row-major, e: 128 x 8 nibble bytes
__global__ void probe(int variant, const __half* a, const __half* b, const uint8_t* e, float* d) {
  const int N = 64;
  const bool sparse = variant != 0;
  const int K = sparse ? 32 : 16;    // logical K
  const int KA = sparse ? 16 : 16;   // physical A columns
  __shared__ __align__(1024) uint8_t sA[128 * 16 * 2];
  __shared__ __align__(1024) uint8_t sB[64 * 32 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // A K-major no swizzle: (m/8)*256 + (k/8)*128 + (m%8)*16 + (k%8)*2
  for (int idx = tid; idx < 128 * KA; idx += blockDim.x) {
    int m = idx / KA, k = idx % KA;
    *(__half*)(sA + (m / 8) * 256 + (k / 8) * 128 + (m % 8) * 16 + (k % 8) * 2) = a[m * KA + k];
  }
  // B K-major: element (k, n) at (n/8)*SBO + (k/8)*128 + (n%8)*16 + (k%8)*2 ; SBO = (K/8)*128
  const int SBO_B = (K / 8) * 128;
  for (int idx = tid; idx < K * N; idx += blockDim.x) {
    int k = idx / N, n = idx % N;
    *(__half*)(sB + (n / 8) * SBO_B + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) = b[k * N + n];
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tb = tmem_base;
  const uint32_t col_d = 0, col_e = 128, col_a = 160;
  // write E words into TMEM column col_e (warp w owns lanes 32w..32w+31)
  if (sparse) {
    int m = warp * 32 + lane;  // this thread's TMEM lane
    uint32_t word = 0;
    if (variant == 1 || variant == 3 || variant == 4) {
      int m0 = m % 8, k1 = (m / 8) % 2, m2 = m / 16;
      for (int m1 = 0; m1 < 2; ++m1)
        for (int c = 0; c < 4; ++c) {
          int row = m0 + 8 * m1 + 16 * m2, seg = 4 * k1 + c;
          uint32_t nib = e[row * 8 + seg];
          if (variant == 3) nib = ((nib & 3) << 2) | ((nib >> 2) & 3);
          word |= nib << (16 * m1 + 4 * c);
        }
    } else {
      for (int s = 0; s < 8; ++s) word |= (uint32_t)e[m * 8 + s] << (4 * s);
    }
    uint32_t taddr = tb + ((uint32_t)(warp * 32) << 16) + col_e;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(taddr), "r"(word));
    if (variant == 4) {
      // A in TMEM: lane m, 8 columns of packed half2 (k' = 2c, 2c+1)
      for (int c = 0; c < 8; ++c) {
        __half2 h = __halves2half2(a[m * 16 + 2 * c], a[m * 16 + 2 * c + 1]);
        uint32_t w = *(uint32_t*)&h;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(taddr - col_e + col_a + c), "r"(w));
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0 && lane == 0) {
    uint64_t adesc = make_desc(smem_u32(sA), 128, 256);
    uint64_t bdesc = make_desc(smem_u32(sB), 128, SBO_B);
    uint32_t idesc = 0;
    idesc |= (sparse ? 1u : 0u) << 2;  // sparse flag
    idesc |= 1u << 4;                  // D fp32
    // a_format=b_format=F16 (0); K-major both (0)
    idesc |= (uint32_t)(N >> 3) << 17;
    idesc |= (uint32_t)(128 >> 4) << 24;
    uint32_t dt = tb + col_d, et = tb + col_e, at = tb + col_a;
    uint32_t acc = 0;
    if (!sparse) {
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                   :: "r"(dt), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    } else if (variant == 4) {
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n"
                   :: "r"(dt), "r"(at), "l"(bdesc), "r"(et), "r"(acc), "r"(idesc));
    } else {
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %5, p;\n}\n"
                   :: "r"(dt), "l"(adesc), "l"(bdesc), "r"(et), "r"(acc), "r"(idesc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // read D: warp w lanes 32w.. ; 64 columns
  {
    int m = warp * 32 + lane;
    for (int c = 0; c < N; ++c) {
      uint32_t r;
      uint32_t taddr = tb + ((uint32_t)(warp * 32) << 16) + col_d + c;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      d[m * N + c] = __uint_as_float(r);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tb));
}

int main(int argc, char** argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 1;
  const int N = 64;
  bool sparse = variant != 0;
  int K = sparse ? 32 : 16;
  srand(1234 + variant);
  std::vector<float> Adense(128 * K, 0.f), B(K * N), D(128 * N), Dref(128 * N, 0.f);
  std::vector<__half> a_h(128 * 16), b_h(K * N);
  std::vector<uint8_t> e(128 * 8, 0);
  for (int m = 0; m < 128; ++m) {
    if (!sparse) {
      for (int k = 0; k < 16; ++k) { float v = (float)(rand() % 7 - 3); Adense[m * K + k] = v; a_h[m * 16 + k] = __float2half(v); }
    } else {
      for (int s = 0; s < 8; ++s) {
        int p0 = rand() % 4, p1 = rand() % 4;
        while (p1 == p0) p1 = rand() % 4;
        if (p0 > p1) { int t = p0; p0 = p1; p1 = t; }
        float v0 = (float)(rand() % 7 - 3), v1 = (float)(rand() % 7 - 3);
        Adense[m * K + 4 * s + p0] = v0; Adense[m * K + 4 * s + p1] = v1;
        a_h[m * 16 + 2 * s] = __float2half(v0); a_h[m * 16 + 2 * s + 1] = __float2half(v1);
        e[m * 8 + s] = (uint8_t)(p0 | (p1 << 2));
      }
    }
  }
  for (int i = 0; i < K * N; ++i) { float v = (float)(rand() % 9 - 4); B[i] = v; b_h[i] = __float2half(v); }
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) { float s = 0; for (int k = 0; k < K; ++k) s += Adense[m * K + k] * B[k * N + n]; Dref[m * N + n] = s; }
  __half *da, *db; uint8_t* de; float* dd;
  CK(cudaMalloc(&da, a_h.size() * 2)); CK(cudaMalloc(&db, b_h.size() * 2)); CK(cudaMalloc(&de, e.size())); CK(cudaMalloc(&dd, D.size() * 4));
  CK(cudaMemcpy(da, a_h.data(), a_h.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b_h.data(), b_h.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(de, e.data(), e.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dd, 0xFF, D.size() * 4));
  probe<<<1, 128>>>(variant, da, db, de, dd);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dd, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0; double maxerr = 0;
  for (int i = 0; i < 128 * N; ++i) { double er = fabs(D[i] - Dref[i]); if (er > 1e-3) { if (bad < 5) printf("  mismatch m=%d n=%d got %g want %g\n", i / N, i % N, D[i], Dref[i]); ++bad; } if (er > maxerr) maxerr = er; }
  // for failures, check whether rows match some other row of the reference (diagnostic)
  printf("variant %d: %s (bad=%d, maxerr=%g)\n", variant, bad ? "FAIL" : "PASS", bad, maxerr);
  return bad ? 1 : 0;
}

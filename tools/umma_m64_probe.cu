// Probe for tcgen05.mma.sp kind::f16 with M = 64 (cta_group::1), ts form.
// Not product code: a one-off hardware experiment that pins how an M = 64
// sparse MMA addresses its D / A / E operands in TMEM, so the step kernel can
// issue M = 64 MMAs on the half of the accumulator lanes a K-block feeds.
//
//   usage: umma_m64_probe <h> <emode> <amode> [accum]
//     h      TMEM lane offset of the half (0 or 16) in the D address
//     emode  0: M=128 E image, E address lane offset h
//            1: M=128 E image, E address lane offset 0
//            2: compact E image (M=64 rows m' at lane m0+8k1+16m2), offset 0
//     amode  0: M=128 A image (row m at lane m), A address lane offset h
//            1: compact A image (row m' at lane m'), offset 0
//     accum  1: first an M=128 MMA with accumulate=0 over all lanes, then the
//               M=64 one with accumulate=1 (checks that the other half keeps
//               the M=128 result)
// Expected if M = 64 row m' = m0 + 16*m1 lives on D lane h + m0 + 32*m1:
// those lanes equal the M=128 reference rows of the same lane; all other
// lanes keep the sentinel (or the M=128 result in accum mode).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
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
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nWAIT%=:\n"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
               "@P1 bra DONE%=;\nbra WAIT%=;\nDONE%=:\n}" :: "r"(smem_u32(b)), "r"(par));
}
__device__ __forceinline__ void tst(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(taddr), "r"(v));
}
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t e, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(e), "r"(acc), "r"(idesc));
}

constexpr int N = 64;
// ewords/awords: per TMEM lane, the E word and 8 A words (the host builds the layout)
__global__ void probe(int h, int emode, int amode, int accum, const uint32_t* e128, const uint32_t* a128,
                      const uint32_t* e64, const uint32_t* a64, const __half* b, float* d) {
  __shared__ __align__(1024) uint8_t sB[64 * 32 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int SBO_B = (32 / 8) * 128;
  for (int idx = tid; idx < 32 * N; idx += blockDim.x) {
    int k = idx / N, n = idx % N;
    *(__half*)(sB + (n / 8) * SBO_B + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) = b[k * N + n];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  // columns: D 0..63, E128 128, E64 130, A128 136..143, A64 144..151
  const uint32_t col_d = 0, col_e128 = 128, col_e64 = 130, col_a128 = 136, col_a64 = 144;
  {
    const int m = warp * 32 + lane;
    const uint32_t row = tb + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < N; ++c) tst(row + col_d + c, 0x7FC00001u);
    tst(row + col_e128, e128[m]);
    tst(row + col_e64, e64[m]);
    for (int c = 0; c < 8; ++c) {
      tst(row + col_a128 + c, a128[m * 8 + c]);
      tst(row + col_a64 + c, a64[m * 8 + c]);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0 && lane == 0) {
    const uint64_t bdesc = make_desc(smem_u32(sB), 128, SBO_B);
    const uint32_t base = (1u << 2) | (1u << 4) | ((uint32_t)(N >> 3) << 17);
    const uint32_t id128 = base | ((uint32_t)(128 >> 4) << 24);
    const uint32_t id64 = base | ((uint32_t)(64 >> 4) << 24);
    const uint32_t hoff = (uint32_t)h << 16;
    if (accum) mma(tb + col_d, tb + col_a128, bdesc, tb + col_e128, id128, 0u);
    uint32_t et = emode == 0 ? tb + hoff + col_e128 : (emode == 1 ? tb + col_e128 : tb + col_e64);
    uint32_t at = amode == 0 ? tb + hoff + col_a128 : tb + col_a64;
    mma(tb + hoff + col_d, at, bdesc, et, id64, accum ? 1u : 0u);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
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

static uint32_t e_word(const std::vector<uint8_t>& nib, int lane, int (*row_of)(int)) {
  // M=128 CUTLASS tmem_e_frg: row m = m0 + 8 m1 + 16 m2, seg = 4 k1 + c -> lane m0 + 8 k1 + 16 m2, bits 16 m1 + 4 c
  int m0 = lane % 8, k1 = (lane / 8) % 2, m2 = lane / 16;
  uint32_t w = 0;
  for (int m1 = 0; m1 < 2; ++m1)
    for (int c = 0; c < 4; ++c) {
      int row = row_of(m0 + 8 * m1 + 16 * m2);
      if (row < 0) continue;
      w |= (uint32_t)nib[row * 8 + 4 * k1 + c] << (16 * m1 + 4 * c);
    }
  return w;
}
static int g_h = 0;
static int row_id(int m) { return m; }
static int row_m64(int mp) { return mp < 64 ? g_h + (mp % 16) + 32 * (mp / 16) : -1; }  // compact row -> image row

int main(int argc, char** argv) {
  int h = argc > 1 ? atoi(argv[1]) : 0;
  int emode = argc > 2 ? atoi(argv[2]) : 0;
  int amode = argc > 3 ? atoi(argv[3]) : 0;
  int accum = argc > 4 ? atoi(argv[4]) : 0;
  g_h = h;
  srand(4321 + h);
  const int K = 32;
  std::vector<float> Adense(128 * K, 0.f), B(K * N), D(128 * N), Dref(128 * N, 0.f);
  std::vector<__half> a_h(128 * 16), b_h(K * N);
  std::vector<uint8_t> nib(128 * 8, 0);
  for (int m = 0; m < 128; ++m)
    for (int s = 0; s < 8; ++s) {
      int p0 = rand() % 4, p1 = rand() % 4;
      while (p1 == p0) p1 = rand() % 4;
      if (p0 > p1) { int t = p0; p0 = p1; p1 = t; }
      float v0 = (float)(rand() % 7 - 3), v1 = (float)(rand() % 7 - 3);
      Adense[m * K + 4 * s + p0] = v0; Adense[m * K + 4 * s + p1] = v1;
      a_h[m * 16 + 2 * s] = __float2half(v0); a_h[m * 16 + 2 * s + 1] = __float2half(v1);
      nib[m * 8 + s] = (uint8_t)(p0 | (p1 << 2));
    }
  for (int i = 0; i < K * N; ++i) { float v = (float)(rand() % 9 - 4); B[i] = v; b_h[i] = __float2half(v); }
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) { float s = 0; for (int k = 0; k < K; ++k) s += Adense[m * K + k] * B[k * N + n]; Dref[m * N + n] = s; }
  std::vector<uint32_t> e128(128), e64(128, 0), a128(128 * 8), a64(128 * 8, 0);
  for (int l = 0; l < 128; ++l) {
    e128[l] = e_word(nib, l, row_id);
    e64[l] = l < 64 ? e_word(nib, l, row_m64) : 0;
    for (int c = 0; c < 8; ++c) {
      __half2 v = __halves2half2(a_h[l * 16 + 2 * c], a_h[l * 16 + 2 * c + 1]);
      a128[l * 8 + c] = *(uint32_t*)&v;
      int src = l < 64 ? row_m64(l) : -1;
      if (src >= 0) {
        __half2 w = __halves2half2(a_h[src * 16 + 2 * c], a_h[src * 16 + 2 * c + 1]);
        a64[l * 8 + c] = *(uint32_t*)&w;
      }
    }
  }
  uint32_t *de128, *da128, *de64, *da64; __half* db; float* dd;
  CK(cudaMalloc(&de128, 512)); CK(cudaMalloc(&de64, 512)); CK(cudaMalloc(&da128, 4096)); CK(cudaMalloc(&da64, 4096));
  CK(cudaMalloc(&db, b_h.size() * 2)); CK(cudaMalloc(&dd, D.size() * 4));
  CK(cudaMemcpy(de128, e128.data(), 512, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(de64, e64.data(), 512, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(da128, a128.data(), 4096, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(da64, a64.data(), 4096, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b_h.data(), b_h.size() * 2, cudaMemcpyHostToDevice));
  probe<<<1, 128>>>(h, emode, amode, accum, de128, da128, de64, da64, db, dd);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dd, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad_in = 0, bad_out = 0, shown = 0;
  for (int l = 0; l < 128; ++l) {
    bool in_half = (l % 32) >= h && (l % 32) < h + 16;
    for (int n = 0; n < N; ++n) {
      float got = D[l * N + n];
      if (in_half) {
        if (fabsf(got - Dref[l * N + n]) > 1e-3f) { ++bad_in; if (shown++ < 4) printf("  lane %d n %d got %g want %g\n", l, n, got, Dref[l * N + n]); }
      } else {
        bool ok = accum ? fabsf(got - Dref[l * N + n]) <= 1e-3f : std::isnan(got);
        if (!ok) { ++bad_out; if (shown++ < 8) printf("  (other half) lane %d n %d got %g\n", l, n, got); }
      }
    }
  }
  printf("m64 h=%d emode=%d amode=%d accum=%d: %s (bad in half %d, disturbed outside %d)\n", h, emode, amode, accum,
         (bad_in || bad_out) ? "FAIL" : "PASS", bad_in, bad_out);
  return (bad_in || bad_out) ? 1 : 0;
}

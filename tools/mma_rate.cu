// Microbenchmark (dev aid, not product code): issue rate of tcgen05.mma(.sp)
// kind::f16 M=128 on sm_100a, one CTA per SM, one issuing thread.
//   usage: mma_rate            (prints a table)
// Columns: form (sp-ts = sparse, A+E in TMEM: the stencil kernel's form;
// dense-ss = dense A/B in smem), N, B-operand SBO (bytes between 8-row
// N groups; the stencil kernel's B image uses r_in*KC*128), accumulator
// chains (1 = every MMA into one accumulator), cycles per MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nWAIT%=:\n"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
               "@P1 bra DONE%=;\nbra WAIT%=;\nDONE%=:\n}" ::"r"(b), "r"(par));
}

__global__ void rate(int form, int n, int sbo, int chains, int S, int rounds, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  unsigned long long t0 = 0, t1 = 0;
  // form bit 2: whole warp 0 runs the loop (converged), one elected lane issues
  const bool conv = (form & 4) != 0;
  form &= 3;
  if (conv ? warp == 0 : threadIdx.x == 0) {
    const uint32_t idesc_sp = (1u << 2) | (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t idesc_dn = (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t bbase = smem_u32(smem);
    const uint32_t abase = bbase + 160 * 1024;
    for (int r = 0; r < rounds + 1; ++r) {
      if (r == 1) t0 = clock64();
      for (int s = 0; s < S; ++s) {
        const uint32_t d = tmem + (chains > 1 ? (s % chains) * n : 0);
        const uint32_t acc = (chains > 1 ? s >= chains : s > 0) ? 1u : 0u;
        const uint64_t bdesc = make_desc(bbase + (s % 8) * 512, 128, sbo);
        if (form == 0 && conv) {
          const uint32_t e = tmem + 256 + 2 * (s % 16), a = tmem + 320 + 8 * (s % 16);
          asm volatile("{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|q, 0xffffffff;\n"
                       "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n" ::"r"(d),
                       "r"(a), "l"(bdesc), "r"(e), "r"(acc), "r"(idesc_sp));
        } else if (form == 0) {
          const uint32_t e = tmem + 256 + 2 * (s % 16), a = tmem + 320 + 8 * (s % 16);
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n" ::"r"(d),
                       "r"(a), "l"(bdesc), "r"(e), "r"(acc), "r"(idesc_sp));
        } else {
          const uint64_t adesc = make_desc(abase, 128, 256);
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %3, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n}\n" ::"r"(d),
                       "l"(adesc), "l"(bdesc), "r"(acc), "r"(idesc_dn));
        }
      }
      if (conv) {
        asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                     "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&bar)));
      } else {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      }
      mbar_wait(smem_u32(&bar), r & 1);
    }
    t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Fully unrolled, operands precomputed: the tightest issue sequence.
template <int S>
__global__ void rate_unrolled(int n, int sbo, int rounds, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (warp == 0) {
    const uint32_t idesc = (1u << 2) | (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t bbase = smem_u32(smem);
    const uint64_t bdesc0 = make_desc(bbase, 128, sbo);
    unsigned long long t0 = 0;
    for (int r = 0; r < rounds + 1; ++r) {
      if (r == 1) t0 = clock64();
#pragma unroll
      for (int s = 0; s < S; ++s) {
        asm volatile("{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|q, 0xffffffff;\n"
                     "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n" ::"r"(tmem),
                     "r"(tmem + 320 + 8 * s), "l"(bdesc0 + (uint64_t)(s * 32)), "r"(tmem + 256 + 2 * s), "r"(s > 0 ? 1u : 0u),
                     "r"(idesc));
      }
      asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                   "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&bar)));
      mbar_wait(smem_u32(&bar), r & 1);
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int S = 16, rounds = 200;
  struct C { int form, n, sbo, chains; } cs[] = {
      {0, 64, 512, 1}, {0, 128, 4352, 1}, {0, 256, 512, 1},
      {4, 64, 512, 1}, {4, 128, 4352, 1}, {4, 256, 512, 1}, {4, 128, 512, 2},
      {1, 128, 256, 1}, {1, 256, 256, 1},
  };
  for (auto c : cs) {
    for (int grid : {148}) {
      rate<<<grid, 128, 200 * 1024>>>(c.form, c.n, c.sbo, c.chains, S, rounds, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%-8s N=%3d sbo=%5d chains=%d grid=%3d: %.1f cycles/MMA  (floor %d)  %s\n", (c.form & 3) ? "dense-ss" : (c.form & 4) ? "sp-ts-conv" : "sp-ts",
             c.n, c.sbo, c.chains, grid, (double)h / (rounds * S), 128 * c.n / 256, cudaGetErrorString(e));
    }
  }
  cudaFuncSetAttribute(rate_unrolled<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(rate_unrolled<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int n : {64, 128, 256}) {
    unsigned long long h = 0;
    rate_unrolled<16><<<148, 128, 200 * 1024>>>(n, 512, rounds, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("unrolled S=16 N=%3d: %.1f cycles/MMA (floor %d) %s\n", n, (double)h / (rounds * 16), 128 * n / 256, cudaGetErrorString(e));
    rate_unrolled<4><<<148, 128, 200 * 1024>>>(n, 512, rounds, d);
    e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("unrolled S=4  N=%3d: %.1f cycles/MMA (floor %d) %s\n", n, (double)h / (rounds * 4), 128 * n / 256, cudaGetErrorString(e));
  }
  return 0;
}

// Energy per sparse MMA (dev aid, not product code): 148 CTAs, one converged
// warp each, issue unrolled tcgen05.mma.sp.cta_group::1.kind::f16 (A and E in
// TMEM, B in smem, one accumulator) for ~2 s per shape; board energy from
// NVML's total-energy counter.  Question answered: does an M = 64 MMA cost
// less energy than an M = 128 one (the stencil's MMAs compute mostly
// structurally-zero rows of the accumulator)?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mma_energy tools/mma_energy.cu -lnvidia-ml
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <nvml.h>
#include <unistd.h>

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

// mode 0: issue MMAs; mode 1: same loop without the MMAs (commit + wait only)
__global__ void burn(int m, int n, int rounds, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u);  // nonzero fp16 data
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
  {  // A (cols 320..447) and E (256..287) with nonzero values / valid nibbles
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 128; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lane_base + 320 + c), "r"(0x3c003800u));
    for (int c = 0; c < 32; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lane_base + 256 + c), "r"(0x44444444u));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint32_t idesc = (1u << 2) | (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
    const uint64_t bdesc0 = make_desc(smem_u32(smem), 128, 4352);
    for (int r = 0; r < rounds; ++r) {
      if (mode == 0) {
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          asm volatile("{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|q, 0xffffffff;\n"
                       "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n" ::"r"(tmem),
                       "r"(tmem + 320 + 8 * s), "l"(bdesc0 + (uint64_t)(s * 32)), "r"(tmem + 256 + 2 * s),
                       "r"(s > 0 ? 1u : 0u), "r"(idesc));
        }
      }
      asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                   "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&bar)));
      mbar_wait(smem_u32(&bar), r & 1);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  nvmlInit();
  nvmlDevice_t dev;
  nvmlDeviceGetHandleByIndex(0, &dev);
  cudaFuncSetAttribute(burn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct S { int m, n, mode; } cs[] = {{128, 128, 1}, {128, 128, 0}, {64, 128, 0}, {128, 64, 0}, {64, 64, 0}, {128, 128, 0}};
  for (auto c : cs) {
    // calibrate rounds for ~2 s
    int rounds = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    burn<<<148, 128, 200 * 1024>>>(c.m, c.n, rounds, c.mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    rounds = (int)(rounds * 2000.0f / (ms > 0.01f ? ms : 0.01f));
    sleep(1);
    unsigned long long ea = 0, eb = 0;
    nvmlDeviceGetTotalEnergyConsumption(dev, &ea);
    cudaEventRecord(e0);
    burn<<<148, 128, 200 * 1024>>>(c.m, c.n, rounds, c.mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    nvmlDeviceGetTotalEnergyConsumption(dev, &eb);
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned int clk = 0;
    nvmlDeviceGetClockInfo(dev, NVML_CLOCK_SM, &clk);
    const double mmas = 148.0 * rounds * (c.mode == 0 ? 8 : 0);
    printf("M=%3d N=%3d %s: %.0f ms, %.0f W, %u MHz at end, %.2f ns/MMA/SM, energy %.3f nJ per MMA (board, incl. idle)\n", c.m,
           c.n, c.mode ? "no-MMA loop" : "sparse MMA ", ms, (eb - ea) / ms, clk, mmas ? ms * 1e6 * 148 / mmas : 0.0,
           mmas ? (eb - ea) * 1e6 / mmas : 0.0);
    printf("   error: %s\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

// Issue cost of the step kernel's MMA sequence (not product code): cycles per
// tcgen05.mma.sp (M = 128, ts form) for S MMAs per tile at N = 32 (B27) and
// N = 128 (B9), one CTA per SM, commit per tile without waiting (so the
// figure is issue- or tensor-bound, whichever is slower; the tensor floor is
// 128 N / 256 cycles).
//   form 0: elect.sync inside every MMA's asm (the kernel before this probe)
//   form 1: one elect.sync per tile; the elected lane runs the unrolled
//           sequence in a divergent branch
//   form 2: converged warp, one elect.sync per tile kept in a register, a
//           per-MMA predicate from it
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

template <int S, int N, int FORM>
__global__ void issue(int rounds, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
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
    const uint32_t idesc = (1u << 2) | (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bdesc0 = make_desc(smem_u32(smem), 128, 512);
    unsigned long long t0 = 0;
    for (int r = 0; r < rounds + 1; ++r) {
      if (r == 1) t0 = clock64();
      const uint32_t dcol = tmem + (r & 1) * N;  // two accumulator stages
      if constexpr (FORM == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s)
          asm volatile("{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|q, 0xffffffff;\n"
                       "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n" ::"r"(dcol),
                       "r"(tmem + 320 + 8 * (s % 24)), "l"(bdesc0 + (uint64_t)(s * 32)), "r"(tmem + 256 + 2 * (s % 24)),
                       "r"(s > 0 ? 1u : 0u), "r"(idesc));
      } else if constexpr (FORM == 1) {
        // one elect per tile; the elected lane issues the unrolled sequence
        uint32_t leader;
        asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\nselp.u32 %0, 1, 0, q;\n}" : "=r"(leader));
        if (leader) {
#pragma unroll
          for (int s = 0; s < S; ++s)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n" ::"r"(dcol),
                         "r"(tmem + 320 + 8 * (s % 24)), "l"(bdesc0 + (uint64_t)(s * 32)),
                         "r"(tmem + 256 + 2 * (s % 24)), "r"(s > 0 ? 1u : 0u), "r"(idesc));
        }
        __syncwarp();
      } else {
        // converged warp, elect once, per-MMA predicate from a register
        uint32_t leader;
        asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\nselp.u32 %0, 1, 0, q;\n}" : "=r"(leader));
#pragma unroll
        for (int s = 0; s < S; ++s)
          asm volatile("{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 q, %6, 0;\n"
                       "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %5, p;\n}\n" ::"r"(dcol),
                       "r"(tmem + 320 + 8 * (s % 24)), "l"(bdesc0 + (uint64_t)(s * 32)),
                       "r"(tmem + 256 + 2 * (s % 24)), "r"(s > 0 ? 1u : 0u), "r"(idesc), "r"(leader));
      }
      asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                   "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
                       smem_u32(&bar)));
    }
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}" ::"r"(
                     smem_u32(&bar)),
                 "r"((uint32_t)(rounds & 1)));
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int S, int N, int FORM>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int rounds = 400;
  cudaFuncSetAttribute(issue<S, N, FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  issue<S, N, FORM><<<148, 128, 160 * 1024>>>(rounds, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-26s S=%2d N=%3d: %6.1f cycles/MMA (tensor floor %d) %s\n", name, S, N, (double)h / (rounds * S),
         128 * N / 256, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<30, 32, 0>("elect per MMA");
  run<30, 32, 1>("elected lane, divergent");
  run<30, 32, 2>("converged, predicate reg");
  run<9, 128, 0>("elect per MMA");
  run<9, 128, 1>("elected lane, divergent");
  run<9, 128, 2>("converged, predicate reg");
  return 0;
}

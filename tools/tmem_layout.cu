// Pins the register <- TMEM mapping of tcgen05.ld.16x256b (and .x2 column
// stepping, and the upper 16-lane half) on the hardware: one warp stores
// value (lane << 16 | column) with tcgen05.st.32x32b, then reads it back with
// tcgen05.ld.16x256b and prints which (lane, column) each register of each
// thread received.   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_layout tools/tmem_layout.cu
#include <cstdio>
#include <cstdint>

__global__ void probe(uint32_t* out) {
  __shared__ uint32_t holder;
  const int lane = threadIdx.x;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
      (uint32_t)__cvta_generic_to_shared(&holder)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  for (int c = 0; c < 32; ++c) {
    uint32_t v = ((uint32_t)lane << 16) | (uint32_t)c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + c), "r"(v));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t r[8];
  // lanes 0..15, columns 0..15 (x2)
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(tmem));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int i = 0; i < 8; ++i) out[lane * 16 + i] = r[i];
  // lanes 16..31, columns 8..15 (x1, lane field + 16, column + 8)
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(tmem + (16u << 16) + 8));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int i = 0; i < 4; ++i) out[lane * 16 + 8 + i] = r[i];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 32 * 16 * 4);
  cudaMemset(d, 0xff, 32 * 16 * 4);
  probe<<<1, 32>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  uint32_t h[32 * 16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("thread: 16x256b.x2 at (lane 0, col 0): r0..r7 as lane:col | 16x256b.x1 at (lane 16, col 8): r0..r3\n");
  for (int t = 0; t < 32; ++t) {
    printf("t%02d:", t);
    for (int i = 0; i < 12; ++i) {
      if (i == 8) printf(" |");
      printf(" %2u:%-2u", h[t * 16 + i] >> 16, h[t * 16 + i] & 0xffff);
    }
    printf("\n");
  }
  return 0;
}

// Developer probe (not part of the product): thread <-> (lane, column) maps of
// tcgen05.ld.16x256b and tcgen05.st.16x128b, found by writing a known pattern
// with 32x32b stores / reading back with 32x32b loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2212_11296_b200/csrc scripts/tmem_shape_probe.cu -o scripts/_exp/shape_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace vqb;

__global__ void __launch_bounds__(128, 1) k_probe(uint32_t* out) {
  __shared__ uint32_t tslot;
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 64);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tq = tmem + ((uint32_t)(w * 32) << 16);
  // pattern: value = (lane_in_tmem << 8) | column, columns 0..15
  uint32_t z[8];
  for (int h = 0; h < 2; ++h) {
    for (int i = 0; i < 8; ++i) z[i] = ((uint32_t)(w * 32 + lane) << 8) | (uint32_t)(h * 8 + i);
    tc::tmem_st8u(tq + h * 8, z);
  }
  tc::tmem_wait_st();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  // 16x256b.x2 load at lane offset 0 and 16 of the warp's quadrant
  for (int half = 0; half < 2; ++half) {
    uint32_t r[8];
    const uint32_t a = tq + ((uint32_t)(half * 16) << 16);
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(a));
    tc::tmem_wait_ld();
    for (int i = 0; i < 8; ++i) out[((w * 2 + half) * 32 + lane) * 8 + i] = r[i];
  }
  __syncthreads();
  // 16x128b.x2 store test: write (tag) to columns 32..39, read back with 32x32b
  for (int half = 0; half < 2; ++half) {
    const uint32_t a = tq + ((uint32_t)(half * 16) << 16) + 32;
    uint32_t s[4];
    for (int i = 0; i < 4; ++i) s[i] = ((uint32_t)lane << 8) | (uint32_t)i | (half ? 0x10000u : 0u);
    asm volatile("tcgen05.st.sync.aligned.16x128b.x2.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(s[0]),
                 "r"(s[1]), "r"(s[2]), "r"(s[3])
                 : "memory");
  }
  tc::tmem_wait_st();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(tq + 32));
    tc::tmem_wait_ld();
    for (int i = 0; i < 8; ++i) out[4 * 2 * 32 * 8 + (w * 32 + lane) * 8 + i] = r[i];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 64);
}

int main() {
  uint32_t* d;
  const int n = 4 * 2 * 32 * 8 + 128 * 8;
  cudaMalloc(&d, n * 4);
  k_probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  static uint32_t h[4 * 2 * 32 * 8 + 128 * 8];
  cudaMemcpy(h, d, n * 4, cudaMemcpyDeviceToHost);
  for (int w = 0; w < 2; ++w)
    for (int half = 0; half < 2; ++half) {
      printf("ld 16x256b.x2 warp %d half %d: thread: (lane,col) per reg\n", w, half);
      for (int t = 0; t < 32; ++t) {
        printf("  t%2d:", t);
        for (int i = 0; i < 8; ++i) {
          const uint32_t v = h[((w * 2 + half) * 32 + t) * 8 + i];
          printf(" (%3u,%2u)", v >> 8, v & 255);
        }
        printf("\n");
      }
    }
  printf("st 16x128b.x2 read back (32x32b): lane: per column 32..39 -> (half, thread, reg)\n");
  for (int l = 0; l < 32; ++l) {
    printf("  lane %2d:", l);
    for (int i = 0; i < 8; ++i) {
      const uint32_t v = h[4 * 2 * 32 * 8 + l * 8 + i];
      printf(" (%u,%2u,%u)", v >> 16, (v >> 8) & 255, v & 255);
    }
    printf("\n");
  }
  return 0;
}

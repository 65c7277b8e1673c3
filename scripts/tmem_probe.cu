// Developer probe (not part of the product): tcgen05.ld throughput per SM
// (32x32b.x16: 2 KB per warp instruction) with W warps loading their lane
// quadrant's columns back to back, and tcgen05.st throughput likewise.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2212_11296_b200/csrc scripts/tmem_probe.cu -o scripts/_tmem_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace vqb;

template <int MODE>  // 0: ld x16, 1: st x8 (u32), 2: ld x16 + 16 dependent FMAs
__global__ void __launch_bounds__(1024, 1) k_probe(int nw, int reps, unsigned long long* out,
                                                    float* sink) {
  __shared__ uint32_t tslot;
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  const int w = threadIdx.x >> 5;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  if (w < nw) {
    const uint32_t tq = tmem + ((uint32_t)((w & 3) * 32) << 16);
    for (int r = 0; r < reps; ++r) {
      const uint32_t col = (uint32_t)(((w >> 2) * 48 + (r % 3) * 16) & 511);
      if (MODE == 1) {
        const uint32_t z[8] = {0u, 1u, 2u, 3u, 4u, 5u, 6u, (uint32_t)r};
        tc::tmem_st8u(tq + col, z);
        tc::tmem_wait_st();
      } else {
        float v[16];
        tc::tmem_ld16(tq + col, v);
        tc::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += v[i];
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  if (acc == 1234.5f) sink[0] = acc;
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4);
  const int reps = 2000;
  for (int mode = 0; mode < 2; ++mode)
    for (int nw : {4, 8, 16, 32}) {
      if (mode == 0) k_probe<0><<<148, 1024>>>(nw, reps, d, sink);
      else k_probe<1><<<148, 1024>>>(nw, reps, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long c;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)nw * reps * (mode == 0 ? 2048 : 1024);
      printf("%s warps %2d: %8.1f cycles per op per warp, %6.1f B/clk/SM\n",
             mode == 0 ? "tcgen05.ld 32x32b.x16" : "tcgen05.st 32x32b.x8 ", nw,
             (double)c / reps, bytes / c);
    }
  return 0;
}

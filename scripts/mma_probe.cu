// Developer probe (not part of the product): tensor-pipe cost of one
// tcgen05.mma kind::f16 instruction by shape, A from shared memory (SS) or
// from TMEM (TS), issued back to back by one thread of one CTA per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2212_11296_b200/csrc scripts/mma_probe.cu -o /tmp/mma_probe
//   /tmp/mma_probe
// Measured (B200): ~50 cycles per MMA for N <= 64 issued unrolled, 67 at N = 128,
// 132 at N = 256 (~4.0k MAC/clk); concurrent tcgen05.ld traffic from 16 warps
// slows a TS N = 32 chain by < 7%.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace vqb;

// LDW extra warps (1..LDW) stream tcgen05.ld of their lane quadrant while the
// MMAs run: does TMEM read traffic slow the tensor pipe?
template <int CHAIN, int TS, int LDW = 0>
__global__ void __launch_bounds__(32 * (1 + 16), 1) k_probe(int n, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const uint32_t sb = tc::smem_u32(smem);
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    stop = 0;
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {  // the whole warp runs the loop; one elected lane issues
    const uint32_t idesc = tc::make_idesc_bf16(128, n) | (TS ? (1u << 16) : 0u);
    const uint64_t da = tc::make_desc_sw128(sb);
    const uint64_t db = tc::make_desc_sw128(sb + 16384);
    uint32_t ph = 0;
    long long t0 = 0;
    for (int r = 0; r <= reps; ++r) {
      if (r == 1) t0 = clock64();
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < CHAIN; ++k) {
          if (TS)
            tc::mma_bf16_ts(tmem + 256, tmem + (uint32_t)(k & 7) * 8,
                            db + (uint64_t)((k & 3) * 2), idesc, k > 0 ? 1u : 0u);
          else
            tc::mma_bf16(tmem + 256, da + (uint64_t)((k & 3) * 2), db + (uint64_t)((k & 3) * 2),
                         idesc, k > 0 ? 1u : 0u);
        }
        tc::mma_commit(&bar);
      }
      __syncwarp();
      tc::mbar_wait(&bar, ph);
      ph ^= 1;
    }
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    if (threadIdx.x == 0) stop = 1;
  } else if (threadIdx.x / 32 <= LDW) {
    const int w = threadIdx.x / 32;
    const uint32_t tq = tmem + ((uint32_t)((w & 3) * 32) << 16);
    float acc = 0.f;
    while (!stop) {
      float v[16];
      tc::tmem_ld16(tq + (uint32_t)((w * 16) & 255), v);
      tc::tmem_wait_ld();
      acc += v[0];
    }
    if (acc == 12345.f) out[1] = 1;
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

template <int CHAIN, int TS, int LDW = 0>
void run(int n, unsigned long long* d) {
  const int smem = 16384 + 32768 + 1024;
  const int reps = 200;
  cudaFuncSetAttribute(k_probe<CHAIN, TS, LDW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_probe<CHAIN, TS, LDW><<<148, 32 * (1 + 16), smem>>>(n, reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / reps;
  printf("%s M=128 N=%3d K=16 chain %2d ld-warps %2d: %8.1f cycles per chain, %7.1f per MMA, %6.0f MAC/clk\n",
         TS ? "TS" : "SS", n, CHAIN, LDW, per, per / CHAIN, 128.0 * n * 16 * CHAIN / per);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  for (int n : {32, 64, 128, 256}) {
    run<1, 0>(n, d);
    run<16, 0>(n, d);
    run<64, 0>(n, d);
  }
  for (int n : {32, 64, 128}) {
    run<16, 1>(n, d);
    run<64, 1>(n, d);
  }
  run<16, 1, 4>(32, d);
  run<16, 1, 8>(32, d);
  run<16, 1, 16>(32, d);
  run<16, 0, 16>(128, d);
  return 0;
}

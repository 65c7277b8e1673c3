// Developer probe (not part of the product): the attention's per-head MMA
// pattern in isolation, one CTA per SM, one thread issuing, timed from the
// first issue to the commit's mbarrier completion.
//   S  : SS, A = Q (128 x 16 K-major SW128), B = keys (N x 16 K-major SW128), dh / 16 steps
//   PV : TS, A = P (TMEM), B = V (16 keys x dh, MN-major SW128 rows of 64), N_S / 16 steps
//   PVk: TS, B K-major (V^T staged), same shape
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2212_11296_b200/csrc scripts/mma_probe2.cu -o /tmp/mma_probe2
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace vqb;

// mode 0: S (SS, N=ns, K-steps=ks); 1: PV MN-major B (N=n, K-steps=ks); 2: PV K-major B;
// 3: SS with MN-major B (N=n)
template <int mode, int ks>
__global__ void __launch_bounds__(128, 1) k_probe(int n, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t sb = tc::smem_u32(smem);
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const bool leader = tc::elect_one();
    uint32_t idesc = tc::make_idesc_bf16(128, n);
    if (mode == 1 || mode == 3) idesc |= 1u << 16;
    const uint64_t da = tc::make_desc_sw128(sb);
    const uint64_t db = tc::make_desc_sw128(sb + 16384);
    uint32_t ph = 0;
    long long t0 = 0;
    for (int r = 0; r <= reps; ++r) {
      if (r == 1) t0 = clock64();
      if (leader) {
#pragma unroll
        for (int k = 0; k < ks; ++k) {
          if (mode == 0)
            tc::mma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, k != 0);
          else if (mode == 1)
            tc::mma_bf16_ts(tmem + 384, tmem + 8u * k, db + 128u * k, idesc, k != 0);
          else if (mode == 2)
            tc::mma_bf16_ts(tmem + 384, tmem + 8u * k, db + 2u * (k & 3) + 64u * (k >> 2), idesc,
                            k != 0);
          else if (mode == 3)
            tc::mma_bf16(tmem + 384, da + 2 * (k & 3), db + 128u * k, idesc, k != 0);
          else if (mode == 4)  // two independent accumulators (even / odd steps)
            tc::mma_bf16_ts(tmem + 384 + 64u * (k & 1), tmem + 8u * k, db + 128u * k, idesc,
                            k >= 2);
          else if (mode == 5)  // four independent accumulators
            tc::mma_bf16_ts(tmem + 256 + 64u * (k & 3), tmem + 8u * k, db + 128u * k, idesc,
                            k >= 4);
          else  // mode 6: a PV chain followed by an independent 2-step S chain
            tc::mma_bf16_ts(tmem + 384, tmem + 8u * k, db + 128u * k, idesc, k != 0);
        }
        if (mode == 6) {
          const uint32_t is = tc::make_idesc_bf16(128, 160);
          tc::mma_bf16(tmem + 200, da, db, is, 0);
          tc::mma_bf16(tmem + 200, da + 2, db + 2, is, 1);
        }
        tc::mma_commit(&bar);
      }
      __syncwarp();
      tc::mbar_wait(&bar, ph);
      ph ^= 1;
    }
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

template <int mode, int ks>
void run(const char* name, int n, unsigned long long* d) {
  const int smem = 98304 + 1024, reps = 200;
  cudaFuncSetAttribute(k_probe<mode, ks>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_probe<mode, ks><<<148, 128, smem>>>(n, reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / reps;
  printf("%-28s N=%3d steps %2d: %8.1f cycles per chain (issue->commit), %6.1f per MMA\n", name,
         n, ks, per, per / ks);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  run<0, 2>("S   SS K-major", 64, d);
  run<0, 2>("S   SS K-major", 160, d);
  run<0, 2>("S   SS K-major", 192, d);
  run<0, 4>("S   SS K-major", 160, d);
  run<1, 1>("PV  TS MN-major B", 32, d);
  run<1, 4>("PV  TS MN-major B", 32, d);
  run<1, 10>("PV  TS MN-major B", 32, d);
  run<1, 12>("PV  TS MN-major B", 32, d);
  run<1, 12>("PV  TS MN-major B", 64, d);
  run<2, 12>("PV  TS K-major B", 32, d);
  run<3, 12>("PV  SS MN-major B", 32, d);
  run<4, 12>("PV  TS 2 accumulators", 32, d);
  run<5, 12>("PV  TS 4 accumulators", 32, d);
  run<6, 10>("PV(10) then S(2) indep.", 32, d);
  run<6, 12>("PV(12) then S(2) indep.", 32, d);
  return 0;
}

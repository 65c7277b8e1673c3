// Developer probe (not part of the product): warp-level mma.sync
// m16n8k16 bf16 -> fp32 throughput per SM on sm_100a (independent
// accumulator chains per warp), and MUFU ex2 throughput.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/hmma_probe.cu -o scripts/_hmma_probe
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int CH>
__global__ void k_hmma(int reps, float* out) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3f803f80u ^ (threadIdx.x + i);
  for (int i = 0; i < 2; ++i) b[i] = 0x3f803f80u ^ (threadIdx.x * 3 + i);
  float acc[CH][4] = {};
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < CH; ++c) mma16816(acc[c], a, b);
  }
  float s = 0.f;
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ex2(int reps, float* out) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* o;
  cudaMalloc(&o, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20000;
  for (int warps : {4, 8, 16, 32}) {
    k_hmma<8><<<148 * 2, 32 * warps>>>(10, o);
    cudaEventRecord(e0);
    k_hmma<8><<<148 * 2, 32 * warps>>>(reps, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * 8 * 16 * 8.0 * reps * warps * 148 * 2;
    printf("mma.sync m16n8k16 bf16: %2d warps x 2 CTAs/SM: %7.1f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int warps : {8, 16, 32}) {
    k_ex2<<<148 * 2, 32 * warps>>>(10, o);
    cudaEventRecord(e0);
    k_ex2<<<148 * 2, 32 * warps>>>(reps, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double n = 8.0 * reps * 32 * warps * 148 * 2;
    printf("ex2.approx: %2d warps x 2 CTAs/SM: %7.2f Tex2/s (%5.1f per clk per SM at 1.965 GHz)\n", warps,
           n / ms / 1e9, n / ms / 1e9 * 1e12 / 148 / 1.965e9);
  }
  return 0;
}

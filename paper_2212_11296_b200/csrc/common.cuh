// Shared device helpers for the local-energy kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

#define VQB_EMPTY_KEY 0xFFFFFFFFFFFFFFFFull
#define VQB_INT_MAX 0x7FFFFFFF

namespace vqb {

typedef __nv_bfloat16 bf16;

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<bf16>(bf16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// Value as the next product will see it: bf16-rounded in bf16 mode.
template <typename T>
__device__ __forceinline__ float operand_round(float v) {
  return to_f<T>(from_f<T>(v));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint64_t hash64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// Reference GELU (tanh form), proj/src/tensor.cpp:126-132, evaluated as
// 0.5 v (1 + tanh u) = v / (1 + e^{-2u}): one ex2 and one reciprocal on the
// MUFU unit instead of tanhf (which made the W1 GEMM's epilogue, not its
// MMAs, the bottleneck), and no cancellation in 1 + tanh u for u << 0
// (relative error a few ulp everywhere; e^{-2u} = inf gives -0).
__device__ __forceinline__ float gelu_f(float v) {
  const float c = 0.7978845608028654f;
  const float u = c * (v + 0.044715f * v * v * v);
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-2.8853900817779268f * u));  // e^{-2u}
  return __fdividef(v, 1.0f + e);
}

// Dynamic shared-memory opt-in for `fn` on the CURRENT device. The attribute
// is a per-device setting, so it is tracked per (kernel, device): a process
// that drives several GPUs (one host thread per device) opts in on each of
// them. Thread-safe; a failure throws instead of surfacing later as a launch
// error.
inline void smem_optin(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) throw std::runtime_error("cudaGetDevice failed");
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{fn, dev}];
  if (have >= bytes) return;
  const cudaError_t e =
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e != cudaSuccess)
    throw std::runtime_error("shared-memory opt-in of " + std::to_string(bytes) +
                             " bytes failed: " + cudaGetErrorString(e));
  have = bytes;
}

// Largest dynamic shared memory one CTA may opt in to on the current device.
inline size_t smem_optin_limit() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return 227 * 1024;
  return size_t(v);
}

}  // namespace vqb

// Kernel-level test hooks (include/vqnqs_b200_debug.h).
#include <cmath>
#include <cstdio>
#include <vector>
#include <cstring>

#include "../../include/vqnqs_b200_debug.h"
#include "common.cuh"
#include "simt_kernels.cuh"
#include "tc_kernels.cuh"

using namespace vqb;

extern "C" int vqnqs_debug_gemm_bf16(int64_t M, int N, int K, const void* A, const void* WT,
                                     const void* W, const float* bias, void* out,
                                     const float* resid, int epi, int use_tc) {
  int64_t* dM = nullptr;
  if (cudaMalloc(&dM, 8) != cudaSuccess) return 6;
  cudaMemcpy(dM, &M, 8, cudaMemcpyHostToDevice);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (use_tc) {
    tc_gemm(dM, M, N, K, A, K, nullptr, WT, bias, out, N, epi, resid, N, nullptr, 0, sms);
  } else {
    const int64_t tiles = ((M + 63) / 64) * ((N + 63) / 64);
    const int grid = int(std::min<int64_t>(tiles, sms * 8));
    const bf16* a = static_cast<const bf16*>(A);
    const bf16* w = static_cast<const bf16*>(W);
    if (epi == EPI_STORE)
      k_gemm_simt<bf16, EPI_STORE><<<grid, 256>>>(dM, N, K, a, K, nullptr, w, bias, out, N, resid,
                                                  N, nullptr);
    else if (epi == EPI_GELU)
      k_gemm_simt<bf16, EPI_GELU><<<grid, 256>>>(dM, N, K, a, K, nullptr, w, bias, out, N, resid,
                                                 N, nullptr);
    else
      k_gemm_simt<bf16, EPI_RESID><<<grid, 256>>>(dM, N, K, a, K, nullptr, w, bias, out, N, resid,
                                                  N, nullptr);
  }
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(dM);
  return e == cudaSuccess ? 0 : 6;
}

extern "C" int vqnqs_debug_vq(int64_t M, int d, const float* x, const float* cb32, int Q,
                              int32_t* code, int use_tc, unsigned long long* n_rescored) {
  int64_t* dM = nullptr;
  if (cudaMalloc(&dM, 8) != cudaSuccess) return 6;
  cudaMemcpy(dM, &M, 8, cudaMemcpyHostToDevice);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<float> h(size_t(Q) * d);
  cudaMemcpy(h.data(), cb32, h.size() * 4, cudaMemcpyDeviceToHost);
  std::vector<float> wn2(Q);
  std::vector<uint16_t> hb(h.size());
  double wmax = 0;
  for (int j = 0; j < Q; ++j) {
    double a = 0;
    for (int c = 0; c < d; ++c) a += double(h[size_t(j) * d + c]) * h[size_t(j) * d + c];
    wn2[j] = float(a);
    wmax = std::max(wmax, std::sqrt(a));
  }
  for (size_t i = 0; i < h.size(); ++i) {
    uint32_t u;
    std::memcpy(&u, &h[i], 4);
    hb[i] = uint16_t(u >> 16);  // cb assumed bf16-exact
  }
  float* dwn2 = nullptr;
  void* dcb = nullptr;
  cudaMalloc(&dwn2, Q * 4);
  cudaMalloc(&dcb, hb.size() * 2);
  cudaMemcpy(dwn2, wn2.data(), Q * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dcb, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  if (use_tc) {
    bf16 *xh = nullptr, *xl = nullptr;
    float *xn2 = nullptr, *rr2 = nullptr;
    cudaMalloc(&xh, size_t(M) * d * 2);
    cudaMalloc(&xl, size_t(M) * d * 2);
    cudaMalloc(&xn2, size_t(M) * 4);
    cudaMalloc(&rr2, size_t(M) * 4);
    k_vq_prep<<<sms * 4, 256>>>(dM, d, x, xh, xl, xn2, rr2);
    const CUtensorMap tmB = make_tmap_bf16(dcb, uint64_t(Q), uint64_t(d), 256);
    VqScratch vqs;
    tc_vq(dM, M, d, xh, xl, xn2, rr2, tmB, cb32, dwn2, float(wmax * (1 + 1e-6)), Q, code,
          n_rescored, vqs, 0, sms);
    cudaDeviceSynchronize();
    vqs.release();
    cudaFree(xh);
    cudaFree(xl);
    cudaFree(xn2);
    cudaFree(rr2);
  } else {
    const int LOCS = d > 384 ? 32 : 64;
    const size_t vsmem = (size_t(LOCS) * (d + 1) + 32 * size_t(d + 1) + 2 * 256) * 4;
    if (LOCS == 64) {
      cudaFuncSetAttribute(k_vq<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(vsmem));
      k_vq<64><<<sms * 4, 256, vsmem>>>(dM, d, x, cb32, Q, code);
    } else {
      cudaFuncSetAttribute(k_vq<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(vsmem));
      k_vq<32><<<sms * 4, 256, vsmem>>>(dM, d, x, cb32, Q, code);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "vqnqs_debug_vq: %s\n", cudaGetErrorString(e));
    return 7;
  }
  e = cudaDeviceSynchronize();
  cudaFree(dM);
  cudaFree(dwn2);
  cudaFree(dcb);
  return e == cudaSuccess ? 0 : 6;
}

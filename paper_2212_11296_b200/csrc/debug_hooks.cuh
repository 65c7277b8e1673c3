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
  const VqCodebook pc = prepare_codebook(h.data(), Q, d);
  const std::vector<float>& wn2 = pc.wn2;
  const std::vector<uint16_t>& hb = pc.bf;
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
    tc_vq(dM, M, d, xh, xl, xn2, rr2, tmB, cb32, dwn2, float(pc.wmax), float(pc.werr), Q, code,
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
      smem_optin(reinterpret_cast<const void*>(k_vq<64>), vsmem);
      k_vq<64><<<sms * 4, 256, vsmem>>>(dM, d, d, x, cb32, Q, code, 1);
    } else {
      smem_optin(reinterpret_cast<const void*>(k_vq<32>), vsmem);
      k_vq<32><<<sms * 4, 256, vsmem>>>(dM, d, d, x, cb32, Q, code, 1);
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

// The tcgen05 gathered causal attention (k_tc_attention) on an explicit
// location layout, with the same tile packing and per-layer tile tables the
// engine builds (k_build_tiles, k_tile_info). Device pointers:
//   K[S], row_t1[S*R1] (first changed token, -1 for the base row),
//   row_perm[S*R1] (active-layout row order), row_aoff[S*R1] (layout offset
//   of a row's first active location within its sample), act_off[S],
//   I[M] (location -> sample-local unique row), Uoff[S], qkv [U x 3d] bf16.
// Outputs: xh, xl [M x d] bf16 (x = xh + xl), xn2 [M], rr2 [M].
extern "C" int vqnqs_debug_tc_attention(int S, int R1, int T, int d, int nh, const int32_t* K,
                                        const int32_t* row_t1, const int32_t* row_perm,
                                        const int64_t* row_aoff, const int64_t* act_off,
                                        int64_t M, const int32_t* I, const int64_t* Uoff,
                                        const void* qkv, void* xh, void* xl, float* xn2,
                                        float* rr2) {
  const int dh = d / nh;
  if (!tc_attn_ok(1, d, dh, T)) return 3;
  const int cap = 256;  // the engine's tile column cap
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t R = int64_t(S) * R1;
  int32_t *lrow = nullptr, *tcnt = nullptr, *ntiles = nullptr;
  int16_t* lpos = nullptr;
  int64_t *toff = nullptr, *dM = nullptr;
  AttnTile* tiles = nullptr;
  uint8_t* tinfo = nullptr;
  const int64_t tcap = R + 16;  // every row its own tile at worst
  cudaMalloc(&lrow, M * 4);
  cudaMalloc(&lpos, M * 2);
  cudaMalloc(&tcnt, S * 4);
  cudaMalloc(&ntiles, 4);
  cudaMalloc(&toff, (S + 1) * 8);
  cudaMalloc(&dM, 8);
  cudaMalloc(&tiles, R * sizeof(AttnTile));
  cudaMalloc(&tinfo, tcap * TINFO_BYTES);
  cudaMemcpy(dM, &M, 8, cudaMemcpyHostToDevice);
  k_enumerate<<<int((R * T + 255) / 256), 256>>>(S, R1, T, K, row_t1, row_aoff, act_off, lrow,
                                                 lpos);
  k_build_tiles<<<(S + 127) / 128, 128>>>(0, S, R1, T, cap, K, row_t1, row_perm, act_off, tcnt,
                                          nullptr, nullptr, tiles, ntiles);
  k_scan<<<1, 1024>>>(S, tcnt, toff, toff + S, 0);
  k_build_tiles<<<(S + 127) / 128, 128>>>(1, S, R1, T, cap, K, row_t1, row_perm, act_off, tcnt, toff,
                                          toff + S, tiles, ntiles);
  k_tile_info<<<sms * 8, 128>>>(tiles, ntiles, R1, T, row_t1, act_off, lrow, lpos, I, Uoff,
                                tinfo);
  const size_t asmem = AttnSmem(T).total + 1024;
  launch_tc_attention(dh, sms, asmem, (cudaStream_t)0, (const uint8_t*)tinfo,
                      (const int32_t*)ntiles, T, d, dh, float(1.0 / std::sqrt(double(dh))),
                      static_cast<const bf16*>(qkv), static_cast<bf16*>(xh),
                      static_cast<bf16*>(xl), xn2, rr2);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) fprintf(stderr, "vqnqs_debug_tc_attention: %s\n", cudaGetErrorString(e));
  cudaFree(lrow);
  cudaFree(lpos);
  cudaFree(tcnt);
  cudaFree(ntiles);
  cudaFree(toff);
  cudaFree(dM);
  cudaFree(tiles);
  cudaFree(tinfo);
  return e == cudaSuccess ? 0 : 6;
}

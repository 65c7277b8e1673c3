// Host launchers for the tcgen05 kernels (bf16 configurations).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "tc_gemm.cuh"
#include "tc_vq.cuh"

namespace vqb {

// tcgen05 GEMM applies when operands are bf16 and K, N tile cleanly.
inline bool tc_gemm_ok(int prec, int N, int K) {
  return prec == 1 && K % 64 == 0 && N % 64 == 0;
}
// The VQ kernel keeps all Q code norms resident in shared memory.
// The certified argmin is exact in both precisions (ties to the lowest
// index, ambiguous rows re-scored in double), so the fp32 engine uses it too.
inline bool tc_vq_ok(int d, int Q) {
  return d % 64 == 0 && Q % 256 == 0 && tcv_smem_bytes(Q) <= smem_optin_limit();
}

template <int BN, int EPI>
inline void launch_tc_gemm_ws(const int64_t* Mp, int64_t Mcap, int N, int K, const bf16* A,
                              int lda, const bf16* WT, const float* bias, void* out, int ldo,
                              const float* resid, int ldr, cudaStream_t st, int sms) {
  const size_t smem = tcw_smem_bytes<BN>();
  smem_optin(reinterpret_cast<const void*>(k_tc_gemm_ws<BN, EPI>), smem);
  const CUtensorMap tmA = make_tmap_bf16(A, uint64_t(Mcap), uint64_t(K), 128, uint64_t(lda));
  const CUtensorMap tmW = make_tmap_bf16(WT, uint64_t(N), uint64_t(K), BN);
  const int64_t tiles = ((Mcap + 127) / 128) * (N / BN);
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(tiles, sms)));
  k_tc_gemm_ws<BN, EPI><<<grid, TCW_THREADS, smem, st>>>(tmA, tmW, Mp, N, K, bias, out, ldo,
                                                         resid, ldr);
}

template <int BN>
inline void launch_tc_gemm_ws_bn(const int64_t* Mp, int64_t Mcap, int N, int K, const bf16* A,
                                 int lda, const bf16* WT, const float* bias, void* out, int ldo,
                                 int epi, const float* resid, int ldr, cudaStream_t st, int sms) {
  if (epi == EPI_STORE)
    launch_tc_gemm_ws<BN, EPI_STORE>(Mp, Mcap, N, K, A, lda, WT, bias, out, ldo, resid, ldr, st,
                                     sms);
  else if (epi == EPI_GELU)
    launch_tc_gemm_ws<BN, EPI_GELU>(Mp, Mcap, N, K, A, lda, WT, bias, out, ldo, resid, ldr, st,
                                    sms);
  else
    launch_tc_gemm_ws<BN, EPI_RESID>(Mp, Mcap, N, K, A, lda, WT, bias, out, ldo, resid, ldr, st,
                                     sms);
}

// W-stationary launcher (tc_gemm.cuh): bf16 epilogues, N % 256 == 0, the
// resident W^T slice within the shared-memory budget.
inline bool tc_gemm_wst_ok(int N, int K, int epi) {
#ifdef VQNQS_NO_WST
  return false;
#endif
  return (epi == EPI_STORE || epi == EPI_GELU) && N % TCS_BN == 0 && K % 64 == 0 &&
         tcs_smem_bytes(K) <= smem_optin_limit();
}
template <int EPI>
inline void launch_tc_gemm_wst(const int64_t* Mp, int64_t Mcap, int N, int K, const bf16* A,
                               int lda, const bf16* WT, const float* bias, void* out, int ldo,
                               cudaStream_t st, int sms) {
  const size_t smem = tcs_smem_bytes(K);
  smem_optin(reinterpret_cast<const void*>(k_tc_gemm_wst<EPI>), smem);
  const CUtensorMap tmA = make_tmap_bf16(A, uint64_t(Mcap), uint64_t(K), 128, uint64_t(lda));
  const CUtensorMap tmW = make_tmap_bf16(WT, uint64_t(N), uint64_t(K), TCS_BN);
  const int tilesN = N / TCS_BN;
  const int64_t tilesM = (Mcap + 127) / 128;
  // a multiple of the slice count, at most one CTA per SM and per (slice, row tile)
  const int per = int(std::max<int64_t>(1, std::min<int64_t>(tilesM, sms / tilesN)));
  k_tc_gemm_wst<EPI><<<per * tilesN, TCW_THREADS, smem, st>>>(tmA, tmW, Mp, N, K, bias,
                                                              static_cast<bf16*>(out), ldo);
}

inline void tc_gemm(const int64_t* Mp, int64_t Mcap, int N, int K, const void* A, int lda,
                    const int32_t* gA, const void* WT, const float* bias, void* out, int ldo,
                    int epi, const float* resid, int ldr, const int64_t* gR, cudaStream_t st,
                    int sms) {
  const bf16* a = static_cast<const bf16*>(A);
  const bf16* w = static_cast<const bf16*>(WT);
  if (gA || gR) throw std::runtime_error("tc_gemm: gathered operands are not supported");
  if (tc_gemm_wst_ok(N, K, epi)) {
    if (epi == EPI_GELU)
      launch_tc_gemm_wst<EPI_GELU>(Mp, Mcap, N, K, a, lda, w, bias, out, ldo, st, sms);
    else
      launch_tc_gemm_wst<EPI_STORE>(Mp, Mcap, N, K, a, lda, w, bias, out, ldo, st, sms);
    return;
  }
  // warp-specialised TMA path (contiguous A rows, identity residual rows)
  if (N % 256 == 0)
    launch_tc_gemm_ws_bn<256>(Mp, Mcap, N, K, a, lda, w, bias, out, ldo, epi, resid, ldr, st, sms);
  else if (N % 128 == 0)
    launch_tc_gemm_ws_bn<128>(Mp, Mcap, N, K, a, lda, w, bias, out, ldo, epi, resid, ldr, st, sms);
  else
    launch_tc_gemm_ws_bn<64>(Mp, Mcap, N, K, a, lda, w, bias, out, ldo, epi, resid, ldr, st, sms);
}

// bf16 copy and |x|^2, |x - bf16(x)|^2 of fp32 attention rows, for the VQ
// operand when the attention ran on CUDA cores (the tcgen05 attention
// epilogue writes these itself). One warp per row.
__global__ void k_vq_prep(const int64_t* __restrict__ Mp, int d, const float* __restrict__ x,
                          bf16* __restrict__ xh, bf16* __restrict__ xl, float* __restrict__ xn2,
                          float* __restrict__ rr2) {
  const int64_t M = *Mp;
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * wpb + (threadIdx.x >> 5); r < M; r += (int64_t)gridDim.x * wpb) {
    float n2 = 0.f, q2 = 0.f;
    for (int c = lane; c < d; c += 32) {
      const float v = x[r * d + c];
      const bf16 h = __float2bfloat16_rn(v);
      const float df = v - __bfloat162float(h);
      const bf16 l = __float2bfloat16_rn(df);
      const float rr = __bfloat162float(l);  // |xl|^2 feeds the certified-argmin bound
      xh[r * d + c] = h;
      xl[r * d + c] = l;
      n2 = fmaf(v, v, n2);
      q2 = fmaf(rr, rr, q2);
    }
    n2 = warp_sum(n2);
    q2 = warp_sum(q2);
    if (lane == 0) {
      xn2[r] = n2;
      rr2[r] = q2;
    }
  }
}

// Host-side codebook preparation for tc_vq: the bf16 operand copy (round to
// nearest), |W_j|^2 of the given codebook, max_j |W_j| and
// max_j |W_j - bf16(W_j)| (the certified bound's two codebook terms).
struct VqCodebook {
  std::vector<uint16_t> bf;
  std::vector<float> wn2;
  double wmax = 0, werr = 0;
};
template <typename T>
inline VqCodebook prepare_codebook(const T* cb, int Q, int d) {
  VqCodebook o;
  o.bf.resize(size_t(Q) * d);
  o.wn2.resize(Q);
  for (int j = 0; j < Q; ++j) {
    double a = 0, e = 0;
    for (int c = 0; c < d; ++c) {
      const double w = double(cb[size_t(j) * d + c]);
      a += w * w;
      float f = float(w);
      uint32_t u;
      std::memcpy(&u, &f, 4);
      if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
      const uint16_t b = uint16_t(u >> 16);
      o.bf[size_t(j) * d + c] = b;
      uint32_t ub = uint32_t(b) << 16;
      float fb;
      std::memcpy(&fb, &ub, 4);
      e += (w - double(fb)) * (w - double(fb));
    }
    o.wn2[j] = float(a);
    o.wmax = std::max(o.wmax, std::sqrt(a));
    o.werr = std::max(o.werr, std::sqrt(e));
  }
  o.wmax *= 1.0 + 1e-6;
  o.werr *= 1.0 + 1e-6;
  return o;
}

// xh/xl: [Mcap x d] bf16 planes; tmB: the layer's codebook tensor map
// (make_tmap_bf16(cbA, Q, d, 256)).
inline void tc_vq(const int64_t* Mp, int64_t Mcap, int d, const bf16* xh, const bf16* xl,
                  const float* xn2, const float* xl2, const CUtensorMap& tmB, const float* cb32,
                  const float* wn2, float wmax, float werr, int Q, int32_t* code,
                  unsigned long long* n_rescored, VqScratch& q, cudaStream_t st, int sms) {
  const size_t smem = tcv_smem_bytes(Q);
  smem_optin(reinterpret_cast<const void*>(k_tc_vq), smem);
  q.ensure(size_t(Mcap));
  cudaMemsetAsync(q.qcount, 0, sizeof(uint32_t), st);
  const CUtensorMap tmA = make_tmap_bf16(xh, uint64_t(Mcap), uint64_t(d), 128);
  const CUtensorMap tmL = make_tmap_bf16(xl, uint64_t(Mcap), uint64_t(d), 128);
  const int64_t tiles = (Mcap + 127) / 128;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(tiles, sms)));
  k_tc_vq<<<grid, TCV_THREADS, smem, st>>>(tmA, tmL, tmB, Mp, d, xn2, xl2, wn2, wmax, werr, Q, code,
                                           q.cand, q.ncand, q.qrows, q.qcount);
  k_vq_rescore<<<sms * 2, 256, 0, st>>>(q.qcount, q.qrows, q.ncand, q.cand, xh, xl, cb32, d, Q,
                                        code, n_rescored);
}

}  // namespace vqb

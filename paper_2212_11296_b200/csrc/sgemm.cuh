// fp32 GEMM on CUDA cores for the score-function gradient (grad.cu): the
// products of autodiff.cpp's matmul nodes (proj/src/autodiff.cpp:332-438,
// forward a W, backward g W^T and a^T g) in fp32 with fp32 accumulation.
//
//   C[M x N] = op(A)[M x K] op(B)[K x N] + beta C     (row-major, leading dims)
//   op(A) = A[m lda + k] or, transposed, A[k lda + m]; op(B) likewise.
//
// 128 x 128 tiles, BK = 8, 256 threads with 8 x 8 outputs each (rows
// 4 ty + {0..3, 64..67}, columns 4 tx + {0..3, 64..67}: conflict-free float4
// shared-memory reads), the next k-block staged through registers while the
// current one is multiplied. Products with few output tiles and a long k
// (the weight gradients a^T g, k = rows) split k over blockIdx.z into a
// workspace, then add the splits in order. Every output is a fixed-order
// sum, so results are deterministic.
#pragma once

#include "common.cuh"

namespace vqb {

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_sgemm(int M, int N, int K, int kchunk,
                                               const float* __restrict__ A, int64_t lda,
                                               const float* __restrict__ B, int64_t ldb,
                                               float* __restrict__ C, int64_t ldc, float beta) {
  constexpr int BM = 128, BN = 128, BK = 8;
  // split z covers k in [z kchunk, (z + 1) kchunk) and writes its own slice
  const int kb = blockIdx.z * kchunk, ke = min(K, kb + kchunk);
  if (gridDim.z > 1) {
    C += (int64_t)blockIdx.z * M * N;
    ldc = N;
    beta = 0.f;
  }
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float ra[4], rb[4];
  // element e (0..1023) of a k-block: A tile entry (k, m), B tile entry (k, n)
  auto a_idx = [&](int e, int& k, int& m) {
    if (TA) { k = e >> 7; m = e & 127; }   // m contiguous in memory
    else { m = e >> 3; k = e & 7; }        // k contiguous
  };
  auto b_idx = [&](int e, int& k, int& n) {
    if (TB) { n = e >> 3; k = e & 7; }     // k contiguous
    else { k = e >> 7; n = e & 127; }      // n contiguous
  };
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int k, m, n;
      a_idx(tid + 256 * q, k, m);
      const int gm = m0 + m, gk = k0 + k;
      ra[q] = (gm < M && gk < ke) ? (TA ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk])
                                 : 0.f;
      b_idx(tid + 256 * q, k, n);
      const int gn = n0 + n, gk2 = k0 + k;
      rb[q] = (gn < N && gk2 < ke) ? (TB ? B[(int64_t)gn * ldb + gk2] : B[(int64_t)gk2 * ldb + gn])
                                  : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int k, m, n;
      a_idx(tid + 256 * q, k, m);
      As[buf][k][m] = ra[q];
      b_idx(tid + 256 * q, k, n);
      Bs[buf][k][n] = rb[q];
    }
  };
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  load(kb);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][4 * ty]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + 4 * ty]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][4 * tx]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + 4 * tx]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? 4 * ty + i : 64 + 4 * ty + i - 4);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? 4 * tx + j : 64 + 4 * tx + j - 4);
      if (n >= N) continue;
      float* c = C + (int64_t)m * ldc + n;
      *c = beta != 0.f ? acc[i][j] + beta * *c : acc[i][j];
    }
  }
}

// C = sum_z W[z] + beta C, z in order
__global__ void k_splitk_sum(int64_t MN, int N, int splits, const float* __restrict__ W,
                             float* __restrict__ C, int64_t ldc, float beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < MN;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int z = 0; z < splits; ++z) v += W[z * MN + i];
    float* c = C + (i / N) * ldc + i % N;
    *c = beta != 0.f ? v + beta * *c : v;
  }
}

// ws: workspace of at least sgemm_ws_floats(M, N, K) floats (may be null
// when that is 0)
inline int sgemm_splits(int64_t M, int64_t N, int64_t K, int sms) {
  const int64_t tiles = ((M + 127) / 128) * ((N + 127) / 128);
  if (tiles >= sms || K < 1024) return 1;
  return int(std::min<int64_t>((2 * sms + tiles - 1) / tiles, K / 512));
}
inline int64_t sgemm_ws_floats(int64_t M, int64_t N, int64_t K, int sms) {
  const int z = sgemm_splits(M, N, K, sms);
  return z > 1 ? int64_t(z) * M * N : 0;
}

inline void sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                  const float* B, int64_t ldb, float* C, int64_t ldc, float beta, float* ws,
                  int sms, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  const int z = sgemm_splits(M, N, K, sms);
  const int kchunk = z > 1 ? int(((K + z - 1) / z + 7) / 8 * 8) : int(K);
  const int zz = z > 1 ? int((K + kchunk - 1) / kchunk) : 1;
  const dim3 grid(unsigned((N + 127) / 128), unsigned((M + 127) / 128), unsigned(zz));
  float* out = zz > 1 ? ws : C;
  const int m = int(M), n = int(N), k = int(K);
#define VQB_SGEMM(a, b) \
  k_sgemm<a, b><<<grid, 256, 0, st>>>(m, n, k, kchunk, A, lda, B, ldb, out, ldc, beta)
  if (!tA && !tB) VQB_SGEMM(false, false);
  else if (tA && !tB) VQB_SGEMM(true, false);
  else if (!tA && tB) VQB_SGEMM(false, true);
  else VQB_SGEMM(true, true);
#undef VQB_SGEMM
  if (zz > 1)
    k_splitk_sum<<<sms * 4, 256, 0, st>>>(M * N, n, zz, ws, C, ldc, beta);
}

}  // namespace vqb

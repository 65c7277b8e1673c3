// CUDA-core kernels for (b) and (c): the portable correctness path and the
// fp32 configurations (c1, c2), where tcgen05 has no exact fp32 mode.
//   k_gemm_simt  per-location linear layers on unique rows, fused epilogues
//   k_attention  gathered causal multi-head attention over active locations
//   k_vq         exact fp32 nearest-codeword search (ties -> lowest index)
#pragma once

#include "common.cuh"

namespace vqb {

enum { EPI_STORE = 0, EPI_GELU = 1, EPI_RESID = 2 };

// C[M x N] = A[M x K] . B[K x N] + bias, B row-major [in x out] like the
// reference's weights (proj/src/tensor.cpp:43-55). A rows may be gathered
// (row gA[m]); EPI_RESID adds resid[gR ? gR[m] : m] in fp32 after the bias,
// matching y = r + (a W + b) (proj/src/dedup.cpp:255-256,262-265).
// Persistent over 64x64 tiles; M is read from device memory.
template <typename TA, int EPI>
__global__ void __launch_bounds__(256) k_gemm_simt(
    const int64_t* __restrict__ Mp, int N, int K, const TA* __restrict__ A, int lda,
    const int32_t* __restrict__ gA, const TA* __restrict__ B, const float* __restrict__ bias,
    void* __restrict__ out, int ldo, const float* __restrict__ resid, int ldr,
    const int64_t* __restrict__ gR) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int64_t M = *Mp;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t tilesM = (M + BM - 1) / BM, tilesN = (N + BN - 1) / BN;
  for (int64_t tile = blockIdx.x; tile < tilesM * tilesN; tile += gridDim.x) {
    const int64_t m0 = (tile / tilesN) * BM;
    const int n0 = int(tile % tilesN) * BN;
    // fp32 products summed per BK block, the block sums added in double:
    // the K-length accumulation error stays at a few fp32 ulps instead of
    // growing with sqrt(K) (K = 4d = 3072 at c5)
    double dacc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dacc[i][j] = 0.0;
    for (int k0 = 0; k0 < K; k0 += BK) {
      float acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = tid + q * 256;
        const int r = e >> 4, kk = e & 15;
        const int64_t m = m0 + r;
        float v = 0.f;
        if (m < M && k0 + kk < K) {
          const int64_t ar = gA ? (int64_t)gA[m] : m;
          v = to_f<TA>(A[ar * lda + k0 + kk]);
        }
        As[kk][r] = v;
        const int kb = e >> 6, n = e & 63;
        Bs[kb][n] =
            (n0 + n < N && k0 + kb < K) ? to_f<TA>(B[(int64_t)(k0 + kb) * N + n0 + n]) : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dacc[i][j] += acc[i][j];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t m = m0 + ty * 4 + i;
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + tx * 4 + j;
        if (n >= N) continue;
        const float v = (float)(dacc[i][j] + (double)bias[n]);
        if (EPI == EPI_STORE) {
          static_cast<TA*>(out)[m * ldo + n] = from_f<TA>(v);
        } else if (EPI == EPI_GELU) {
          static_cast<TA*>(out)[m * ldo + n] = from_f<TA>(gelu_f(v));
        } else {
          const int64_t rr = gR ? gR[m] : m;
          static_cast<float*>(out)[m * ldo + n] = resid[rr * ldr + n] + v;
        }
      }
    }
  }
}

// Gathered causal attention for one (row, head): softmax(q k^T / sqrt(dh),
// causal) v over the row's T positions (proj/src/tensor.cpp:199-231), only
// for the row's active query positions p >= a. Keys/values at positions
// t < a are the base row's (they are identical). q/k/v come from the unique
// QKV table through the location->row index I, never expanded
// (proj/src/dedup.cpp:31-37,128-134). Probabilities are normalised before
// the value product and rounded to the operand type like the reference's
// product operands.
template <typename TA>
__global__ void __launch_bounds__(128) k_attention(
    int R1, int T, int d, int dh, float scale, const int32_t* __restrict__ Ks,
    const int32_t* __restrict__ row_t1, const int64_t* __restrict__ row_aoff,
    const int64_t* __restrict__ act_off, const int32_t* __restrict__ I,
    const int64_t* __restrict__ Uoff, const TA* __restrict__ qkv, float* __restrict__ att) {
  extern __shared__ float sm[];
  const int r = blockIdx.x, h = blockIdx.y;
  const int s = r / R1, k = r % R1;
  if (k >= Ks[s]) return;
  const int a = k == 0 ? 0 : row_t1[r] + 1;
  if (a >= T) return;
  float* Kt = sm;                    // [T][dh+1]
  float* Vt = Kt + T * (dh + 1);     // [T][dh]
  float* P = Vt + T * dh;            // [4][T]
  float* Qw = P + 4 * T;             // [4][dh]
  const int64_t base = act_off[s], rloc = base + row_aoff[r], uo = Uoff[s];
  const int ld = 3 * d;
  for (int idx = threadIdx.x; idx < T * dh; idx += blockDim.x) {
    const int t = idx / dh, e = idx % dh;
    const int64_t loc = t < a ? base + t : rloc + (t - a);
    const int64_t u = uo + I[loc];
    Kt[t * (dh + 1) + e] = to_f<TA>(qkv[u * ld + d + h * dh + e]);
    Vt[t * dh + e] = to_f<TA>(qkv[u * ld + 2 * d + h * dh + e]);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* Pw = P + warp * T;
  float* q = Qw + warp * dh;
  for (int p = a + warp; p < T; p += 4) {
    const int64_t loc = rloc + (p - a);
    const int64_t u = uo + I[loc];
    for (int e = lane; e < dh; e += 32) q[e] = to_f<TA>(qkv[u * ld + h * dh + e]);
    __syncwarp();
    float mx = -INFINITY;
    for (int t = lane; t <= p; t += 32) {
      float sc = 0.f;
      for (int e = 0; e < dh; ++e) sc = fmaf(q[e], Kt[t * (dh + 1) + e], sc);
      sc *= scale;
      Pw[t] = sc;
      mx = fmaxf(mx, sc);
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int t = lane; t <= p; t += 32) {
      const float ev = expf(Pw[t] - mx);
      Pw[t] = ev;
      sum += ev;
    }
    sum = warp_sum(sum);
    for (int t = lane; t <= p; t += 32) Pw[t] = operand_round<TA>(Pw[t] / sum);
    __syncwarp();
    for (int e = lane; e < dh; e += 32) {
      float o = 0.f;
      for (int t = 0; t <= p; ++t) o = fmaf(Pw[t], Vt[t * dh + e], o);
      att[loc * d + h * dh + e] = o;
    }
    __syncwarp();
  }
}

#ifndef VQNQS_ATTQ_UNROLL
#define VQNQS_ATTQ_UNROLL 4
#endif
constexpr int ATTQ_UNROLL = VQNQS_ATTQ_UNROLL;  // K/V fill loads in flight per thread
// four consecutive operand elements as fp32 (16-byte / 8-byte aligned source)
__device__ __forceinline__ float4 load4f(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ float4 load4f(const bf16* p) {
  const uint2 w = *reinterpret_cast<const uint2*>(p);
  return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u),
                     __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u));
}

// The same attention with NQ consecutive queries of the row per warp pass
// (register-blocked: q of the NQ queries in registers, every K element read
// from shared memory once per NQ products, every V element once per NQ
// products, the NQ probabilities of a key as one vector load). Each score,
// exponential, sum and output is formed by the same operations in the same
// order as in k_attention, so the two kernels agree bit for bit.
template <typename TA, int DH, int NQ>
__global__ void __launch_bounds__(128) k_attention_q(
    int R1, int T, int d, float scale, const int32_t* __restrict__ Ks,
    const int32_t* __restrict__ row_t1, const int64_t* __restrict__ row_aoff,
    const int64_t* __restrict__ act_off, const int32_t* __restrict__ I,
    const int64_t* __restrict__ Uoff, const TA* __restrict__ qkv, float* __restrict__ att) {
  extern __shared__ float sm[];
  constexpr int NE = (DH + 31) / 32;  // output elements per lane
  const int r = blockIdx.x, h = blockIdx.y;
  const int s = r / R1, k = r % R1;
  if (k >= Ks[s]) return;
  const int a = k == 0 ? 0 : row_t1[r] + 1;
  if (a >= T) return;
  float* Kt = sm;                  // [T][DH+1]
  float* Vt = Kt + ((T * (DH + 1) + 3) & ~3);  // [T][DH], 16-byte aligned
  float* P = Vt + T * DH;          // [4][T][NQ]
  float* Qs = P + 4 * T * NQ;      // [4][NQ][DH]
  const int64_t base = act_off[s], rloc = base + row_aoff[r], uo = Uoff[s];
  const int ld = 3 * d;
  // K and V of the row's T positions, four elements per load
#pragma unroll ATTQ_UNROLL
  for (int idx = threadIdx.x; idx < T * (DH / 4); idx += blockDim.x) {
    const int t = idx / (DH / 4), e = 4 * (idx % (DH / 4));
    const int64_t loc = t < a ? base + t : rloc + (t - a);
    const TA* src = qkv + (uo + I[loc]) * ld + d + h * DH + e;
    const float4 kq = load4f(src), vq = load4f(src + d);
    float* kr = Kt + t * (DH + 1) + e;
    kr[0] = kq.x;
    kr[1] = kq.y;
    kr[2] = kq.z;
    kr[3] = kq.w;
    *reinterpret_cast<float4*>(Vt + t * DH + e) = vq;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* Pw = P + warp * T * NQ;
  float* Qw = Qs + warp * NQ * DH;
  for (int p0 = a + NQ * warp; p0 < T; p0 += 4 * NQ) {
    const int nq = min(NQ, T - p0);   // live queries p0 .. p0 + nq - 1
    const int pmax = p0 + nq - 1;
    // q of the NQ queries: staged through shared memory, then in registers
    for (int idx = lane; idx < NQ * DH; idx += 32) {
      const int j = idx / DH, e = idx % DH;
      float qv = 0.f;
      if (j < nq) {
        const int64_t u = uo + I[rloc + (p0 + j - a)];
        qv = to_f<TA>(qkv[u * ld + h * DH + e]);
      }
      Qw[idx] = qv;
    }
    __syncwarp();
    float q[NQ][DH];
#pragma unroll
    for (int j = 0; j < NQ; ++j)
#pragma unroll
      for (int e = 0; e < DH; ++e) q[j][e] = Qw[j * DH + e];
    float mx[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) mx[j] = -INFINITY;
    for (int t = lane; t <= pmax; t += 32) {
      float sc[NQ];
#pragma unroll
      for (int j = 0; j < NQ; ++j) sc[j] = 0.f;
      const float* kr = Kt + t * (DH + 1);
#pragma unroll
      for (int e = 0; e < DH; ++e) {
        const float kv = kr[e];
#pragma unroll
        for (int j = 0; j < NQ; ++j) sc[j] = fmaf(q[j][e], kv, sc[j]);
      }
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        sc[j] *= scale;
        Pw[t * NQ + j] = sc[j];
        if (t <= p0 + j) mx[j] = fmaxf(mx[j], sc[j]);
      }
    }
    float sum[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      mx[j] = warp_max(mx[j]);
      sum[j] = 0.f;
    }
    __syncwarp();
    for (int t = lane; t <= pmax; t += 32) {
#pragma unroll
      for (int j = 0; j < NQ; ++j)
        if (t <= p0 + j && j < nq) {
          const float ev = expf(Pw[t * NQ + j] - mx[j]);
          Pw[t * NQ + j] = ev;
          sum[j] += ev;
        }
    }
#pragma unroll
    for (int j = 0; j < NQ; ++j) sum[j] = warp_sum(sum[j]);
    for (int t = lane; t <= pmax; t += 32) {
#pragma unroll
      for (int j = 0; j < NQ; ++j)
        if (t <= p0 + j && j < nq) Pw[t * NQ + j] = operand_round<TA>(Pw[t * NQ + j] / sum[j]);
    }
    __syncwarp();
    // O = P V: lane e (and e + 32) of every live query; keys 0 .. p0 are
    // common to the NQ queries, the last NQ - 1 keys are causal per query
    float o[NQ][NE];
#pragma unroll
    for (int j = 0; j < NQ; ++j)
#pragma unroll
      for (int c = 0; c < NE; ++c) o[j][c] = 0.f;
    if (lane < DH) {
      for (int t = 0; t <= p0; ++t) {
        float pv[NQ];
#pragma unroll
        for (int j = 0; j < NQ; ++j) pv[j] = Pw[t * NQ + j];
#pragma unroll
        for (int c = 0; c < NE; ++c) {
          const float vv = Vt[t * DH + lane + 32 * c];
#pragma unroll
          for (int j = 0; j < NQ; ++j) o[j][c] = fmaf(pv[j], vv, o[j][c]);
        }
      }
      for (int t = p0 + 1; t <= pmax; ++t) {
#pragma unroll
        for (int c = 0; c < NE; ++c) {
          const float vv = Vt[t * DH + lane + 32 * c];
#pragma unroll
          for (int j = 1; j < NQ; ++j)
            if (t <= p0 + j) o[j][c] = fmaf(Pw[t * NQ + j], vv, o[j][c]);
        }
      }
#pragma unroll
      for (int j = 0; j < NQ; ++j)
        if (j < nq) {
          const int64_t loc = rloc + (p0 + j - a);
#pragma unroll
          for (int c = 0; c < NE; ++c) att[loc * d + h * DH + lane + 32 * c] = o[j][c];
        }
    }
    __syncwarp();
  }
}

// Nearest codeword per location and VQ head (vq_apply_rows,
// proj/src/model.cpp:283-319): argmin_j sum_c (x_c - W_jc)^2 in fp32 over one
// head's d columns (row stride ldx), ties to the lowest j; the pick goes to
// code[l * cstride]. With H heads the engine launches once per head with x,
// cb and code offset to that head. LOCS locations per CTA x 32-code chunks
// staged in shared memory.
template <int LOCS>
__global__ void __launch_bounds__(256) k_vq(const int64_t* __restrict__ Mp, int d, int ldx,
                                            const float* __restrict__ att,
                                            const float* __restrict__ cb, int Q,
                                            int32_t* __restrict__ code, int cstride) {
  extern __shared__ float sm[];
  constexpr int G = 256 / LOCS;  // code groups per chunk
  constexpr int CH = 32;         // codes per chunk
  constexpr int PER = CH / G;
  float* X = sm;                          // [LOCS][d+1]
  float* W = X + LOCS * (d + 1);          // [CH][d+1]
  float* rd = W + CH * (d + 1);           // [G][LOCS]
  int* rj = reinterpret_cast<int*>(rd + G * LOCS);
  const int64_t M = *Mp;
  const int tid = threadIdx.x, li = tid % LOCS, jg = tid / LOCS;
  for (int64_t l0 = (int64_t)blockIdx.x * LOCS; l0 < M; l0 += (int64_t)gridDim.x * LOCS) {
    for (int idx = tid; idx < LOCS * d; idx += 256) {
      const int r = idx / d, c = idx % d;
      X[r * (d + 1) + c] = (l0 + r < M) ? att[(l0 + r) * ldx + c] : 0.f;
    }
    float best = INFINITY;
    int bj = 0;
    for (int j0 = 0; j0 < Q; j0 += CH) {
      __syncthreads();
      for (int idx = tid; idx < CH * d; idx += 256) {
        const int j = idx / d, c = idx % d;
        W[j * (d + 1) + c] = (j0 + j < Q) ? cb[(int64_t)(j0 + j) * d + c] : 0.f;
      }
      __syncthreads();
      for (int jj = jg * PER; jj < jg * PER + PER; ++jj) {
        if (j0 + jj >= Q) break;
        const float* xr = X + li * (d + 1);
        const float* wr = W + jj * (d + 1);
        float s2 = 0.f;
        for (int c = 0; c < d; ++c) {
          const float df = xr[c] - wr[c];
          s2 = fmaf(df, df, s2);
        }
        if (s2 < best) {
          best = s2;
          bj = j0 + jj;
        }
      }
    }
    rd[jg * LOCS + li] = best;
    rj[jg * LOCS + li] = bj;
    __syncthreads();
    if (jg == 0 && l0 + li < M) {
      float b = rd[li];
      int j = rj[li];
      for (int q = 1; q < G; ++q) {
        const float v = rd[q * LOCS + li];
        const int vj = rj[q * LOCS + li];
        if (v < b || (v == b && vj < j)) {
          b = v;
          j = vj;
        }
      }
      code[(l0 + li) * cstride] = j;
    }
    __syncthreads();
  }
}

}  // namespace vqb

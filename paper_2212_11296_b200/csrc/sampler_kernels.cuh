// §8(f) rank 1: the autoregressive sampler on the GPU
// (VqTransformer::sample, proj/src/model.cpp:485-525).
//
// The reference re-runs the decoder on the whole prefix at every step. Here
// each step advances every sample by ONE position through all blocks with a
// per-block K/V cache: position t's hidden state depends only on tokens < t
// (causal attention), so the conditional row is the same one the reference
// reads. Per step: embedding -> per block [LN1, QKV GEMM on B rows, cached
// causal attention, VQ, per-code continuation + LN2, W1/GELU, W2 + residual]
// -> LN_f, head, log_softmax (fp64) -> inverse-CDF draw with the reference's
// uniform (drawn on the host in the reference's order: step-major, then
// sample index) -> token and running log-prob.
#pragma once

#include "common.cuh"

namespace vqb {

// x[b] = tok_embed[t == 0 ? BOS : tok[b][t-1]] + pos_embed[t]  (BOS = V)
__global__ void k_dec_embed(int B, int d, int T, int V, int t, const int32_t* __restrict__ tok,
                            const float* __restrict__ tok_embed,
                            const float* __restrict__ pos_embed, float* __restrict__ x) {
  const int b = blockIdx.x;
  if (b >= B) return;
  const int id = t == 0 ? V : tok[(int64_t)b * T + t - 1];
  for (int c = threadIdx.x; c < d; c += blockDim.x)
    x[(int64_t)b * d + c] = tok_embed[(int64_t)id * d + c] + pos_embed[(int64_t)t * d + c];
}

// One warp per (sample, head): append position t's k, v to the cache
// [B][T][d], then softmax(q k_j^T * scale) over j <= t and o = sum_j P_j v_j.
// Products are formed from the stored operands (bf16 in the bf16 configs)
// with fp32 accumulation; in bf16 mode P is rounded to bf16 before the value
// product, where the reference's emulated product boundary rounds.
// Scores: a group of dh/4 lanes takes one key (4 dims per lane, one
// contiguous dh-element row read per group) and reduces with shuffles, so a
// warp scores 128/dh keys per step with coalesced loads.
template <typename TA>
__global__ void k_dec_attention(int B, int d, int nh, int T, int t, float scale,
                                const TA* __restrict__ qkv, TA* __restrict__ Kc,
                                TA* __restrict__ Vc, float* __restrict__ o) {
  extern __shared__ float dsm[];
  const int wpb = blockDim.x >> 5;
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t job = (int64_t)blockIdx.x * wpb + wi;
  if (job >= (int64_t)B * nh) return;
  const int b = (int)(job / nh), h = (int)(job % nh);
  const int dh = d / nh;
  float* q = dsm + wi * (dh + T);
  float* P = q + dh;
  const TA* row = qkv + (int64_t)b * 3 * d;
  TA* kc = Kc + (int64_t)b * T * d + h * dh;
  TA* vc = Vc + (int64_t)b * T * d + h * dh;
  for (int e = lane; e < dh; e += 32) {
    q[e] = to_f<TA>(row[h * dh + e]);
    kc[(int64_t)t * d + e] = row[d + h * dh + e];
    vc[(int64_t)t * d + e] = row[2 * d + h * dh + e];
  }
  __syncwarp();
  float m = -INFINITY;
  const bool grouped = dh % 4 == 0 && dh <= 128 && ((dh / 4) & (dh / 4 - 1)) == 0;
  if (grouped) {
    const int lpk = dh / 4, kpi = 32 / lpk;  // lanes per key, keys per step
    const int sub = lane % lpk, kq = lane / lpk;
    float q4[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) q4[e] = q[sub * 4 + e];
    for (int j0 = 0; j0 <= t; j0 += kpi) {
      const int j = j0 + kq;
      float s = 0.f;
      if (kq < kpi && j <= t) {
        const TA* kj = kc + (int64_t)j * d + sub * 4;
#pragma unroll
        for (int e = 0; e < 4; ++e) s = fmaf(q4[e], to_f<TA>(kj[e]), s);
      }
      for (int o = lpk >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (kq < kpi && j <= t && sub == 0) {
        s *= scale;
        P[j] = s;
        m = fmaxf(m, s);
      }
    }
  } else {
    for (int j = lane; j <= t; j += 32) {
      const TA* kj = kc + (int64_t)j * d;
      float s = 0.f;
      for (int e = 0; e < dh; ++e) s = fmaf(q[e], to_f<TA>(kj[e]), s);
      s *= scale;
      P[j] = s;
      m = fmaxf(m, s);
    }
  }
  m = warp_max(m);
  __syncwarp();
  float sum = 0.f;
  for (int j = lane; j <= t; j += 32) {
    const float e = expf(P[j] - m);
    P[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
  for (int j = lane; j <= t; j += 32) P[j] = to_f<TA>(from_f<TA>(P[j] * inv));
  __syncwarp();
  if (grouped) {
    // values: the same lane groups, 4 dims per lane, keys strided by group,
    // then a shuffle reduction across the groups
    const int lpk = dh / 4, kpi = 32 / lpk;
    const int sub = lane % lpk, kq = lane / lpk;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j = kq; j <= t; j += kpi) {
      const TA* vj = vc + (int64_t)j * d + sub * 4;
      const float pj = P[j];
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] = fmaf(pj, to_f<TA>(vj[e]), acc[e]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      for (int off = lpk; off < 32; off <<= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], off);
    if (kq == 0) {
#pragma unroll
      for (int e = 0; e < 4; ++e) o[(int64_t)b * d + h * dh + sub * 4 + e] = acc[e];
    }
  } else {
    for (int e = lane; e < dh; e += 32) {
      float acc = 0.f;
      for (int j = 0; j <= t; ++j) acc = fmaf(P[j], to_f<TA>(vc[(int64_t)j * d + e]), acc);
      o[(int64_t)b * d + h * dh + e] = acc;
    }
  }
}

__global__ void k_fill_i16(int64_t n, int16_t v, int16_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v;
}

__global__ void k_iota64(int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i;
}

// Inverse-CDF draw of token t (proj/src/model.cpp:503-518), double, in the
// reference's order of the vocabulary; lp accumulates the picked log-prob.
__global__ void k_dec_sample(int B, int T, int V, int t, const double* __restrict__ lpV,
                             const double* __restrict__ u, int32_t* __restrict__ tok,
                             double* __restrict__ lp) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double* row = lpV + (int64_t)b * V;
  const double ub = u[(int64_t)t * B + b];
  double cum = 0.0;
  int picked = -1, last_pos = 0;
  for (int c = 0; c < V; ++c) {
    const double p = exp(row[c]);
    if (p > 0) last_pos = c;
    cum += p;
    if (ub < cum) {
      picked = c;
      break;
    }
  }
  if (picked < 0) picked = last_pos;  // guard against rounding
  tok[(int64_t)b * T + t] = picked;
  lp[b] = (t == 0 ? 0.0 : lp[b]) + row[picked];
}

// detokenize (proj/src/model.cpp:250-261), local_dim 2
__global__ void k_detokenize(int B, int N, int g, int T, const int32_t* __restrict__ tok,
                             uint8_t* __restrict__ cfg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * N) return;
  const int64_t b = i / N;
  const int site = (int)(i % N);
  cfg[i] = (uint8_t)((tok[b * T + site / g] >> (site % g)) & 1);
}

}  // namespace vqb

// the score-function gradient's backward on the GPU.
//
// g = d/dtheta sum_i w_i log P(s_i), the quantity vmc_gradient builds on the
// reference's tape (proj/src/trainer.cpp:213-246: build_log_prob +
// weighted_sum + backward, proj/src/model.cpp:570-603, proj/src/autodiff.cpp)
// with the straight-through VQ surrogate of Graph::vq_quantize
// (autodiff.cpp:536-655: hard picks forward; backward through
// p = softmax(-|x - W_j| / tau)).
//
// The dense decoder over all B x T locations runs forward once with its
// activations kept (fp32 values, double LayerNorm statistics and VQ
// distances), then backward layer by layer: every GEMM-shaped product on
// the fp32 CUDA-core GEMM of sgemm.cuh, the per-row / per-(sample, head)
// work in the kernels below, every reduction over rows in a fixed order (no
// atomics), so the gradient is deterministic. Micro-batches of samples
// accumulate into the same gradient buffers.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "engine.h"
#include "sgemm.cuh"

namespace vqb {
namespace {

#define GCK(x)                                                                            \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      throw RuntimeError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                         __FILE__ + ":" + std::to_string(__LINE__));                      \
  } while (0)

template <typename T>
struct GBuf {
  T* p = nullptr;
  size_t n = 0;
  GBuf() = default;
  GBuf(const GBuf&) = delete;
  GBuf& operator=(const GBuf&) = delete;
  ~GBuf() {
    if (p) cudaFree(p);
  }
  void ensure(size_t want) {
    if (want <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (cudaMalloc(&p, std::max<size_t>(want, 1) * sizeof(T)) != cudaSuccess) {
      p = nullptr;
      throw RuntimeError("device allocation failed (gradient)");
    }
    n = want;
  }
  void zero() {
    if (p) GCK(cudaMemset(p, 0, n * sizeof(T)));
  }
};

// ------------------------------------------------------------------ kernels

// ids / targets (BOS shift, proj/src/model.cpp:570-586) and the embedding sum
__global__ void kg_embed(int T, int d, int V, int g, int n, const uint8_t* __restrict__ cfg,
                         const float* __restrict__ tok_emb, const float* __restrict__ pos_emb,
                         float* __restrict__ x, int* __restrict__ ids, int* __restrict__ tgt) {
  const int64_t r = blockIdx.x;
  const int b = int(r / T), p = int(r % T);
  auto tok = [&](int q) {
    int t = 0;
    for (int j = 0; j < g; ++j)
      if (q * g + j < n) t |= int(cfg[(int64_t)b * n + q * g + j] & 1) << j;
    return t;
  };
  const int id = p == 0 ? V : tok(p - 1);
  if (threadIdx.x == 0) {
    ids[r] = id;
    tgt[r] = tok(p);
  }
  for (int c = threadIdx.x; c < d; c += blockDim.x)
    x[r * d + c] = tok_emb[(int64_t)id * d + c] + pos_emb[(int64_t)p * d + c];
}

// LayerNorm forward (kernels::layer_norm, proj/src/tensor.cpp:57-83), warp per
// row, double statistics
__global__ void kg_ln_fwd(int64_t R, int d, const float* __restrict__ x,
                          const float* __restrict__ gm, const float* __restrict__ bt,
                          float* __restrict__ y, double* __restrict__ mean,
                          double* __restrict__ rstd) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  const float* xr = x + r * d;
  double s = 0.0;
  for (int c = lane; c < d; c += 32) s += xr[c];
  const double mu = warp_sum(s) / d;
  double q = 0.0;
  for (int c = lane; c < d; c += 32) {
    const double t = xr[c] - mu;
    q += t * t;
  }
  const double rs = 1.0 / sqrt(warp_sum(q) / d + 1e-5);
  for (int c = lane; c < d; c += 32) y[r * d + c] = float((xr[c] - mu) * rs * gm[c] + bt[c]);
  if (lane == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

// LayerNorm backward (autodiff.cpp:89-131): out = base + rstd (ghat - mean(ghat)
// - xhat mean(ghat xhat)), ghat = gy * gamma
__global__ void kg_ln_bwd(int64_t R, int d, const float* __restrict__ x,
                          const double* __restrict__ mean, const double* __restrict__ rstd,
                          const float* __restrict__ gm, const float* __restrict__ gy,
                          const float* __restrict__ base, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  const double mu = mean[r], rs = rstd[r];
  double g1 = 0.0, g2 = 0.0;
  for (int c = lane; c < d; c += 32) {
    const double xh = (x[r * d + c] - mu) * rs;
    const double gh = double(gy[r * d + c]) * gm[c];
    g1 += gh;
    g2 += gh * xh;
  }
  g1 = warp_sum(g1) / d;
  g2 = warp_sum(g2) / d;
  for (int c = lane; c < d; c += 32) {
    const double xh = (x[r * d + c] - mu) * rs;
    const double gh = double(gy[r * d + c]) * gm[c];
    out[r * d + c] = float(double(base ? base[r * d + c] : 0.f) + rs * (gh - g1 - xh * g2));
  }
}

// d gamma += sum_r gy xhat, d beta += sum_r gy: row-block partials then a
// fixed-order column sum (deterministic)
__global__ void kg_ln_param_part(int64_t R, int d, int rows_per, const float* __restrict__ x,
                                 const double* __restrict__ mean,
                                 const double* __restrict__ rstd, const float* __restrict__ gy,
                                 float* __restrict__ pg, float* __restrict__ pb) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per, r1 = min(R, r0 + rows_per);
  float sg = 0.f, sb = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    const float g = gy[r * d + c];
    sg += g * float((x[r * d + c] - mean[r]) * rstd[r]);
    sb += g;
  }
  pg[(int64_t)blockIdx.y * d + c] = sg;
  pb[(int64_t)blockIdx.y * d + c] = sb;
}

// out[c] += sum_r A[r, c] (row-block partials first: kg_colsum_part)
__global__ void kg_colsum_part(int64_t R, int N, int lda, int rows_per, const float* __restrict__ A,
                               float* __restrict__ part) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per, r1 = min(R, r0 + rows_per);
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += A[r * lda + c];
  part[(int64_t)blockIdx.y * N + c] = s;
}
__global__ void kg_colsum_final(int nparts, int N, const float* __restrict__ part,
                                float* __restrict__ out, float sign) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  float s = 0.f;
  for (int i = 0; i < nparts; ++i) s += part[(int64_t)i * N + c];
  out[c] += sign * s;
}

__global__ void kg_add_bias(int64_t R, int N, float* __restrict__ y, const float* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < R * N) y[i] += b[i % N];
}

// y = a + b + bias (row broadcast)
__global__ void kg_add3(int64_t R, int N, const float* __restrict__ a, const float* __restrict__ b,
                        const float* __restrict__ bias, float* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < R * N) y[i] = a[i] + (b[i] + bias[i % N]);
}

__device__ __forceinline__ double gelu_d(double v) {
  const double c = 0.7978845608028654;
  return 0.5 * v * (1.0 + tanh(c * (v + 0.044715 * v * v * v)));
}
__device__ __forceinline__ double gelu_grad(double v) {
  const double c = 0.7978845608028654;
  const double th = tanh(c * (v + 0.044715 * v * v * v));
  return 0.5 * (1.0 + th) + 0.5 * v * (1.0 - th * th) * c * (1.0 + 3.0 * 0.044715 * v * v);
}
__global__ void kg_gelu(int64_t n, const float* __restrict__ x, float* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = float(gelu_d(x[i]));
}
__global__ void kg_gelu_bwd(int64_t n, const float* __restrict__ pre, float* __restrict__ g) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) g[i] = float(g[i] * gelu_grad(pre[i]));
}

// causal attention forward per (sample, head) (autodiff.cpp:336-379): the
// probabilities are kept for the backward. One CTA of T threads, thread = row.
constexpr int KG_REG_DH = 32;  // head width up to which a row lives in registers

// Shared-memory layouts are padded (row stride dh + 1, T + 1) so the
// thread-per-query-row loops are bank-conflict free, and the probability tile
// is built in shared memory and stored row-major with coalesced writes. The
// arithmetic (every sum and its order) is that of the straightforward
// per-row loops.
__global__ void kg_attn_fwd(int T, int d, int nh, float sc, const float* __restrict__ qkv,
                            float* __restrict__ P, float* __restrict__ att) {
  extern __shared__ float sm[];
  const int dh = d / nh, dp = dh + 1, tp = T + 1;
  const int b = blockIdx.x / nh, h = blockIdx.x % nh;
  float* qs = sm;
  float* ks = qs + T * dp;
  float* vs = ks + T * dp;
  float* Ps = vs + T * dp;  // Ps[j * tp + r] = P[r][j]
  for (int i = threadIdx.x; i < T * dh; i += blockDim.x) {
    const int r = i / dh, c = i % dh;
    const float* row = qkv + ((int64_t)b * T + r) * 3 * d + h * dh + c;
    qs[r * dp + c] = row[0];
    ks[r * dp + c] = row[d];
    vs[r * dp + c] = row[2 * d];
  }
  __syncthreads();
  const int r = threadIdx.x;
  if (r < T && dh <= KG_REG_DH) {
    // the row's q and its output accumulators in registers (each sum keeps
    // its order: c ascending for a score, j ascending for an output)
    float qr[KG_REG_DH], orow[KG_REG_DH];
#pragma unroll
    for (int c = 0; c < KG_REG_DH; ++c) {
      qr[c] = c < dh ? qs[r * dp + c] : 0.f;
      orow[c] = 0.f;
    }
    float mx = -INFINITY;
    for (int j = 0; j <= r; ++j) {
      float sv = 0.f;
#pragma unroll
      for (int c = 0; c < KG_REG_DH; ++c)
        if (c < dh) sv = fmaf(qr[c], ks[j * dp + c], sv);
      sv *= sc;
      Ps[j * tp + r] = sv;
      mx = fmaxf(mx, sv);
    }
    float sum = 0.f;
    for (int j = 0; j <= r; ++j) {
      const float e = expf(Ps[j * tp + r] - mx);
      Ps[j * tp + r] = e;
      sum += e;
    }
    for (int j = 0; j <= r; ++j) Ps[j * tp + r] /= sum;
    for (int j = r + 1; j < T; ++j) Ps[j * tp + r] = 0.f;
    for (int j = 0; j <= r; ++j) {
      const float pj = Ps[j * tp + r];
#pragma unroll
      for (int c = 0; c < KG_REG_DH; ++c)
        if (c < dh) orow[c] = fmaf(pj, vs[j * dp + c], orow[c]);
    }
#pragma unroll
    for (int c = 0; c < KG_REG_DH; ++c)
      if (c < dh) att[((int64_t)b * T + r) * d + h * dh + c] = orow[c];
  } else if (r < T) {
    float mx = -INFINITY;
    for (int j = 0; j <= r; ++j) {
      float s = 0.f;
      for (int c = 0; c < dh; ++c) s = fmaf(qs[r * dp + c], ks[j * dp + c], s);
      s *= sc;
      Ps[j * tp + r] = s;
      mx = fmaxf(mx, s);
    }
    float sum = 0.f;
    for (int j = 0; j <= r; ++j) {
      const float e = expf(Ps[j * tp + r] - mx);
      Ps[j * tp + r] = e;
      sum += e;
    }
    for (int j = 0; j <= r; ++j) Ps[j * tp + r] /= sum;
    for (int j = r + 1; j < T; ++j) Ps[j * tp + r] = 0.f;
    for (int c = 0; c < dh; ++c) {
      float o = 0.f;
      for (int j = 0; j <= r; ++j) o = fmaf(Ps[j * tp + r], vs[j * dp + c], o);
      att[((int64_t)b * T + r) * d + h * dh + c] = o;
    }
  }
  __syncthreads();
  float* Pg = P + (int64_t)blockIdx.x * T * T;
  for (int i = threadIdx.x; i < T * T; i += blockDim.x) {
    const int rr = i / T, j = i % T;
    Pg[i] = Ps[j * tp + rr];
  }
}

// attention backward per (sample, head) (autodiff.cpp:380-437):
// dP = dO V^T, dS = P (dP - rowsum(dP P)), dV = P^T dO, dQ = dS K sc,
// dK = dS^T Q sc, written into dqkv [R x 3d]
__global__ void kg_attn_bwd(int T, int d, int nh, float sc, const float* __restrict__ qkv,
                            const float* __restrict__ P, const float* __restrict__ dO,
                            float* __restrict__ dqkv) {
  extern __shared__ float sm[];
  const int dh = d / nh, dp = dh + 1, tp = T + 1;
  const int b = blockIdx.x / nh, h = blockIdx.x % nh;
  float* qs = sm;
  float* ks = qs + T * dp;
  float* vs = ks + T * dp;
  float* gs = vs + T * dp;
  float* dS = gs + T * dp;  // dS[r * tp + j]
  float* Ps = dS + T * tp;  // Ps[r * tp + j] = P[r][j]
  for (int i = threadIdx.x; i < T * dh; i += blockDim.x) {
    const int r = i / dh, c = i % dh;
    const int64_t row = (int64_t)b * T + r;
    qs[r * dp + c] = qkv[row * 3 * d + h * dh + c];
    ks[r * dp + c] = qkv[row * 3 * d + d + h * dh + c];
    vs[r * dp + c] = qkv[row * 3 * d + 2 * d + h * dh + c];
    gs[r * dp + c] = dO[row * d + h * dh + c];
  }
  const float* Pg = P + (int64_t)blockIdx.x * T * T;
  for (int i = threadIdx.x; i < T * T; i += blockDim.x) Ps[(i / T) * tp + i % T] = Pg[i];
  __syncthreads();
  const int r = threadIdx.x;
  const bool regs = dh <= KG_REG_DH;
  if (r < T && regs) {
    const float* pr = Ps + r * tp;
    float gr[KG_REG_DH];
#pragma unroll
    for (int c = 0; c < KG_REG_DH; ++c) gr[c] = c < dh ? gs[r * dp + c] : 0.f;
    float dot = 0.f;
    for (int j = 0; j <= r; ++j) {
      float dpv = 0.f;
#pragma unroll
      for (int c = 0; c < KG_REG_DH; ++c)
        if (c < dh) dpv = fmaf(gr[c], vs[j * dp + c], dpv);
      dS[r * tp + j] = dpv;
      dot += dpv * pr[j];
    }
    for (int j = 0; j <= r; ++j) dS[r * tp + j] = pr[j] * (dS[r * tp + j] - dot);
    for (int j = r + 1; j < T; ++j) dS[r * tp + j] = 0.f;
  } else if (r < T) {
    const float* pr = Ps + r * tp;
    float dot = 0.f;
    for (int j = 0; j <= r; ++j) {
      float dpv = 0.f;
      for (int c = 0; c < dh; ++c) dpv = fmaf(gs[r * dp + c], vs[j * dp + c], dpv);
      dS[r * tp + j] = dpv;
      dot += dpv * pr[j];
    }
    for (int j = 0; j <= r; ++j) dS[r * tp + j] = pr[j] * (dS[r * tp + j] - dot);
    for (int j = r + 1; j < T; ++j) dS[r * tp + j] = 0.f;
  }
  __syncthreads();
  if (r < T && regs) {
    // accumulators in registers, each sum in its original order
    const int64_t row = (int64_t)b * T + r;
    float acc[KG_REG_DH];
#pragma unroll
    for (int c = 0; c < KG_REG_DH; ++c) acc[c] = 0.f;
    for (int j = 0; j <= r; ++j) {
      const float sj = dS[r * tp + j];
#pragma unroll
      for (int c = 0; c < KG_REG_DH; ++c)
        if (c < dh) acc[c] = fmaf(sj, ks[j * dp + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < KG_REG_DH; ++c)
      if (c < dh) dqkv[row * 3 * d + h * dh + c] = acc[c] * sc;
    float dv[KG_REG_DH];
#pragma unroll
    for (int c = 0; c < KG_REG_DH; ++c) {
      acc[c] = 0.f;
      dv[c] = 0.f;
    }
    for (int i = r; i < T; ++i) {
      const float si = dS[i * tp + r], pi = Ps[i * tp + r];
#pragma unroll
      for (int c = 0; c < KG_REG_DH; ++c)
        if (c < dh) {
          acc[c] = fmaf(si, qs[i * dp + c], acc[c]);
          dv[c] = fmaf(pi, gs[i * dp + c], dv[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < KG_REG_DH; ++c)
      if (c < dh) {
        dqkv[row * 3 * d + d + h * dh + c] = acc[c] * sc;
        dqkv[row * 3 * d + 2 * d + h * dh + c] = dv[c];
      }
  } else if (r < T) {
    const int64_t row = (int64_t)b * T + r;
    for (int c = 0; c < dh; ++c) {
      float dq = 0.f;
      for (int j = 0; j <= r; ++j) dq = fmaf(dS[r * tp + j], ks[j * dp + c], dq);
      dqkv[row * 3 * d + h * dh + c] = dq * sc;
    }
    // column r: dK_r = sum_i dS[i, r] Q_i sc, dV_r = sum_i P[i, r] dO_i
    for (int c = 0; c < dh; ++c) {
      float dk = 0.f, dv = 0.f;
      for (int i = r; i < T; ++i) {
        dk = fmaf(dS[i * tp + r], qs[i * dp + c], dk);
        dv = fmaf(Ps[i * tp + r], gs[i * dp + c], dv);
      }
      dqkv[row * 3 * d + d + h * dh + c] = dk * sc;
      dqkv[row * 3 * d + 2 * d + h * dh + c] = dv;
    }
  }
}

// VQ forward (autodiff.cpp:536-580, gumbel off): distances in double, c
// ascending; argmin with ties to the lowest index. Warp per row. Keeps
// |x - W_j| for the surrogate backward.
// Block-tiled VQ forward: 32 rows per block (8 warps x 4 rows), codes in
// chunks of 32 staged in shared memory (lane = code, row stride d + 1: no bank
// conflicts), the rows' x in shared memory; per (row, code) the same
// sequential double sum over c as kg_vq_fwd, so results are identical.
constexpr int KGVQ_ROWS = 32;
inline size_t kg_vq_tiled_smem(int d) { return size_t(KGVQ_ROWS) * (2 * d + 1) * sizeof(float); }
__global__ void __launch_bounds__(256) kg_vq_fwd_tiled(int64_t R, int d, int Q,
                                                       const float* __restrict__ x,
                                                       const float* __restrict__ cb,
                                                       float* __restrict__ dist,
                                                       int* __restrict__ pick,
                                                       float* __restrict__ xq) {
  extern __shared__ float sm[];
  float* Xs = sm;                         // [32 rows][d]
  float* Ws = sm + KGVQ_ROWS * d;         // [32 codes][d + 1]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * KGVQ_ROWS;
  for (int i = threadIdx.x; i < KGVQ_ROWS * d; i += blockDim.x) {
    const int64_t r = r0 + i / d;
    Xs[i] = r < R ? x[r0 * d + i] : 0.f;
  }
  double best[4];
  int jb[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    best[k] = 1e300;
    jb[k] = 0x7fffffff;
  }
  for (int j0 = 0; j0 < Q; j0 += 32) {
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * d; i += blockDim.x) {
      const int jj = i / d, c = i % d;
      Ws[jj * (d + 1) + c] = j0 + jj < Q ? cb[(int64_t)(j0 + jj) * d + c] : 0.f;
    }
    __syncthreads();
    const int j = j0 + lane;
    double s2[4] = {0.0, 0.0, 0.0, 0.0};
    const float* wr = Ws + lane * (d + 1);
    for (int c = 0; c < d; ++c) {
      const double wc = double(wr[c]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double df = double(Xs[(w + 8 * k) * d + c]) - wc;
        s2[k] += df * df;
      }
    }
    if (j < Q) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t r = r0 + w + 8 * k;
        if (r < R) {
          dist[r * Q + j] = float(sqrt(s2[k]));
          if (s2[k] < best[k]) {  // j ascending per lane: strict < keeps the lowest index
            best[k] = s2[k];
            jb[k] = j;
          }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double bk = best[k];
    int jk = jb[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, bk, o);
      const int oj = __shfl_xor_sync(0xffffffffu, jk, o);
      if (ob < bk || (ob == bk && oj < jk)) {
        bk = ob;
        jk = oj;
      }
    }
    if (jk == 0x7fffffff) jk = 0;  // no finite distance: the reference's argmin keeps index 0
    const int64_t r = r0 + w + 8 * k;
    if (r < R) {
      if (lane == 0) pick[r] = jk;
      const float* wq = cb + (int64_t)jk * d;
      for (int c = lane; c < d; c += 32) xq[r * d + c] = wq[c];
    }
  }
}

__global__ void kg_vq_fwd(int64_t R, int d, int Q, const float* __restrict__ x,
                          const float* __restrict__ cb, float* __restrict__ dist,
                          int* __restrict__ pick, float* __restrict__ xq) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  const float* xr = x + r * d;
  double best = 1e300;
  int jb = 0x7fffffff;
  for (int j = lane; j < Q; j += 32) {
    const float* wr = cb + (int64_t)j * d;
    double s2 = 0.0;
    for (int c = 0; c < d; ++c) {
      const double df = double(xr[c]) - double(wr[c]);
      s2 += df * df;
    }
    dist[r * Q + j] = float(sqrt(s2));
    if (s2 < best) {
      best = s2;
      jb = j;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oj = __shfl_xor_sync(0xffffffffu, jb, o);
    if (ob < best || (ob == best && oj < jb)) {
      best = ob;
      jb = oj;
    }
  }
  if (jb == 0x7fffffff) jb = 0;  // no finite distance: the reference's argmin keeps index 0
  if (lane == 0) pick[r] = jb;
  const float* w = cb + (int64_t)__shfl_sync(0xffffffffu, jb, 0) * d;
  for (int c = lane; c < d; c += 32) xq[r * d + c] = w[c];
}

// VQ surrogate backward, per row (autodiff.cpp:586-652): p = softmax(-dist/tau),
// a_j = g . W_j (A, precomputed), sbar = sum p a, F_j = p_j (a_j - sbar) /
// (tau dist_j) (0 where dist < 1e-12). Writes Pm, F and rowsum(F).
__global__ void kg_vq_bwd_row(int64_t R, int Q, float tau, const float* __restrict__ dist,
                              const float* __restrict__ A, float* __restrict__ Pm,
                              float* __restrict__ F, float* __restrict__ fsum) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  const float* dr = dist + r * Q;
  double mx = -1e300;
  for (int j = lane; j < Q; j += 32) mx = fmax(mx, -double(dr[j]) / tau);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double sum = 0.0;
  for (int j = lane; j < Q; j += 32) sum += exp(-double(dr[j]) / tau - mx);
  sum = warp_sum(sum);
  double sbar = 0.0;
  for (int j = lane; j < Q; j += 32) {
    const double p = exp(-double(dr[j]) / tau - mx) / sum;
    Pm[r * Q + j] = float(p);
    sbar += p * A[r * Q + j];
  }
  sbar = warp_sum(sbar);
  double fs = 0.0;
  for (int j = lane; j < Q; j += 32) {
    const double dj = dr[j];
    const double f =
        dj < 1e-12 ? 0.0 : double(Pm[r * Q + j]) * (double(A[r * Q + j]) - sbar) / (tau * dj);
    F[r * Q + j] = float(f);
    fs += f;
  }
  fs = warp_sum(fs);
  if (lane == 0) fsum[r] = float(fs);
}

// gx = (F W)_r - rowsum(F)_r x_r   (in place on the F W product)
__global__ void kg_vq_gx(int64_t R, int d, const float* __restrict__ fsum,
                         const float* __restrict__ x, float* __restrict__ gx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < R * d) gx[i] -= fsum[i / d] * x[i];
}

// gW_j -= colsum(F)_j W_j
__global__ void kg_vq_gw_diag(int Q, int d, const float* __restrict__ fcol,
                              const float* __restrict__ cb, float* __restrict__ gw) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < (int64_t)Q * d) gw[i] -= fcol[i / d] * cb[i];
}

// log_softmax over the head logits (with the last-position pad mask), the
// per-sample log-prob, and dlogits = w_b (onehot(target) - softmax)
// (autodiff.cpp:150-164, 485-534). Thread per row for the softmax.
__global__ void kg_head_fwd_bwd(int64_t R, int T, int V, int lastV,
                                const float* __restrict__ logits, const int* __restrict__ tgt,
                                const double* __restrict__ w, double* __restrict__ logp,
                                float* __restrict__ dlog) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int p = int(r % T);
  double lg[16];
  double mx = -1e300;
  for (int c = 0; c < V; ++c) {
    lg[c] = logits[r * V + c];
    if (lastV < V && p == T - 1 && c >= lastV) lg[c] += -1e30;
    mx = fmax(mx, lg[c]);
  }
  double s = 0.0;
  for (int c = 0; c < V; ++c) s += exp(lg[c] - mx);
  const double lse = mx + log(s);
  const double wb = w[r / T];
  for (int c = 0; c < V; ++c) {
    const double y = lg[c] - lse;
    logp[r * V + c] = y;
    dlog[r * V + c] = float((c == tgt[r] ? wb : 0.0) - exp(y) * wb);
  }
}

__global__ void kg_lp_sum(int B, int T, int V, const double* __restrict__ logp,
                          const int* __restrict__ tgt, double* __restrict__ lp) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double s = 0.0;
  for (int p = 0; p < T; ++p) {
    const int64_t r = (int64_t)b * T + p;
    s += logp[r * V + tgt[r]];
  }
  lp[b] = s;
}

// embedding backward, fixed order: tok rows by scanning the ids, positions by
// summing over samples
__global__ void kg_embed_bwd(int64_t R, int T, int d, int ntok, const int* __restrict__ ids,
                             const float* __restrict__ gx, float* __restrict__ gtok,
                             float* __restrict__ gpos) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  const int which = blockIdx.y;  // 0..ntok-1 token rows, then T positions
  float s = 0.f;
  if (which < ntok) {
    for (int64_t r = 0; r < R; ++r)
      if (ids[r] == which) s += gx[r * d + c];
    gtok[(int64_t)which * d + c] += s;
  } else {
    const int p = which - ntok;
    for (int64_t r = p; r < R; r += T) s += gx[r * d + c];
    gpos[(int64_t)p * d + c] += s;
  }
}

}  // namespace

// ------------------------------------------------------------------ engine

class GradImpl {
 public:
  vqnqs_model_desc c{};
  int dev = 0;
  int d, nh, Q, L, V, T, g, N, lastV;
  cudaStream_t st = nullptr;
  int sms = 148;
  std::vector<ParamSpec> spec;
  std::vector<float*> W;  // device copies, parameters() order
  std::vector<float*> Gr;  // gradients, parameters() order
  std::vector<float*> wqkv, bqkv, gwqkv, gbqkv;  // concatenated per block
  // activations (one micro-batch)
  GBuf<float> x_all, h1, qkv, P, att, dist, xq, x1, h2, pre, hf, logits, dlog, tmp, tmp2, tmp4,
      dx, dx1, dqkv, Pm, F, A, part, part2, fsum, fcol, gws;
  GBuf<double> m1, r1, m2, r2, mf, rf, logp, dw, dlp;
  GBuf<int> ids, tgt, pick;
  GBuf<uint8_t> dcfg;

  int pidx(int b, int k) const { return 2 + b * 17 + k; }  // block b, k-th param

  GradImpl(const vqnqs_model_desc& desc, const double* const* params, int n_params, int device)
      : c(desc), dev(device) {
    validate(c);
    spec = param_layout(c);
    if (n_params != int(spec.size())) throw ShapeError("parameter count mismatch");
    if (!c.vq_enabled || c.trailing_half_block || c.vq_heads != 1 || c.phase_enabled)
      throw CapabilityError("GPU gradient: VQ in every block, vq_heads = 1, no phase network");
    GCK(cudaSetDevice(dev));
    GCK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    GCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    d = c.d_hidden;
    nh = c.n_heads;
    Q = c.vq_codebook;
    L = c.n_blocks;
    g = c.group_size;
    V = 1 << g;
    N = c.n_sites;
    T = (N + g - 1) / g;
    lastV = (N % g == 0) ? V : 1 << (N % g);
    if (T > 1024 || V > 16) throw CapabilityError("GPU gradient: T <= 1024, vocab <= 16");
    for (size_t i = 0; i < spec.size(); ++i) {
      const size_t n = size_t(spec[i].rows * spec[i].cols);
      std::vector<float> f(params[i], params[i] + n);
      float *w = nullptr, *gr = nullptr;
      GCK(cudaMalloc(&w, n * 4));
      GCK(cudaMalloc(&gr, n * 4));
      GCK(cudaMemcpy(w, f.data(), n * 4, cudaMemcpyHostToDevice));
      W.push_back(w);
      Gr.push_back(gr);
    }
    for (int b = 0; b < L; ++b) {
      // wq, wk, wv [d x d] -> [d x 3d]
      std::vector<float> cat(size_t(d) * 3 * d), bc(3 * d);
      for (int k = 0; k < 3; ++k) {
        const double* w = params[pidx(b, 2 + 2 * k)];
        const double* bb = params[pidx(b, 3 + 2 * k)];
        for (int r = 0; r < d; ++r)
          for (int cc = 0; cc < d; ++cc) cat[size_t(r) * 3 * d + k * d + cc] = float(w[size_t(r) * d + cc]);
        for (int cc = 0; cc < d; ++cc) bc[k * d + cc] = float(bb[cc]);
      }
      float *w = nullptr, *bb = nullptr, *gw = nullptr, *gb = nullptr;
      GCK(cudaMalloc(&w, cat.size() * 4));
      GCK(cudaMalloc(&bb, bc.size() * 4));
      GCK(cudaMalloc(&gw, cat.size() * 4));
      GCK(cudaMalloc(&gb, bc.size() * 4));
      GCK(cudaMemcpy(w, cat.data(), cat.size() * 4, cudaMemcpyHostToDevice));
      GCK(cudaMemcpy(bb, bc.data(), bc.size() * 4, cudaMemcpyHostToDevice));
      wqkv.push_back(w);
      bqkv.push_back(bb);
      gwqkv.push_back(gw);
      gbqkv.push_back(gb);
    }
  }
  ~GradImpl() {
    cudaSetDevice(dev);
    for (auto* p : W) cudaFree(p);
    for (auto* p : Gr) cudaFree(p);
    for (auto* p : wqkv) cudaFree(p);
    for (auto* p : bqkv) cudaFree(p);
    for (auto* p : gwqkv) cudaFree(p);
    for (auto* p : gbqkv) cudaFree(p);
    if (st) cudaStreamDestroy(st);
  }

  // row-major C = op(A) op(B) (+ beta C) on the fp32 CUDA-core GEMM
  void gemm(bool tA, bool tB, int64_t M, int64_t Nn, int64_t K, const float* A, int64_t lda,
            const float* Bm, int64_t ldb, float* C, int64_t ldc, float beta) {
    gws.ensure(size_t(std::max<int64_t>(1, sgemm_ws_floats(M, Nn, K, sms))));
    sgemm(tA, tB, M, Nn, K, A, lda, Bm, ldb, C, ldc, beta, gws.p, sms, st);
  }
  void colsum(int64_t R, int Nn, int lda, const float* A, float* out, float sign = 1.f) {
    const int rows_per = 256;
    const int parts = int((R + rows_per - 1) / rows_per);
    part.ensure(size_t(parts) * Nn);
    kg_colsum_part<<<dim3((Nn + 127) / 128, parts), 128, 0, st>>>(R, Nn, lda, rows_per, A, part.p);
    kg_colsum_final<<<(Nn + 127) / 128, 128, 0, st>>>(parts, Nn, part.p, out, sign);
  }
  void ln_params(int64_t R, const float* x, const double* mu, const double* rs, const float* gy,
                 float* gg, float* gb) {
    const int rows_per = 256;
    const int parts = int((R + rows_per - 1) / rows_per);
    part.ensure(size_t(parts) * d);
    part2.ensure(size_t(parts) * d);
    kg_ln_param_part<<<dim3((d + 127) / 128, parts), 128, 0, st>>>(R, d, rows_per, x, mu, rs, gy,
                                                                   part.p, part2.p);
    kg_colsum_final<<<(d + 127) / 128, 128, 0, st>>>(parts, d, part.p, gg, 1.f);
    kg_colsum_final<<<(d + 127) / 128, 128, 0, st>>>(parts, d, part2.p, gb, 1.f);
  }

  void micro_batch(const uint8_t* cfg_host, int B, const double* w_host, float tau, double* lp_out) {
    const int64_t R = int64_t(B) * T;
    const int d3 = 3 * d, d4 = 4 * d;
    x_all.ensure(size_t(L + 1) * R * d);
    h1.ensure(size_t(L) * R * d);
    qkv.ensure(size_t(L) * R * d3);
    P.ensure(size_t(L) * B * nh * T * T);
    att.ensure(size_t(L) * R * d);
    dist.ensure(size_t(L) * R * Q);
    xq.ensure(size_t(L) * R * d);
    x1.ensure(size_t(L) * R * d);
    h2.ensure(size_t(L) * R * d);
    pre.ensure(size_t(L) * R * d4);
    m1.ensure(size_t(L) * R);
    r1.ensure(size_t(L) * R);
    m2.ensure(size_t(L) * R);
    r2.ensure(size_t(L) * R);
    pick.ensure(size_t(L) * R);
    hf.ensure(size_t(R) * d);
    mf.ensure(R);
    rf.ensure(R);
    logits.ensure(size_t(R) * V);
    dlog.ensure(size_t(R) * V);
    logp.ensure(size_t(R) * V);
    tmp.ensure(size_t(R) * d);
    tmp4.ensure(size_t(R) * d4);
    tmp2.ensure(size_t(R) * d4);
    dx.ensure(size_t(R) * d);
    dx1.ensure(size_t(R) * d);
    dqkv.ensure(size_t(R) * d3);
    Pm.ensure(size_t(R) * Q);
    F.ensure(size_t(R) * Q);
    A.ensure(size_t(R) * Q);
    fsum.ensure(R);
    fcol.ensure(Q);
    ids.ensure(R);
    tgt.ensure(R);
    dcfg.ensure(size_t(B) * N);
    dw.ensure(B);
    dlp.ensure(B);
    GCK(cudaMemcpyAsync(dcfg.p, cfg_host, size_t(B) * N, cudaMemcpyHostToDevice, st));
    GCK(cudaMemcpyAsync(dw.p, w_host, size_t(B) * 8, cudaMemcpyHostToDevice, st));
    const int rowGrid = int((R + 7) / 8);
    auto ew = [&](int64_t n) { return int((n + 255) / 256); };
    const float sc = float(1.0 / std::sqrt(double(d / nh)));
    const size_t asm_f = (size_t(3) * T * (d / nh + 1) + size_t(T) * (T + 1)) * 4;
    const size_t asm_b = (size_t(4) * T * (d / nh + 1) + 2 * size_t(T) * (T + 1)) * 4;
    GCK(cudaFuncSetAttribute(kg_attn_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, int(asm_f)));
    GCK(cudaFuncSetAttribute(kg_attn_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, int(asm_b)));
    if (kg_vq_tiled_smem(d) <= 200 * 1024)
      GCK(cudaFuncSetAttribute(kg_vq_fwd_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(kg_vq_tiled_smem(d))));
    const int athreads = ((T + 31) / 32) * 32;

    // ---------------- forward
    kg_embed<<<int(R), 64, 0, st>>>(T, d, V, g, N, dcfg.p, W[0], W[1], x_all.p, ids.p, tgt.p);
    for (int b = 0; b < L; ++b) {
      float* xb = x_all.p + size_t(b) * R * d;
      float* xn = x_all.p + size_t(b + 1) * R * d;
      float* h1b = h1.p + size_t(b) * R * d;
      float* qb = qkv.p + size_t(b) * R * d3;
      float* Pb = P.p + size_t(b) * B * nh * T * T;
      float* ab = att.p + size_t(b) * R * d;
      float* db = dist.p + size_t(b) * R * Q;
      float* xqb = xq.p + size_t(b) * R * d;
      float* x1b = x1.p + size_t(b) * R * d;
      float* h2b = h2.p + size_t(b) * R * d;
      float* preb = pre.p + size_t(b) * R * d4;
      kg_ln_fwd<<<rowGrid, 256, 0, st>>>(R, d, xb, W[pidx(b, 0)], W[pidx(b, 1)], h1b,
                                         m1.p + size_t(b) * R, r1.p + size_t(b) * R);
      gemm(false, false, R, d3, d, h1b, d, wqkv[b], d3, qb, d3, 0.f);
      kg_add_bias<<<ew(R * d3), 256, 0, st>>>(R, d3, qb, bqkv[b]);
      kg_attn_fwd<<<B * nh, athreads, asm_f, st>>>(T, d, nh, sc, qb, Pb, ab);
      if (kg_vq_tiled_smem(d) <= 200 * 1024) {
        kg_vq_fwd_tiled<<<int((R + KGVQ_ROWS - 1) / KGVQ_ROWS), 256, kg_vq_tiled_smem(d), st>>>(
            R, d, Q, ab, W[pidx(b, 10)], db, pick.p + size_t(b) * R, xqb);
      } else {
        kg_vq_fwd<<<rowGrid, 256, 0, st>>>(R, d, Q, ab, W[pidx(b, 10)], db,
                                           pick.p + size_t(b) * R, xqb);
      }
      // x1 = x + (xq Wo + bo)
      gemm(false, false, R, d, d, xqb, d, W[pidx(b, 8)], d, tmp.p, d, 0.f);
      kg_add3<<<ew(R * d), 256, 0, st>>>(R, d, xb, tmp.p, W[pidx(b, 9)], x1b);
      kg_ln_fwd<<<rowGrid, 256, 0, st>>>(R, d, x1b, W[pidx(b, 11)], W[pidx(b, 12)], h2b,
                                         m2.p + size_t(b) * R, r2.p + size_t(b) * R);
      gemm(false, false, R, d4, d, h2b, d, W[pidx(b, 13)], d4, preb, d4, 0.f);
      kg_add_bias<<<ew(R * d4), 256, 0, st>>>(R, d4, preb, W[pidx(b, 14)]);
      kg_gelu<<<ew(R * d4), 256, 0, st>>>(R * d4, preb, tmp4.p);
      gemm(false, false, R, d, d4, tmp4.p, d4, W[pidx(b, 15)], d, tmp.p, d, 0.f);
      kg_add3<<<ew(R * d), 256, 0, st>>>(R, d, x1b, tmp.p, W[pidx(b, 16)], xn);
    }
    const int base = 2 + 17 * L;  // lnf_g, lnf_b, head_w, head_b
    float* xL = x_all.p + size_t(L) * R * d;
    kg_ln_fwd<<<rowGrid, 256, 0, st>>>(R, d, xL, W[base], W[base + 1], hf.p, mf.p, rf.p);
    gemm(false, false, R, V, d, hf.p, d, W[base + 2], V, logits.p, V, 0.f);
    kg_add_bias<<<ew(R * V), 256, 0, st>>>(R, V, logits.p, W[base + 3]);
    kg_head_fwd_bwd<<<ew(R), 256, 0, st>>>(R, T, V, lastV, logits.p, tgt.p, dw.p, logp.p, dlog.p);
    kg_lp_sum<<<(B + 127) / 128, 128, 0, st>>>(B, T, V, logp.p, tgt.p, dlp.p);

    // ---------------- backward
    gemm(true, false, d, V, R, hf.p, d, dlog.p, V, Gr[base + 2], V, 1.f);  // dW_head
    colsum(R, V, V, dlog.p, Gr[base + 3]);
    gemm(false, true, R, d, V, dlog.p, V, W[base + 2], V, tmp.p, d, 0.f);  // dhf
    ln_params(R, xL, mf.p, rf.p, tmp.p, Gr[base], Gr[base + 1]);
    kg_ln_bwd<<<rowGrid, 256, 0, st>>>(R, d, xL, mf.p, rf.p, W[base], tmp.p, nullptr, dx.p);
    for (int b = L - 1; b >= 0; --b) {
      float* xb = x_all.p + size_t(b) * R * d;
      float* h1b = h1.p + size_t(b) * R * d;
      float* qb = qkv.p + size_t(b) * R * d3;
      float* Pb = P.p + size_t(b) * B * nh * T * T;
      float* ab = att.p + size_t(b) * R * d;
      float* db = dist.p + size_t(b) * R * Q;
      float* xqb = xq.p + size_t(b) * R * d;
      float* x1b = x1.p + size_t(b) * R * d;
      float* h2b = h2.p + size_t(b) * R * d;
      float* preb = pre.p + size_t(b) * R * d4;
      // x_out = x1 + gelu(pre) W2 + b2
      kg_gelu<<<ew(R * d4), 256, 0, st>>>(R * d4, preb, tmp4.p);
      gemm(true, false, d4, d, R, tmp4.p, d4, dx.p, d, Gr[pidx(b, 15)], d, 1.f);  // dW2
      colsum(R, d, d, dx.p, Gr[pidx(b, 16)]);
      gemm(false, true, R, d4, d, dx.p, d, W[pidx(b, 15)], d, tmp2.p, d4, 0.f);  // d gelu
      kg_gelu_bwd<<<ew(R * d4), 256, 0, st>>>(R * d4, preb, tmp2.p);             // d pre
      gemm(true, false, d, d4, R, h2b, d, tmp2.p, d4, Gr[pidx(b, 13)], d4, 1.f);  // dW1
      colsum(R, d4, d4, tmp2.p, Gr[pidx(b, 14)]);
      gemm(false, true, R, d, d4, tmp2.p, d4, W[pidx(b, 13)], d4, tmp.p, d, 0.f);  // d h2
      ln_params(R, x1b, m2.p + size_t(b) * R, r2.p + size_t(b) * R, tmp.p, Gr[pidx(b, 11)],
                Gr[pidx(b, 12)]);
      kg_ln_bwd<<<rowGrid, 256, 0, st>>>(R, d, x1b, m2.p + size_t(b) * R, r2.p + size_t(b) * R,
                                         W[pidx(b, 11)], tmp.p, dx.p, dx1.p);
      // x1 = x + xq Wo + bo
      gemm(true, false, d, d, R, xqb, d, dx1.p, d, Gr[pidx(b, 8)], d, 1.f);  // dWo
      colsum(R, d, d, dx1.p, Gr[pidx(b, 9)]);
      gemm(false, true, R, d, d, dx1.p, d, W[pidx(b, 8)], d, tmp.p, d, 0.f);  // g = d xq
      // VQ surrogate backward
      const float* cbw = W[pidx(b, 10)];
      float* gcb = Gr[pidx(b, 10)];
      gemm(false, true, R, Q, d, tmp.p, d, cbw, d, A.p, Q, 0.f);  // a = g W^T
      kg_vq_bwd_row<<<rowGrid, 256, 0, st>>>(R, Q, tau, db, A.p, Pm.p, F.p, fsum.p);
      gemm(true, false, Q, d, R, Pm.p, Q, tmp.p, d, gcb, d, 1.f);  // += P^T g
      gemm(true, false, Q, d, R, F.p, Q, ab, d, gcb, d, 1.f);      // += F^T x
      GCK(cudaMemsetAsync(fcol.p, 0, size_t(Q) * 4, st));
      colsum(R, Q, Q, F.p, fcol.p);
      kg_vq_gw_diag<<<ew(int64_t(Q) * d), 256, 0, st>>>(Q, d, fcol.p, cbw, gcb);  // -= colsum(F) W
      gemm(false, false, R, d, Q, F.p, Q, cbw, d, tmp.p, d, 0.f);  // d att = F W - rowsum(F) x
      kg_vq_gx<<<ew(R * d), 256, 0, st>>>(R, d, fsum.p, ab, tmp.p);
      // attention
      kg_attn_bwd<<<B * nh, athreads, asm_b, st>>>(T, d, nh, sc, qb, Pb, tmp.p, dqkv.p);
      gemm(true, false, d, d3, R, h1b, d, dqkv.p, d3, gwqkv[b], d3, 1.f);  // dWqkv
      colsum(R, d3, d3, dqkv.p, gbqkv[b]);
      gemm(false, true, R, d, d3, dqkv.p, d3, wqkv[b], d3, tmp.p, d, 0.f);  // d h1
      ln_params(R, xb, m1.p + size_t(b) * R, r1.p + size_t(b) * R, tmp.p, Gr[pidx(b, 0)],
                Gr[pidx(b, 1)]);
      kg_ln_bwd<<<rowGrid, 256, 0, st>>>(R, d, xb, m1.p + size_t(b) * R, r1.p + size_t(b) * R,
                                         W[pidx(b, 0)], tmp.p, dx1.p, dx.p);
    }
    kg_embed_bwd<<<dim3((d + 127) / 128, V + 1 + T), 128, 0, st>>>(R, T, d, V + 1, ids.p, dx.p,
                                                                   Gr[0], Gr[1]);
    GCK(cudaGetLastError());
    GCK(cudaMemcpyAsync(lp_out, dlp.p, size_t(B) * 8, cudaMemcpyDeviceToHost, st));
    GCK(cudaStreamSynchronize(st));
  }

  void run(const uint8_t* configs, int64_t B, const double* weights, double tau, double* grads,
           double* lp) {
    GCK(cudaSetDevice(dev));
    if (B < 1) throw ConfigError("gradient needs at least one configuration");
    for (size_t i = 0; i < spec.size(); ++i)
      GCK(cudaMemsetAsync(Gr[i], 0, size_t(spec[i].rows * spec[i].cols) * 4, st));
    for (int b = 0; b < L; ++b) {
      GCK(cudaMemsetAsync(gwqkv[b], 0, size_t(d) * 3 * d * 4, st));
      GCK(cudaMemsetAsync(gbqkv[b], 0, size_t(3) * d * 4, st));
    }
    // activations per sample: ~ (L (14 d + 3 d + Q + 4 d + nh T) + ...) T floats
    const double per = double(T) * (double(L) * (22.0 * d + 2.0 * Q + nh * T + 8) + 8.0 * d) * 4;
    const int64_t Bmax = std::max<int64_t>(1, std::min<int64_t>(int64_t(12e9 / per), 4096));
    for (int64_t s0 = 0; s0 < B; s0 += Bmax) {
      const int Bc = int(std::min<int64_t>(Bmax, B - s0));
      micro_batch(configs + s0 * N, Bc, weights + s0, float(tau), lp + s0);
    }
    // gradients to the host in parameters() order (the concatenated QKV
    // gradients split back into wq/bq, wk/bk, wv/bv)
    size_t off = 0;
    std::vector<float> h;
    for (size_t i = 0; i < spec.size(); ++i) {
      const size_t n = size_t(spec[i].rows * spec[i].cols);
      h.resize(n);
      const int bi = i >= 2 ? int((i - 2) / 17) : -1;
      const int k = i >= 2 ? int((i - 2) % 17) : -1;
      if (bi >= 0 && bi < L && k >= 2 && k <= 7) {
        const int which = (k - 2) / 2;
        if ((k - 2) % 2 == 0) {
          std::vector<float> cat(size_t(d) * 3 * d);
          GCK(cudaMemcpy(cat.data(), gwqkv[bi], cat.size() * 4, cudaMemcpyDeviceToHost));
          for (int r = 0; r < d; ++r)
            for (int cc = 0; cc < d; ++cc) h[size_t(r) * d + cc] = cat[size_t(r) * 3 * d + which * d + cc];
        } else {
          std::vector<float> bc(3 * d);
          GCK(cudaMemcpy(bc.data(), gbqkv[bi], bc.size() * 4, cudaMemcpyDeviceToHost));
          for (int cc = 0; cc < d; ++cc) h[cc] = bc[which * d + cc];
        }
      } else {
        GCK(cudaMemcpy(h.data(), Gr[i], n * 4, cudaMemcpyDeviceToHost));
      }
      for (size_t e = 0; e < n; ++e) grads[off + e] = h[e];
      off += n;
    }
  }
};

GradEngine::GradEngine(const vqnqs_model_desc& d, const double* const* params, int n_params,
                       int device)
    : p_(new GradImpl(d, params, n_params, device)) {}
GradEngine::~GradEngine() { delete p_; }
void GradEngine::log_prob_grad(const uint8_t* configs, int64_t B, const double* weights,
                               double vq_tau, double* grads, double* lp) {
  p_->run(configs, B, weights, vq_tau, grads, lp);
}

}  // namespace vqb

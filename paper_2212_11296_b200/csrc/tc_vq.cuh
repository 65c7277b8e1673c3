// (c) Vector quantizer on tcgen05 with a certified argmin
// (vq_apply_rows, proj/src/model.cpp:283-319; ties to the lowest index).
//
// Input per attention-output row x: its two-term bf16 split x = xh + xl + r
// (xh = bf16(x), xl = bf16(x - xh), |r| <= 2^-18 |x|), |x|^2 and |r|^2, all
// written by the attention epilogue. For 128 rows per tile:
//   1. tensor cores accumulate acc_j = xh.W_j + xl.W_j for every codeword
//      (W is bf16-exact: the bf16 configs snap weights to bf16) into up to
//      512 TMEM columns per pass; A/B stream through a cp.async ring;
//   2. D~_j = |W_j|^2 - 2 acc_j differs from D_j = |x - W_j|^2 - |x|^2 by at
//      most E = 2(|r| + d 2^-23 |x|) max_j |W_j| + rounding slack;
//   3. a streaming pass keeps every code with D~_j <= running min + 2E;
//      a single survivor is the answer, otherwise the survivors are
//      re-scored as sum_c ((xh_c + xl_c) - W_jc)^2 in double, c ascending —
//      the reference's own arithmetic (proj/src/model.cpp:298-303) — and the
//      lowest index wins (strict <, :304).
// 512 threads: warp w drains TMEM lanes 32(w%4).. (its rows); the four
// warpgroups split the code columns and merge candidates through smem.
#pragma once

#include "common.cuh"
#include "tc_common.cuh"

namespace vqb {

constexpr int TCV_NC = 512;  // codes per pass (TMEM columns)
constexpr int TCV_A_BYTES = 128 * 128;
constexpr int TCV_STAGE_BYTES = 2 * TCV_A_BYTES + TCV_NC * 128;
constexpr int TCV_STAGES = 2;
constexpr int TCV_CAND = 4;
constexpr int TCV_THREADS = 512;

inline size_t tcv_smem_bytes(int Q) {
  return size_t(TCV_STAGES) * TCV_STAGE_BYTES + 1024 + 256 + size_t(Q) * 4 + 4 * 128 * 24 + 64;
}

__device__ __forceinline__ double vq_exact_d2(const bf16* __restrict__ xh,
                                              const bf16* __restrict__ xl,
                                              const float* __restrict__ wr, int d) {
  double s2 = 0.0;
  for (int c = 0; c < d; c += 8) {
    const uint4 h = *reinterpret_cast<const uint4*>(xh + c);
    const uint4 l = *reinterpret_cast<const uint4*>(xl + c);
    const float4 w0 = *reinterpret_cast<const float4*>(wr + c);
    const float4 w1 = *reinterpret_cast<const float4*>(wr + c + 4);
    const bf16* hb = reinterpret_cast<const bf16*>(&h);
    const bf16* lb = reinterpret_cast<const bf16*>(&l);
    const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double df = (double(__bfloat162float(hb[j])) + double(__bfloat162float(lb[j]))) -
                        double(w[j]);
      s2 += df * df;
    }
  }
  return s2;
}

__global__ void __launch_bounds__(TCV_THREADS, 1) k_tc_vq(
    const int64_t* __restrict__ Mp, int d, const bf16* __restrict__ xh,
    const bf16* __restrict__ xl, const float* __restrict__ xn2g, const float* __restrict__ rr2g,
    const bf16* __restrict__ cbA, const float* __restrict__ cb32,
    const float* __restrict__ wn2_g, float wmax, int Q, int32_t* __restrict__ code,
    unsigned long long* __restrict__ n_rescored) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + TCV_STAGES * TCV_STAGE_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + TCV_STAGES);
  float* wn2 = reinterpret_cast<float*>(smem + TCV_STAGES * TCV_STAGE_BYTES + 256);
  float* red_min = wn2 + Q;                               // [4][128]
  int* red_cnt = reinterpret_cast<int*>(red_min + 512);   // [4][128]
  double* red_d = reinterpret_cast<double*>(red_cnt + 512);  // [4][128]
  int* red_j = reinterpret_cast<int*>(red_d + 512);        // [4][128]
  int* red_jf = red_j + 512;                               // [4][128]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row = tid & 127, part = tid >> 7;
  const int64_t M = *Mp;
  if (tid == 0) {
    for (int s = 0; s < TCV_STAGES; ++s) tc::mbar_init(&mbar[s], 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  for (int j = tid; j < Q; j += TCV_THREADS) wn2[j] = wn2_g[j];
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = tc::smem_u32(smem);
  constexpr uint32_t idesc = tc::make_idesc_bf16(128, 256);
  const int KB = d / 64;
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t g = 0;
  unsigned long long rescored = 0;

  for (int64_t m0 = (int64_t)blockIdx.x * 128; m0 < M; m0 += (int64_t)gridDim.x * 128) {
    const int64_t my = m0 + row;
    const bool live = my < M;
    const float xn = live ? sqrtf(xn2g[my]) : 0.f;
    const float rn = live ? sqrtf(rr2g[my]) : 0.f;
    const float E = 2.f * (rn * wmax + float(d) * 1.2e-7f * xn * wmax) +
                    4e-7f * (wmax * wmax + 2.f * xn * wmax);
    const float w2 = 2.f * E;
    float run_min = INFINITY;
    float cd[TCV_CAND];
    int cj[TCV_CAND];
    int nc = 0;
    bool overflow = false;
    for (int q0 = 0; q0 < Q; q0 += TCV_NC) {
      const int NC = min(TCV_NC, Q - q0);
      auto load = [&](int kb, uint32_t gg) {
        const uint32_t s = gg % TCV_STAGES;
        const uint32_t sa = sbase + s * TCV_STAGE_BYTES, sl = sa + TCV_A_BYTES,
                       sb = sa + 2 * TCV_A_BYTES;
        const int k0 = kb * 64;
#pragma unroll
        for (int i = 0; i < 2; ++i) {  // A hi/lo: 128 rows x 8 chunks each
          const int e = tid + i * TCV_THREADS;
          const int r = e >> 3, c = e & 7;
          const bool ok = m0 + r < M;
          const int64_t off = (ok ? (m0 + r) * d : 0) + k0 + c * 8;
          tc::cp_async16_zfill(sa + tc::sw128_chunk(r, c), xh + off, ok);
          tc::cp_async16_zfill(sl + tc::sw128_chunk(r, c), xl + off, ok);
        }
        for (int e = tid; e < NC * 8; e += TCV_THREADS) {  // B: NC codes x 8 chunks
          const int r = e >> 3, c = e & 7;
          tc::cp_async16(sb + tc::sw128_chunk(r, c), cbA + (int64_t)(q0 + r) * d + k0 + c * 8);
        }
      };
      {
        const uint32_t gg = g;
        if (gg >= TCV_STAGES) tc::mbar_wait(&mbar[gg % TCV_STAGES], ((gg / TCV_STAGES) - 1) & 1);
        load(0, gg);
        tc::cp_async_commit();
      }
      for (int kb = 0; kb < KB; ++kb) {
        if (kb + 1 < KB) {
          const uint32_t gg = g + kb + 1;
          if (gg >= TCV_STAGES) tc::mbar_wait(&mbar[gg % TCV_STAGES], ((gg / TCV_STAGES) - 1) & 1);
          load(kb + 1, gg);
        }
        tc::cp_async_commit();
        tc::cp_async_wait<1>();
        tc::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
          tc::fence_after();
          const uint32_t s = (g + kb) % TCV_STAGES;
          const uint32_t sa = sbase + s * TCV_STAGE_BYTES, sl = sa + TCV_A_BYTES,
                         sb = sa + 2 * TCV_A_BYTES;
          for (int half = 0; half < NC / 256; ++half) {
            const uint32_t bb = sb + half * 256 * 128;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc::mma_bf16(tmem + half * 256, tc::make_desc_sw128(sa + k * 32),
                           tc::make_desc_sw128(bb + k * 32), idesc, (kb | k) != 0);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc::mma_bf16(tmem + half * 256, tc::make_desc_sw128(sl + k * 32),
                           tc::make_desc_sw128(bb + k * 32), idesc, 1u);
          }
          tc::mma_commit(&mbar[s]);
        }
      }
      {
        const uint32_t gl = g + KB - 1;
        tc::mbar_wait(&mbar[gl % TCV_STAGES], (gl / TCV_STAGES) & 1);
      }
      g += KB;
      tc::fence_after();
      // ---- streaming candidate pass: this warpgroup's 32-column chunks
      for (int c0 = part * 32; c0 < NC; c0 += 128) {
        float v[32];
        tc::tmem_ld32(trow + c0, v);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float dt = fmaf(-2.f, v[j], wn2[q0 + c0 + j]);
          if (dt <= run_min + w2) {
            run_min = fminf(run_min, dt);
            int w = 0;
#pragma unroll
            for (int i = 0; i < TCV_CAND; ++i) {
              if (i < nc && cd[i] <= run_min + w2) {
#pragma unroll
                for (int t = 0; t < TCV_CAND; ++t)
                  if (t == w) {
                    cd[t] = cd[i];
                    cj[t] = cj[i];
                  }
                ++w;
              }
            }
            nc = w;
            if (nc < TCV_CAND) {
#pragma unroll
              for (int t = 0; t < TCV_CAND; ++t)
                if (t == nc) {
                  cd[t] = dt;
                  cj[t] = q0 + c0 + j;
                }
              ++nc;
            } else {
              overflow = true;
            }
          }
        }
      }
      tc::fence_before();
      __syncthreads();
    }
    // ---- merge the four warpgroups' candidates
    red_min[part * 128 + row] = run_min;
    __syncthreads();
    const float gmin = fminf(fminf(red_min[row], red_min[128 + row]),
                             fminf(red_min[256 + row], red_min[384 + row]));
    int mine = 0, jfirst = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < TCV_CAND; ++i)
      if (i < nc && cd[i] <= gmin + w2) {
        ++mine;
        jfirst = min(jfirst, cj[i]);
      }
    red_cnt[part * 128 + row] = overflow ? 1000 : mine;
    red_jf[part * 128 + row] = jfirst;
    __syncthreads();
    const int total = red_cnt[row] + red_cnt[128 + row] + red_cnt[256 + row] + red_cnt[384 + row];
    {
      // exact re-scoring when more than one code survives: each warpgroup
      // over its own survivors (or, after an overflow, a quarter of all codes)
      double best = INFINITY;
      int jb = 0x7fffffff;
      if (live && total != 1) {
        const bf16* xhr = xh + my * d;
        const bf16* xlr = xl + my * d;
        if (total < 1000) {
#pragma unroll 1
          for (int i = 0; i < TCV_CAND; ++i)
            if (i < nc && cd[i] <= gmin + w2) {
              const double s2 = vq_exact_d2(xhr, xlr, cb32 + (int64_t)cj[i] * d, d);
              ++rescored;
              if (s2 < best || (s2 == best && cj[i] < jb)) {
                best = s2;
                jb = cj[i];
              }
            }
        } else {
#pragma unroll 1
          for (int j = part; j < Q; j += 4) {
            const double s2 = vq_exact_d2(xhr, xlr, cb32 + (int64_t)j * d, d);
            ++rescored;
            if (s2 < best || (s2 == best && j < jb)) {
              best = s2;
              jb = j;
            }
          }
        }
      }
      red_d[part * 128 + row] = best;
      red_j[part * 128 + row] = jb;
    }
    __syncthreads();
    if (part == 0 && live) {
      int j;
      if (total == 1) {
        j = min(min(red_jf[row], red_jf[128 + row]), min(red_jf[256 + row], red_jf[384 + row]));
      } else {
        double b = red_d[row];
        j = red_j[row];
        for (int p = 1; p < 4; ++p) {
          const double v = red_d[p * 128 + row];
          const int vj = red_j[p * 128 + row];
          if (v < b || (v == b && vj < j)) {
            b = v;
            j = vj;
          }
        }
      }
      code[my] = j;
    }
    __syncthreads();
  }
  if (n_rescored) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rescored += __shfl_xor_sync(0xffffffffu, rescored, o);
    if (lane == 0) atomicAdd(n_rescored, rescored);
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

}  // namespace vqb

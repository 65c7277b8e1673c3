// (c) Vector quantizer on tcgen05 with a certified argmin
// (vq_apply_rows, proj/src/model.cpp:283-319; ties to the lowest index).
//
// For 128 attention-output rows x (fp32) per tile:
//   1. tensor cores compute acc_j = bf16(x) . W_j for every codeword
//      (W is bf16-exact: the bf16 configs snap weights to bf16), Q up to 512
//      codes per pass into 512 TMEM columns;
//   2. the approximate distance D~_j = |W_j|^2 - 2 acc_j differs from the
//      exact D_j = |x - W_j|^2 - |x|^2 by at most E (bf16 rounding of x,
//      measured per row as |x - bf16(x)|, times max_j |W_j|, plus fp32
//      accumulation and rounding slack);
//   3. every code with D~_j <= min D~ + 2E is re-scored as
//      sum_c (x_c - W_jc)^2 in double, c ascending — the reference's own
//      arithmetic (proj/src/model.cpp:298-303) — and the lowest-index minimum
//      wins (strict <, :304).
// So the chosen code is the exact nearest codeword of the fp32 attention
// output, while the distance GEMM runs at bf16 tensor-core rate. Near-ties are the only codes
// re-scored; their count is reported in the profile.
#pragma once

#include "common.cuh"
#include "tc_common.cuh"

namespace vqb {

constexpr int TCV_NC = 512;  // codes per pass (TMEM columns)
constexpr int TCV_STAGE_BYTES = 128 * 128 + TCV_NC * 128;
constexpr int TCV_STAGES = 2;

inline size_t tcv_smem_bytes(int Q) {
  return size_t(TCV_STAGES) * TCV_STAGE_BYTES + 1024 + 256 + 2 * 128 * 4 + size_t(Q) * 4;
}

__global__ void __launch_bounds__(128, 1) k_tc_vq(
    const int64_t* __restrict__ Mp, int d, const float* __restrict__ x,
    const bf16* __restrict__ cbA, const float* __restrict__ cb32,
    const float* __restrict__ wn2_g, float wmax, int Q, int32_t* __restrict__ code,
    unsigned long long* __restrict__ n_rescored) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + TCV_STAGES * TCV_STAGE_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + TCV_STAGES);
  float* xn2 = reinterpret_cast<float*>(smem + TCV_STAGES * TCV_STAGE_BYTES + 256);
  float* xl2 = xn2 + 128;
  float* wn2 = xl2 + 128;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = *Mp;
  if (tid == 0) {
    for (int s = 0; s < TCV_STAGES; ++s) tc::mbar_init(&mbar[s], 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  for (int j = tid; j < Q; j += 128) wn2[j] = wn2_g[j];
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = tc::smem_u32(smem);
  constexpr uint32_t idesc = tc::make_idesc_bf16(128, 256);
  const int KB = d / 64;
  uint32_t g = 0;
  unsigned long long rescored = 0;

  for (int64_t m0 = (int64_t)blockIdx.x * 128; m0 < M; m0 += (int64_t)gridDim.x * 128) {
    xn2[tid] = 0.f;
    xl2[tid] = 0.f;
    double best_d = INFINITY;
    int best_j = 0;
    const int64_t my = m0 + tid;  // epilogue row of this thread (warp w <-> TMEM lanes 32w..)
    for (int q0 = 0; q0 < Q; q0 += TCV_NC) {
      const int NC = min(TCV_NC, Q - q0);
      __syncthreads();
      auto load = [&](int kb, uint32_t gg) {
        const uint32_t s = gg % TCV_STAGES;
        const uint32_t sa = sbase + s * TCV_STAGE_BYTES, sb = sa + 128 * 128;
        const int k0 = kb * 64;
        // A: 128 rows x 64 fp32 -> bf16 (thread: row r = e>>3, chunk c = e&7)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = tid + i * 128;
          const int r = e >> 3, c = e & 7;
          const int64_t m = m0 + r;
          float v[8];
          if (m < M) {
            const float4 a = *reinterpret_cast<const float4*>(x + m * d + k0 + c * 8);
            const float4 b = *reinterpret_cast<const float4*>(x + m * d + k0 + c * 8 + 4);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = 0.f;
          }
          uint32_t pk[4];
          float n2 = 0.f, l2 = 0.f;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            pk[j] = tc::pack_bf16(v[2 * j], v[2 * j + 1]);
            const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&pk[j]);
            const float h0 = __low2float(h), h1 = __high2float(h);
            n2 += v[2 * j] * v[2 * j] + v[2 * j + 1] * v[2 * j + 1];
            l2 += (v[2 * j] - h0) * (v[2 * j] - h0) + (v[2 * j + 1] - h1) * (v[2 * j + 1] - h1);
          }
          tc::st_shared_v4(sa + tc::sw128_chunk(r, c), pk[0], pk[1], pk[2], pk[3]);
          if (q0 == 0) {
            atomicAdd(&xn2[r], n2);
            atomicAdd(&xl2[r], l2);
          }
        }
        // B: NC codes x 64 bf16
        for (int e = tid; e < NC * 8; e += 128) {
          const int r = e >> 3, c = e & 7;
          tc::cp_async16(sb + tc::sw128_chunk(r, c), cbA + (int64_t)(q0 + r) * d + k0 + c * 8);
        }
      };
      for (int kb = 0; kb < KB; ++kb) {
        const uint32_t gg = g + kb;
        if (gg >= TCV_STAGES) tc::mbar_wait(&mbar[gg % TCV_STAGES], ((gg / TCV_STAGES) - 1) & 1);
        load(kb, gg);
        tc::cp_async_commit();
        tc::cp_async_wait<0>();
        tc::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
          tc::fence_after();
          const uint32_t s = gg % TCV_STAGES;
          const uint32_t sa = sbase + s * TCV_STAGE_BYTES, sb = sa + 128 * 128;
          for (int half = 0; half < NC / 256; ++half)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc::mma_bf16(tmem + half * 256, tc::make_desc_sw128(sa + k * 32),
                           tc::make_desc_sw128(sb + half * 256 * 128 + k * 32), idesc,
                           (kb | k) != 0);
          tc::mma_commit(&mbar[s]);
        }
      }
      {
        const uint32_t gl = g + KB - 1;
        tc::mbar_wait(&mbar[gl % TCV_STAGES], (gl / TCV_STAGES) & 1);
      }
      g += KB;
      tc::fence_after();
      __syncthreads();  // xn2 / xl2 complete
      // ---- certified argmin over this pass's NC codes ----
      const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
      const float xn = sqrtf(xn2[tid]), xl = sqrtf(xl2[tid]);
      // |D~ - D| <= 2 (|x_lo| wmax + K 2^-23 |x| wmax) + rounding slack
      const float E = 2.f * (xl * wmax + float(d) * 1.2e-7f * xn * wmax) +
                      4e-7f * (wmax * wmax + 2.f * xn * wmax);
      float dmin = INFINITY;
      for (int c0 = 0; c0 < NC; c0 += 16) {
        float v[16];
        tc::tmem_ld16(trow + c0, v);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) dmin = fminf(dmin, wn2[q0 + c0 + j] - 2.f * v[j]);
      }
      const float thr = dmin + 2.f * E;
      for (int c0 = 0; c0 < NC; c0 += 16) {
        float v[16];
        tc::tmem_ld16(trow + c0, v);
        tc::tmem_wait_ld();
        if (my < M) {
#pragma unroll 1
          for (int j = 0; j < 16; ++j) {
            if (wn2[q0 + c0 + j] - 2.f * v[j] <= thr) {
              const int jj = q0 + c0 + j;
              const float* xr = x + my * d;
              const float* wr = cb32 + (int64_t)jj * d;
              double s2 = 0.0;
              for (int c = 0; c < d; c += 4) {
                const float4 a = *reinterpret_cast<const float4*>(xr + c);
                const float4 w = *reinterpret_cast<const float4*>(wr + c);
                double df = double(a.x) - double(w.x);
                s2 += df * df;
                df = double(a.y) - double(w.y);
                s2 += df * df;
                df = double(a.z) - double(w.z);
                s2 += df * df;
                df = double(a.w) - double(w.w);
                s2 += df * df;
              }
              ++rescored;
              if (s2 < best_d) {
                best_d = s2;
                best_j = jj;
              }
            }
          }
        }
      }
      tc::fence_before();
    }
    if (my < M) code[my] = best_j;
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

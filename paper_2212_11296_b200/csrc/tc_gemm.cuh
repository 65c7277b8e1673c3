// tcgen05 GEMM for the per-location linear layers on unique rows
// (QKV, W1, W2 and the per-code Wo tables; proj/src/dedup.cpp:220-267):
// C = A . W + b with fused epilogues (bf16 store, GELU, fp32 residual add).
// A is bf16 [M x K] row-major, W is supplied transposed (W^T [N x K],
// K-major) so both UMMA operands are K-major.
#pragma once

#include "common.cuh"
#include "tc_common.cuh"
#include "tma.cuh"

namespace vqb {

// Warp-specialised persistent kernel: warp 0 issues TMA for A [128 x 64] and W^T [BN x 64]
// K-blocks into a 4-stage ring, warp 1 issues tcgen05.mma into one of two
// BN-column TMEM accumulators, warps 2-9 (two warpgroups, BN/2 columns each)
// drain the other accumulator through the fused epilogue, so loads, MMAs and
// epilogues of consecutive tiles overlap. The epilogue stages 64-column
// slabs of its 32 rows in a warp-private shared tile and writes (and, for the
// residual epilogue, reads) whole 128/256-byte row segments.
constexpr int TCW_THREADS = 320;
constexpr int TCW_STG_PITCH = 68;  // floats per staged row (64 + 4: conflict-free 16-B writes)
constexpr uint32_t TCW_STG_BYTES = 8 * 32 * TCW_STG_PITCH * 4;

template <int BN>
constexpr int tcw_stages() {
  return BN >= 256 ? 3 : 4;
}

template <int BN>
constexpr size_t tcw_smem_bytes() {
  return 1024 + size_t(tcw_stages<BN>()) * (128 * 128 + BN * 128) + TCW_STG_BYTES + 256;
}

template <int BN, int EPI>
__global__ void __launch_bounds__(TCW_THREADS, 1) k_tc_gemm_ws(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
    const int64_t* __restrict__ Mp, int N, int K, const float* __restrict__ bias,
    void* __restrict__ out, int ldo, const float* __restrict__ resid, int ldr) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  constexpr int TCW_STAGES = tcw_stages<BN>();
  constexpr uint32_t A_BYTES = 128 * 128, B_BYTES = BN * 128, STAGE = A_BYTES + B_BYTES;
  float* stg_all = reinterpret_cast<float*>(smem + TCW_STAGES * STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TCW_STAGES * STAGE + TCW_STG_BYTES);
  uint64_t* empty = full + TCW_STAGES;
  uint64_t* acc_full = empty + TCW_STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = *Mp;
  const int64_t tilesM = (M + 127) / 128;
  const int tilesN = N / BN;
  const int64_t n_tiles = tilesM * tilesN;
  const int KB = K / 64;
  if (tid == 0) {
    for (int s = 0; s < TCW_STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], 8);
    }
    tc::mbar_fence_init();
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmW);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * BN < 32 ? 32 : 2 * BN);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = tc::smem_u32(smem);
  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int m0 = int((t / tilesN) * 128), n0 = int(t % tilesN) * BN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const uint32_t s = it % TCW_STAGES;
          if (it >= TCW_STAGES) tc::mbar_wait(&empty[s], ((it / TCW_STAGES) - 1) & 1);
          const uint32_t sa = sbase + s * STAGE;
          const uint32_t fb = tc::smem_u32(&full[s]);
          tc::mbar_expect_tx(fb, STAGE);
          tc::tma_load_2d(sa, &tmA, kb * 64, m0, fb);
          tc::tma_load_2d(sa + A_BYTES, &tmW, kb * 64, n0, fb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::make_idesc_bf16(128, BN);
      uint32_t it = 0, acc = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++acc) {
        const uint32_t b = acc & 1;
        if (acc >= 2) tc::mbar_wait(&acc_empty[b], ((acc >> 1) - 1) & 1);
        tc::fence_after();
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const uint32_t s = it % TCW_STAGES;
          tc::mbar_wait(&full[s], (it / TCW_STAGES) & 1);
          tc::fence_after();
          const uint32_t sa = sbase + s * STAGE;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc::mma_bf16(tmem + b * BN, tc::make_desc_sw128(sa + k * 32),
                         tc::make_desc_sw128(sa + A_BYTES + k * 32), idesc, (kb | k) != 0);
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&acc_full[b]);
      }
    }
  } else {
    const int part = (warp - 2) >> 2;  // columns [part*BN/2, part*BN/2 + BN/2)
    const int q0 = (warp & 3) * 32;     // this warp's TMEM lanes = tile rows q0..q0+31
    const uint32_t trow = tmem + ((uint32_t)q0 << 16);
    float* stg = stg_all + (warp - 2) * 32 * TCW_STG_PITCH;
    uint32_t acc = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++acc) {
      const uint32_t b = acc & 1;
      const int64_t m0 = (t / tilesN) * 128 + q0;
      const int n0 = int(t % tilesN) * BN;
      tc::mbar_wait(&acc_full[b], (acc >> 1) & 1);
      tc::fence_after();
      constexpr int SLAB = BN / 2 >= 64 ? 64 : BN / 2;  // columns staged at a time
      for (int c0 = part * (BN / 2); c0 < (part + 1) * (BN / 2); c0 += SLAB) {
        // TMEM -> (acc + bias [, GELU]) -> warp-private staging, row = lane
#pragma unroll
        for (int q = 0; q < SLAB / 16; ++q) {
          float v[16];
          tc::tmem_ld16(trow + b * BN + c0 + 16 * q, v);
          tc::tmem_wait_ld();
          const int n = n0 + c0 + 16 * q;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float a = v[j] + bias[n + j];
            if (EPI == EPI_GELU) a = gelu_f(a);
            v[j] = a;
          }
          float4* d4 = reinterpret_cast<float4*>(stg + lane * TCW_STG_PITCH + 16 * q);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        __syncwarp();
        if (EPI == EPI_RESID) {
          // SLAB fp32 per row, 16 B per lane
          constexpr int LPR = SLAB / 4, RPP = 32 / LPR;
#pragma unroll 4
          for (int pass = 0; pass < 32 / RPP; ++pass) {
            const int r = RPP * pass + lane / LPR, cc = (lane % LPR) * 4;
            if (m0 + r < M) {
              const float4 a = *reinterpret_cast<const float4*>(stg + r * TCW_STG_PITCH + cc);
              const int64_t m = m0 + r;
              const float4 rr = *reinterpret_cast<const float4*>(resid + m * ldr + n0 + c0 + cc);
              *reinterpret_cast<float4*>(static_cast<float*>(out) + m * ldo + n0 + c0 + cc) =
                  make_float4(rr.x + a.x, rr.y + a.y, rr.z + a.z, rr.w + a.w);
            }
          }
        } else {
          // SLAB bf16 per row, 16 B (8 values) per lane
          constexpr int LPR = SLAB / 8, RPP = 32 / LPR;
#pragma unroll 4
          for (int pass = 0; pass < 32 / RPP; ++pass) {
            const int r = RPP * pass + lane / LPR, cc = (lane % LPR) * 8;
            if (m0 + r < M) {
              const float4 a = *reinterpret_cast<const float4*>(stg + r * TCW_STG_PITCH + cc);
              const float4 c = *reinterpret_cast<const float4*>(stg + r * TCW_STG_PITCH + cc + 4);
              *reinterpret_cast<uint4*>(static_cast<bf16*>(out) + (m0 + r) * ldo + n0 + c0 + cc) =
                  make_uint4(tc::pack_bf16(a.x, a.y), tc::pack_bf16(a.z, a.w),
                             tc::pack_bf16(c.x, c.y), tc::pack_bf16(c.z, c.w));
            }
          }
        }
        __syncwarp();
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&acc_empty[b]));
    }
  }
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 2 * BN < 32 ? 32 : 2 * BN);
}

// W-stationary variant for the short-K layers (QKV and W1 at d <= 256): the
// streaming kernel above re-reads its W^T slice (BN x K) from L2 for every
// 128-row tile — at K = 256 that is 2/3 of the tile's operand traffic and the
// L2 bandwidth, not HBM or the tensor pipe, bounds it. Here a CTA owns one
// BN = 256 column slice for its whole life: W^T [256 x K] is loaded once
// (K / 64 SW128 blocks, <= 128 KB) and only A [128 x 64] blocks stream through
// a 3-stage ring. bf16 outputs (store / GELU epilogues) are staged as bf16
// (144-byte row pitch), which is what makes the resident slice fit.
constexpr int TCS_BN = 256;
constexpr int TCS_STAGES = 3;
constexpr int TCS_STG_PITCH = 144;  // bytes per staged row: 64 bf16 + 16 (conflict-free 16-B writes)
constexpr uint32_t TCS_STG_BYTES = 8 * 32 * TCS_STG_PITCH;

inline size_t tcs_smem_bytes(int K) {
  return 1024 + size_t(K / 64) * TCS_BN * 128 + size_t(TCS_STAGES) * 128 * 128 + TCS_STG_BYTES + 256;
}

template <int EPI>
__global__ void __launch_bounds__(TCW_THREADS, 1) k_tc_gemm_wst(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
    const int64_t* __restrict__ Mp, int N, int K, const float* __restrict__ bias,
    bf16* __restrict__ out, int ldo) {
  static_assert(EPI == EPI_STORE || EPI == EPI_GELU, "bf16 epilogues only");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  constexpr int BN = TCS_BN;
  constexpr uint32_t A_BYTES = 128 * 128, B_BYTES = BN * 128;
  const int KB = K / 64;
  const uint32_t W_BYTES = (uint32_t)KB * B_BYTES;
  uint8_t* stg_all = smem + W_BYTES + TCS_STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg_all + TCS_STG_BYTES);
  uint64_t* empty = full + TCS_STAGES;
  uint64_t* acc_full = empty + TCS_STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* w_full = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_full + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = *Mp;
  const int64_t tilesM = (M + 127) / 128;
  const int tilesN = N / BN;
  // CTA b: column slice b % tilesN, row tiles b / tilesN, + gridDim / tilesN, ...
  const int n0 = int(blockIdx.x % tilesN) * BN;
  const int64_t mt0 = blockIdx.x / tilesN, mstep = gridDim.x / tilesN;
  if (tid == 0) {
    for (int s = 0; s < TCS_STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], 8);
    }
    tc::mbar_init(w_full, 1);
    tc::mbar_fence_init();
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmW);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * BN);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = tc::smem_u32(smem);
  const uint32_t abase = sbase + W_BYTES;
  if (warp == 0) {
    if (lane == 0 && mt0 < tilesM) {
      const uint32_t wb = tc::smem_u32(w_full);
      tc::mbar_expect_tx(wb, W_BYTES);
      for (int kb = 0; kb < KB; ++kb) tc::tma_load_2d(sbase + kb * B_BYTES, &tmW, kb * 64, n0, wb);
      uint32_t it = 0;
      for (int64_t mt = mt0; mt < tilesM; mt += mstep) {
        const int m0 = int(mt * 128);
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const uint32_t s = it % TCS_STAGES;
          if (it >= TCS_STAGES) tc::mbar_wait(&empty[s], ((it / TCS_STAGES) - 1) & 1);
          const uint32_t fb = tc::smem_u32(&full[s]);
          tc::mbar_expect_tx(fb, A_BYTES);
          tc::tma_load_2d(abase + s * A_BYTES, &tmA, kb * 64, m0, fb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && mt0 < tilesM) {
      constexpr uint32_t idesc = tc::make_idesc_bf16(128, BN);
      tc::mbar_wait(w_full, 0);
      uint32_t it = 0, acc = 0;
      for (int64_t mt = mt0; mt < tilesM; mt += mstep, ++acc) {
        const uint32_t b = acc & 1;
        if (acc >= 2) tc::mbar_wait(&acc_empty[b], ((acc >> 1) - 1) & 1);
        tc::fence_after();
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const uint32_t s = it % TCS_STAGES;
          tc::mbar_wait(&full[s], (it / TCS_STAGES) & 1);
          tc::fence_after();
          const uint32_t sa = abase + s * A_BYTES, sw = sbase + kb * B_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc::mma_bf16(tmem + b * BN, tc::make_desc_sw128(sa + k * 32),
                         tc::make_desc_sw128(sw + k * 32), idesc, (kb | k) != 0);
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&acc_full[b]);
      }
    }
  } else {
    const int part = (warp - 2) >> 2;  // columns [part*128, part*128 + 128)
    const int q0 = (warp & 3) * 32;     // this warp's TMEM lanes = tile rows q0..q0+31
    const uint32_t trow = tmem + ((uint32_t)q0 << 16);
    const uint32_t stg = tc::smem_u32(stg_all) + (uint32_t)(warp - 2) * 32 * TCS_STG_PITCH;
    uint32_t acc = 0;
    for (int64_t mt = mt0; mt < tilesM; mt += mstep, ++acc) {
      const uint32_t b = acc & 1;
      const int64_t m0 = mt * 128 + q0;
      tc::mbar_wait(&acc_full[b], (acc >> 1) & 1);
      tc::fence_after();
      for (int c0 = part * (BN / 2); c0 < (part + 1) * (BN / 2); c0 += 64) {
        // TMEM -> (acc + bias [, GELU]) -> bf16 -> warp-private staging, row = lane
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float v[16];
          tc::tmem_ld16(trow + b * BN + c0 + 16 * q, v);
          tc::tmem_wait_ld();
          const int n = n0 + c0 + 16 * q;
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            float a0 = v[j] + bias[n + j], a1 = v[j + 1] + bias[n + j + 1];
            if (EPI == EPI_GELU) {
              a0 = gelu_f(a0);
              a1 = gelu_f(a1);
            }
            pk[j / 2] = tc::pack_bf16(a0, a1);
          }
          const uint32_t dst = stg + (uint32_t)lane * TCS_STG_PITCH + 32 * q;
          tc::st_shared_v4(dst, pk[0], pk[1], pk[2], pk[3]);
          tc::st_shared_v4(dst + 16, pk[4], pk[5], pk[6], pk[7]);
        }
        __syncwarp();
        // 64 bf16 per row = 128 B: 8 lanes per row, 4 rows per pass
#pragma unroll 4
        for (int pass = 0; pass < 8; ++pass) {
          const int r = 4 * pass + (lane >> 3), cc = (lane & 7) * 8;
          if (m0 + r < M) {
            uint32_t w0, w1, w2, w3;
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                         : "r"(stg + (uint32_t)r * TCS_STG_PITCH + cc * 2));
            *reinterpret_cast<uint4*>(out + (m0 + r) * ldo + n0 + c0 + cc) =
                make_uint4(w0, w1, w2, w3);
          }
        }
        __syncwarp();
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&acc_empty[b]));
    }
  }
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 2 * BN);
}

}  // namespace vqb

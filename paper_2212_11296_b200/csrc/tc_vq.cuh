// (c) Vector quantizer on tcgen05 with a certified argmin
// (vq_apply_rows, proj/src/model.cpp:283-319; ties to the lowest index).
//
// Input per attention-output row x (written by the attention epilogue): the
// two-term bf16 split x = xh + xl + r (xh = bf16(x), xl = bf16(x - xh), so
// |r| <= 2^-8/(1-2^-8) |xl|), |x|^2 and |xl|^2. Warp-specialised persistent
// kernel, 128 rows per tile:
//   warp 0   TMA producer: A = xh, xl [128 x 64] and B = codebook[256 x 64]
//            per K-block into a 3-stage SW128 ring (mbarrier full/empty);
//   warp 1   MMA issuer: acc_j = xh . W_j + xl . W_j, 256 codes per
//            accumulator, two TMEM accumulators (512 columns) so the
//            epilogue of one code chunk overlaps the MMAs of the next;
//   warps 2-17 epilogue (four per TMEM lane quadrant, 64 columns of each
//            accumulator each): D~_j = |W_j|^2 - 2 acc_j is within
//            E = 2(|r| + d 2^-23 |x|) max|W| + slack of the exact
//            D_j(x) - |x|^2, so every code with D~_j <= running min + 2E is
//            kept (<= 8 per part; a part scans a 32-column group only when its
//            minimum comes within 2E of the running minimum, by a bit mask of
//            the survivors); a single survivor is the answer, otherwise the
//            row and its survivors go to
//            a queue and k_vq_rescore re-scores them as
//            sum_c ((xh + xl)_c - W_jc)^2 in double, c ascending — the
//            reference's own arithmetic (proj/src/model.cpp:298-303) — and the
//            lowest index wins (strict <, :304). Deferring the rare re-scoring
//            keeps it off the epilogue's critical path.
// The MMA reads bf16(W); when W is not bf16-exact (an unsnapped model) the
// bound widens by 2|x| max_j |W_j - bf16(W_j)| (werr), so the certificate
// still holds against the fp32 codebook the re-scoring uses.
#pragma once

#include "common.cuh"
#include "tc_common.cuh"
#include "tma.cuh"

namespace vqb {

constexpr int TCV_NCH = 256;  // codes per accumulator
constexpr int TCV_STAGES = 3;
constexpr int TCV_A_BYTES = 128 * 128;
constexpr int TCV_B_BYTES = TCV_NCH * 128;
constexpr int TCV_STAGE_BYTES = 2 * TCV_A_BYTES + TCV_B_BYTES;
constexpr int TCV_CAND = 8;
// producer warp, MMA warp, 16 epilogue warps: four per TMEM lane quadrant,
// each taking 64 of an accumulator's 256 columns (enough warps that the
// epilogue drains one accumulator faster than the MMAs fill the other)
constexpr int TCV_EPI_PARTS = 4;
constexpr int TCV_THREADS = 64 + 32 * 4 * TCV_EPI_PARTS;
constexpr int TCV_QCAND = TCV_EPI_PARTS * TCV_CAND;  // queued survivors per row

inline size_t tcv_smem_bytes(int Q) {
  return 1024 + size_t(TCV_STAGES) * TCV_STAGE_BYTES + 256 + size_t(Q) * 4 +
         2 * size_t(TCV_EPI_PARTS) * 128 * 12 + 64;
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

// Candidate list of one row (lives in local memory; touched only on the rare
// near-minimum codes, kept out of line so the streaming loop stays small).
struct Cands {
  float d[TCV_CAND];
  int j[TCV_CAND];
  int n;
  int overflow;
};

__device__ __noinline__ void cand_add(Cands& C, float dt, int j, float thr) {
  int w = 0;
  for (int i = 0; i < C.n; ++i)
    if (C.d[i] <= thr) {
      C.d[w] = C.d[i];
      C.j[w] = C.j[i];
      ++w;
    }
  C.n = w;
  if (w < TCV_CAND) {
    C.d[w] = dt;
    C.j[w] = j;
    C.n = w + 1;
  } else {
    C.overflow = 1;
  }
}

__device__ __forceinline__ void epi_bar() {  // the epilogue threads
  asm volatile("bar.sync 1, %0;" ::"n"(32 * 4 * TCV_EPI_PARTS) : "memory");
}

__global__ void __launch_bounds__(TCV_THREADS, 1) k_tc_vq(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmL,
    const __grid_constant__ CUtensorMap tmB,
    const int64_t* __restrict__ Mp, int d, const float* __restrict__ xn2g,
    const float* __restrict__ xl2g, const float* __restrict__ wn2_g, float wmax, float werr,
    int Q, int32_t* __restrict__ code,
    int32_t* __restrict__ cand, int32_t* __restrict__ ncand, int32_t* __restrict__ qrows,
    uint32_t* __restrict__ qcount) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* tail = smem + TCV_STAGES * TCV_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  uint64_t* empty = full + TCV_STAGES;
  uint64_t* acc_full = empty + TCV_STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* wn2 = reinterpret_cast<float*>(tail + 256);
  // per-row merge scratch, double-buffered by tile parity (no barrier needed
  // before the next tile reuses it)
  float* red_min0 = wn2 + Q;                                               // [2][parts][128]
  int* red_cnt0 = reinterpret_cast<int*>(red_min0 + 2 * TCV_EPI_PARTS * 128);  // [2][parts][128]
  int* red_jf0 = red_cnt0 + 2 * TCV_EPI_PARTS * 128;                           // [2][parts][128]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = *Mp;
  const int KB = d / 64;
  const int NCH = Q / TCV_NCH;
  const int64_t n_tiles = (M + 127) / 128;
  if (tid == 0) {
    for (int s = 0; s < TCV_STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], 4 * TCV_EPI_PARTS);
    }
    tc::mbar_fence_init();
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmL);
    tc::prefetch_tmap(&tmB);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  for (int j = tid; j < Q; j += TCV_THREADS) wn2[j] = wn2_g[j];
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = tc::smem_u32(smem);

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        for (int c = 0; c < NCH; ++c)
          for (int kb = 0; kb < KB; ++kb, ++it) {
            const uint32_t s = it % TCV_STAGES;
            if (it >= TCV_STAGES) tc::mbar_wait(&empty[s], ((it / TCV_STAGES) - 1) & 1);
            const uint32_t sa = sbase + s * TCV_STAGE_BYTES;
            const uint32_t fb = tc::smem_u32(&full[s]);
            tc::mbar_expect_tx(fb, TCV_STAGE_BYTES);
            tc::tma_load_2d(sa, &tmA, kb * 64, int(t * 128), fb);
            tc::tma_load_2d(sa + TCV_A_BYTES, &tmL, kb * 64, int(t * 128), fb);
            tc::tma_load_2d(sa + 2 * TCV_A_BYTES, &tmB, kb * 64, c * TCV_NCH, fb);
          }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::make_idesc_bf16(128, TCV_NCH);
      uint32_t it = 0, acc = 0;
#ifdef VQNQS_VQ_TRACE  // developer instrumentation: where the MMA warp waits
      long long w_acc = 0, w_full = 0, t_all = clock64();
#endif
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        for (int c = 0; c < NCH; ++c, ++acc) {
          const uint32_t b = acc & 1;
#ifdef VQNQS_VQ_TRACE
          long long t0 = clock64();
#endif
          if (acc >= 2) tc::mbar_wait(&acc_empty[b], ((acc >> 1) - 1) & 1);
#ifdef VQNQS_VQ_TRACE
          w_acc += clock64() - t0;
#endif
          tc::fence_after();
          for (int kb = 0; kb < KB; ++kb, ++it) {
            const uint32_t s = it % TCV_STAGES;
#ifdef VQNQS_VQ_TRACE
            long long t1 = clock64();
#endif
            tc::mbar_wait(&full[s], (it / TCV_STAGES) & 1);
#ifdef VQNQS_VQ_TRACE
            w_full += clock64() - t1;
#endif
            tc::fence_after();
            const uint32_t sa = sbase + s * TCV_STAGE_BYTES;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t bdesc = tc::make_desc_sw128(sa + 2 * TCV_A_BYTES + k * 32);
              tc::mma_bf16(tmem + b * TCV_NCH, tc::make_desc_sw128(sa + k * 32), bdesc, idesc,
                           (kb | k) != 0);
              tc::mma_bf16(tmem + b * TCV_NCH, tc::make_desc_sw128(sa + TCV_A_BYTES + k * 32),
                           bdesc, idesc, 1u);
            }
            tc::mma_commit(&empty[s]);
          }
          tc::mma_commit(&acc_full[b]);
        }
      }
#ifdef VQNQS_VQ_TRACE
      if (blockIdx.x < 3)
        printf("VQTR b%d total %lld wait_acc_empty %lld wait_full %lld stages %u\n", blockIdx.x,
               clock64() - t_all, w_acc, w_full, it);
#endif
    }
  } else {
    // ---------------- epilogue: warp w drains TMEM lanes 32 (w % 4)
    const int row = (warp & 3) * 32 + lane;
    const int part = (warp - 2) >> 2;  // columns [PW part, PW part + PW) of a chunk
    constexpr int PW = TCV_NCH / TCV_EPI_PARTS;
    static_assert(PW == 64, "the epilogue loads a part as two 32-column groups");
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    // the row norms are loaded one tile ahead (their latency would otherwise
    // sit in front of every tile's first accumulator)
    float xn2_nx = 0.f, xl2_nx = 0.f;
    if (blockIdx.x < n_tiles && (int64_t)blockIdx.x * 128 + row < M) {
      xn2_nx = xn2g[(int64_t)blockIdx.x * 128 + row];
      xl2_nx = xl2g[(int64_t)blockIdx.x * 128 + row];
    }
    int tpar = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, tpar ^= 1) {
      const int64_t my = t * 128 + row;
      const bool live = my < M;
      const float xn = live ? sqrtf(xn2_nx) : 0.f;
      const float xln = live ? sqrtf(xl2_nx) : 0.f;
      {
        const int64_t myn = (t + gridDim.x) * 128 + row;
        if (t + gridDim.x < n_tiles && myn < M) {
          xn2_nx = xn2g[myn];
          xl2_nx = xl2g[myn];
        }
      }
      float* red_min = red_min0 + tpar * TCV_EPI_PARTS * 128;
      int* red_cnt = red_cnt0 + tpar * TCV_EPI_PARTS * 128;
      int* red_jf = red_jf0 + tpar * TCV_EPI_PARTS * 128;
      // |r| <= 2^-8 / (1 - 2^-8) |xl|: the residual of the two-term split
      // + 2|x| max_j |W_j - bf16(W_j)|: the MMA sees the bf16-rounded
      // codebook, |W_j|^2 is the exact one (werr = 0 for a snapped codebook)
      const float E = 2.f * (0.00393f * xln * wmax + float(d) * 1.2e-7f * xn * wmax) +
                      4e-7f * (wmax * wmax + 2.f * xn * wmax) + 2.00001f * xn * werr;
      const float w2 = 2.f * E;
      float run_min = INFINITY;
      Cands C;
      C.n = 0;
      C.overflow = 0;
      for (int c = 0; c < NCH; ++c, ++acc) {
        const uint32_t b = acc & 1;
        tc::mbar_wait(&acc_full[b], (acc >> 1) & 1);
        tc::fence_after();
        // both 32-column groups of the part are loaded before one wait
        float vv[2][32];
        tc::tmem_ld32(trow + b * TCV_NCH + part * PW, vv[0]);
        tc::tmem_ld32(trow + b * TCV_NCH + part * PW + 32, vv[1]);
        tc::tmem_wait_ld();
        float gm[2];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const int jbase = c * TCV_NCH + part * PW + 32 * g;
          gm[g] = INFINITY;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            vv[g][j] = fmaf(-2.f, vv[g][j], wn2[jbase + j]);
            gm[g] = fminf(gm[g], vv[g][j]);
          }
        }
        // the threshold uses both groups' minima, so a group is scanned for
        // survivors only when it holds (or nearly holds) the running minimum
        run_min = fminf(run_min, fminf(gm[0], gm[1]));
        const float thr = run_min + w2;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (gm[g] <= thr) {  // rare once the running minimum settles
            const float* v = vv[g];
            const int jbase = c * TCV_NCH + part * PW + 32 * g;
            // the lane's survivors as a bit mask, then one insertion per set
            // bit (j ascending): a lane pays for its own candidates only,
            // instead of the warp stepping through 32 divergent insertions
            uint32_t m = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) m |= (v[j] <= thr ? 1u : 0u) << j;
            // each survivor is recorded with the group minimum, a lower bound
            // of its distance: later pruning (d <= threshold) then keeps a
            // superset of the rows' true survivors, which only the exact
            // re-scoring can shrink (never drops the argmin)
            while (m) {
              const int j = __ffs(m) - 1;
              m &= m - 1;
              cand_add(C, gm[g], jbase + j, thr);
            }
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tc::smem_u32(&acc_empty[b]));
      }
      // ---- merge the two warpgroups' survivors for this row
      red_min[part * 128 + row] = run_min;
      epi_bar();
      float gmin = red_min[row];
#pragma unroll
      for (int q = 1; q < TCV_EPI_PARTS; ++q) gmin = fminf(gmin, red_min[q * 128 + row]);
      int mine = 0, jfirst = 0x7fffffff;
#pragma unroll 1
      for (int i = 0; i < C.n; ++i)
        if (C.d[i] <= gmin + w2) {
          ++mine;
          jfirst = min(jfirst, C.j[i]);
        }
      red_cnt[part * 128 + row] = C.overflow ? 1000 : mine;
      red_jf[part * 128 + row] = jfirst;
      epi_bar();
      int total = 0, before = 0, jf = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < TCV_EPI_PARTS; ++q) {
        const int cq = red_cnt[q * 128 + row];
        if (q < part) before += cq;
        total += cq;
        jf = min(jf, red_jf[q * 128 + row]);
      }
      if (live) {
        if (total == 1) {
          if (part == 0) code[my] = jf;
        } else {
          // queue the row: the parts' survivors in part order
          const bool over = total >= 1000;
          if (!over) {
            int w = before;
#pragma unroll 1
            for (int i = 0; i < C.n; ++i)
              if (C.d[i] <= gmin + w2) cand[my * TCV_QCAND + w++] = C.j[i];
          }
          if (part == 0) {
            ncand[my] = over ? -1 : total;
            qrows[atomicAdd(qcount, 1u)] = (int32_t)my;
          }
        }
      }
      // no barrier here: the next tile merges through the other scratch
      // buffer, and its first barrier orders this tile's reads before the
      // tile after next overwrites this buffer
    }
  }
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// Re-scoring of the queued rows: one warp per row, one lane per survivor,
// each summing sequentially in double (c ascending) exactly like the
// reference; overflowed rows scan the whole codebook. Ties -> lowest index.
__global__ void __launch_bounds__(256) k_vq_rescore(
    const uint32_t* __restrict__ qcount, const int32_t* __restrict__ qrows,
    const int32_t* __restrict__ ncand, const int32_t* __restrict__ cand,
    const bf16* __restrict__ xh, const bf16* __restrict__ xl, const float* __restrict__ cb32,
    int d, int Q, int32_t* __restrict__ code, unsigned long long* __restrict__ n_rescored) {
  // eight lanes per queued row, four rows per warp (a row has ~2 survivors:
  // a lane per survivor left most of a 32-lane warp idle); each distance is
  // one lane's sequential double sum as before
  const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
  const int nq = (int)*qcount;
  unsigned long long done = 0;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t k0 = wid * 4; k0 < nq; k0 += nwarps * 4) {
    const int64_t k = k0 + grp;
    const bool valid = k < nq;
    double best = INFINITY;
    int jb = 0x7fffffff;
    int64_t row = 0;
    if (valid) {
      row = qrows[k];
      const int n = ncand[row];
      const bf16* xhr = xh + row * d;
      const bf16* xlr = xl + row * d;
      if (n >= 0) {
        for (int t = sub; t < n; t += 8) {
          const int j = cand[row * TCV_QCAND + t];
          const double s2 = vq_exact_d2(xhr, xlr, cb32 + (int64_t)j * d, d);
          if (s2 < best || (s2 == best && j < jb)) {
            best = s2;
            jb = j;
          }
        }
        if (sub == 0) done += n;
      } else {
#pragma unroll 1
        for (int j = sub; j < Q; j += 8) {
          const double s2 = vq_exact_d2(xhr, xlr, cb32 + (int64_t)j * d, d);
          if (s2 < best) {  // j ascending per lane: strict < keeps the lowest index
            best = s2;
            jb = j;
          }
        }
        if (sub == 0) done += Q;
      }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oj = __shfl_xor_sync(0xffffffffu, jb, o);
      if (ob < best || (ob == best && oj < jb)) {
        best = ob;
        jb = oj;
      }
    }
    // no finite distance (x or the codebook not finite): the reference's
    // argmin keeps its initial index 0 (proj/src/model.cpp:283-319)
    if (valid && sub == 0) code[row] = jb == 0x7fffffff ? 0 : jb;
  }
  if (n_rescored && sub == 0 && done) atomicAdd(n_rescored, done);
}

// queue storage for the deferred re-scoring (device buffers, grown on demand)
struct VqScratch {
  int32_t* cand = nullptr;
  int32_t* ncand = nullptr;
  int32_t* qrows = nullptr;
  uint32_t* qcount = nullptr;
  size_t cap = 0;
  void ensure(size_t rows) {
    if (rows <= cap && qcount) return;
    release();
    cap = rows + rows / 4 + 1024;
    if (cudaMalloc(&cand, cap * TCV_QCAND * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&ncand, cap * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&qrows, cap * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&qcount, sizeof(uint32_t)) != cudaSuccess)
      throw std::runtime_error("VQ re-scoring queue: out of device memory");
  }
  void release() {
    if (cand) cudaFree(cand);
    if (ncand) cudaFree(ncand);
    if (qrows) cudaFree(qrows);
    if (qcount) cudaFree(qcount);
    cand = ncand = qrows = nullptr;
    qcount = nullptr;
    cap = 0;
  }
};

}  // namespace vqb

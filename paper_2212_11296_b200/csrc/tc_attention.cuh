// (b) Gathered causal attention on tcgen05 (multihead_attention /
// masked_attention, proj/src/tensor.cpp:199-262, over the compressed stream,
// proj/src/dedup.cpp:128-134), for the bf16 configurations.
//
// Work unit: a TILE of up to 128 active query locations made of whole
// connected rows of ONE sample (k_build_tiles packs rows greedily). For a
// query at (row k, position p >= a_k) the keys are the base row's at
// positions t < a_k and row k's own active locations a_k <= t <= p. The own
// keys of every row in the tile are the tile's own locations, so per head:
//   S_base = Q K_base^T   (M=128, N=T_pad)   base row's keys
//   S_own  = Q K_tile^T   (M=128, N=128)     the tile's own keys
//   softmax per query over S_base[:, :a_k] and S_own[:, seg_k .. i]
//   O      = P_base V_base + P_own V_tile    (M=128, N=dh)
// Scores are scaled after the product and the normalised probabilities are
// rounded to bf16 before the value product, exactly where the reference's
// product boundary rounds under bf16 emulation.
//
// All operands are staged with cp.async per 64-wide head group as SW128
// tiles [rows x 64]: Q/K are K-major operands; V, staged the same way
// (key rows, 64 head-dims contiguous), is the MN-major B operand of the value
// product, so nothing is transposed. The softmax reads only the warp's live
// score columns, in two TMEM passes (online max/sum, then probabilities).
// TMEM: S_base | S_own | O(group) = T_pad + 128 + 64 <= 512 columns.
#pragma once

#include "common.cuh"
#include "tc_common.cuh"

namespace vqb {

struct AttnTile {
  int32_t sample;
  int32_t nloc;
  int64_t loc0;  // first active location (global)
};

// Greedy packing of whole rows (consecutive in active-location order) into
// tiles of <= 128 locations, one thread per sample.
__global__ void k_build_tiles(int S, int R1, int T, const int32_t* __restrict__ K,
                              const int32_t* __restrict__ row_t1,
                              const int64_t* __restrict__ act_off, AttnTile* __restrict__ tiles,
                              int32_t* __restrict__ n_tiles) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const int Ks = K[s];
  int cur = 0;
  int64_t start = act_off[s];
  for (int k = 0; k < Ks; ++k) {
    const int n = k == 0 ? T : T - (row_t1[(int64_t)s * R1 + k] + 1);
    if (n <= 0) continue;
    if (cur + n > 128) {
      const int t = atomicAdd(n_tiles, 1);
      tiles[t] = AttnTile{s, cur, start};
      start += cur;
      cur = 0;
    }
    cur += n;
  }
  if (cur > 0) {
    const int t = atomicAdd(n_tiles, 1);
    tiles[t] = AttnTile{s, cur, start};
  }
}

__host__ __device__ inline int attn_tpad(int T) { return ((T + 15) / 16) * 16; }
__host__ __device__ inline int attn_kb_base(int T) { return (attn_tpad(T) + 63) / 64; }

// shared memory carve (bytes, all sub-tiles 1024-aligned)
struct AttnSmem {
  uint32_t q, kown, vown, kbase, vbase, pbase, pown, bar, total;
  __host__ __device__ AttnSmem(int T) {
    const uint32_t KBb = (uint32_t)attn_kb_base(T);
    q = 0;                             // 128 x 64
    kown = q + 128 * 128;              // 128 x 64
    vown = kown + 128 * 128;           // 128 x 64 (MN-major B)
    kbase = vown + 128 * 128;          // (64*KBb) x 64
    vbase = kbase + 64 * KBb * 128;    // (64*KBb) x 64
    pbase = vbase + 64 * KBb * 128;    // P base: 128 x (64*KBb) in KBb blocks
    pown = pbase + KBb * 128 * 128;    // P own: 128 x 128 in 2 blocks
    bar = pown + 2 * 128 * 128;
    total = bar + 64;
  }
};

__device__ __forceinline__ int warp_max_i(int v) { return __reduce_max_sync(0xffffffffu, v); }
__device__ __forceinline__ int warp_min_i(int v) { return __reduce_min_sync(0xffffffffu, v); }

__global__ void __launch_bounds__(128, 1) k_tc_attention(
    const AttnTile* __restrict__ tiles, const int32_t* __restrict__ n_tiles_p, int R1, int T,
    int d, int dh, float scale, const int32_t* __restrict__ row_t1,
    const int64_t* __restrict__ act_off, const int32_t* __restrict__ lrow,
    const int16_t* __restrict__ lpos, const int32_t* __restrict__ I,
    const int64_t* __restrict__ Uoff, const bf16* __restrict__ qkv, float* __restrict__ att) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const AttnSmem L(T);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 2);
  __shared__ int s_amax;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int TP = attn_tpad(T);
  const int KBb = attn_kb_base(T);
  const int n_tiles = *n_tiles_p;
  if (tid == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sb = tc::smem_u32(smem);
  const uint32_t TS_BASE = 0, TS_OWN = (uint32_t)TP, TS_O = (uint32_t)TP + 128;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  const int ld = 3 * d;
  const int G = d / 64;
  const int hpg = 64 / dh;  // heads per 64-wide group
  const float sl2 = scale * 1.4426950408889634f;
  uint32_t ph_s = 0, ph_o = 0;

  for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
    const AttnTile tile = tiles[ti];
    const int s = tile.sample;
    const int64_t uo = Uoff[s];
    const int64_t base = act_off[s];
    // this thread's query (tile row tid): base keys [0, a), own keys [own_lo, tid]
    const bool live = tid < tile.nloc;
    int a = 0, own_lo = tid + 1, own_hi = tid;
    int64_t myloc = 0;
    if (live) {
      myloc = tile.loc0 + tid;
      const int r = lrow[myloc];
      const int p = lpos[myloc];
      a = (r % R1) == 0 ? 0 : row_t1[r] + 1;
      own_lo = tid - (p - a);
    } else {
      own_lo = 1 << 20;
      own_hi = -1;
    }
    if (tid == 0) s_amax = 0;
    __syncthreads();
    atomicMax(&s_amax, a);
    // warp-uniform live column ranges
    const int w_amax = warp_max_i(a);
    const int w_olo = warp_min_i(own_lo), w_ohi = warp_max_i(own_hi);
    const int wb_end = (w_amax + 15) & ~15;
    const int wo_beg = w_olo >= 128 ? 128 : (w_olo & ~15), wo_end = (w_ohi + 16) & ~15;
    for (int gi = 0; gi < G; ++gi) {
      // ---- stage the group's operands (cp.async, zero-filled tails)
      for (int e = tid; e < 128 * 8; e += 128) {
        const int r = e >> 3, c = e & 7;
        const bool ok = r < tile.nloc;
        const int64_t u = ok ? uo + I[tile.loc0 + r] : 0;
        const bf16* src = qkv + u * ld + gi * 64 + c * 8;
        const uint32_t o = tc::sw128_chunk(r, c);
        tc::cp_async16_zfill(sb + L.q + o, src, ok);
        tc::cp_async16_zfill(sb + L.kown + o, src + d, ok);
        tc::cp_async16_zfill(sb + L.vown + o, src + 2 * d, ok);
      }
      for (int e = tid; e < 64 * KBb * 8; e += 128) {
        const int t = e >> 3, c = e & 7;
        const bool ok = t < T;
        const int64_t u = ok ? uo + I[base + t] : 0;
        const bf16* src = qkv + u * ld + d + gi * 64 + c * 8;
        const uint32_t o = tc::sw128_chunk(t, c);
        tc::cp_async16_zfill(sb + L.kbase + o, src, ok);
        tc::cp_async16_zfill(sb + L.vbase + o, src + d, ok);
      }
      tc::cp_async_commit();
      tc::cp_async_wait<0>();
      tc::fence_proxy_async();
      __syncthreads();
      const int t_amax = s_amax;
      const int kb_base = (t_amax + 15) & ~15;  // base keys any row uses
      for (int hh = 0; hh < hpg; ++hh) {
        const uint32_t koff = (uint32_t)(hh * dh * 2);  // head offset inside the 128-B row
        // ---- scores
        if (tid == 0) {
          tc::fence_after();
          const uint32_t idS_b = tc::make_idesc_bf16(128, kb_base > 0 ? kb_base : 16);
          const uint32_t idS_o = tc::make_idesc_bf16(128, 128);
          for (int k = 0; k < dh / 16; ++k) {
            if (kb_base > 0)
              tc::mma_bf16(tmem + TS_BASE, tc::make_desc_sw128(sb + L.q + koff + k * 32),
                           tc::make_desc_sw128(sb + L.kbase + koff + k * 32), idS_b, k != 0);
            tc::mma_bf16(tmem + TS_OWN, tc::make_desc_sw128(sb + L.q + koff + k * 32),
                         tc::make_desc_sw128(sb + L.kown + koff + k * 32), idS_o, k != 0);
          }
          tc::mma_commit(&mbar[0]);
        }
        tc::mbar_wait(&mbar[0], ph_s);
        ph_s ^= 1;
        tc::fence_after();
        // ---- pass 1: online max / sum over the live columns (log2 domain)
        float m = -INFINITY, sum = 0.f;
        for (int c0 = 0; c0 < wb_end; c0 += 16) {
          float v[16];
          tc::tmem_ld16(trow + TS_BASE + c0, v);
          tc::tmem_wait_ld();
          float cm = -INFINITY;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < a) cm = fmaxf(cm, v[j] * sl2);
          if (cm > m) {
            sum *= exp2f(m - cm);
            m = cm;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < a) sum += exp2f(v[j] * sl2 - m);
        }
        for (int c0 = wo_beg; c0 < wo_end; c0 += 16) {
          float v[16];
          tc::tmem_ld16(trow + TS_OWN + c0, v);
          tc::tmem_wait_ld();
          float cm = -INFINITY;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j >= own_lo && c0 + j <= own_hi) cm = fmaxf(cm, v[j] * sl2);
          if (cm > m) {
            sum *= exp2f(m - cm);
            m = cm;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j >= own_lo && c0 + j <= own_hi) sum += exp2f(v[j] * sl2 - m);
        }
        const float inv = 1.f / sum;
        // ---- pass 2: bf16 probabilities into the P tiles (zeros elsewhere)
        for (int c0 = 0; c0 < kb_base; c0 += 16) {
          float v[16];
          if (c0 < wb_end) {
            tc::tmem_ld16(trow + TS_BASE + c0, v);
            tc::tmem_wait_ld();
          }
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const float p0 = (c0 + j < a) ? exp2f(v[j] * sl2 - m) * inv : 0.f;
            const float p1 = (c0 + j + 1 < a) ? exp2f(v[j + 1] * sl2 - m) * inv : 0.f;
            pk[j / 2] = tc::pack_bf16(p0, p1);
          }
          const uint32_t blk = sb + L.pbase + (uint32_t)(c0 >> 6) * (128 * 128);
          const uint32_t cc = (uint32_t)((c0 & 63) >> 3);
          tc::st_shared_v4(blk + tc::sw128_chunk(tid, cc), pk[0], pk[1], pk[2], pk[3]);
          tc::st_shared_v4(blk + tc::sw128_chunk(tid, cc + 1), pk[4], pk[5], pk[6], pk[7]);
        }
        for (int c0 = 0; c0 < 128; c0 += 16) {
          float v[16];
          const bool in = c0 >= wo_beg && c0 < wo_end;
          if (in) {
            tc::tmem_ld16(trow + TS_OWN + c0, v);
            tc::tmem_wait_ld();
          }
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const int t0 = c0 + j, t1 = c0 + j + 1;
            const float p0 = (in && t0 >= own_lo && t0 <= own_hi) ? exp2f(v[j] * sl2 - m) * inv : 0.f;
            const float p1 = (in && t1 >= own_lo && t1 <= own_hi) ? exp2f(v[j + 1] * sl2 - m) * inv : 0.f;
            pk[j / 2] = tc::pack_bf16(p0, p1);
          }
          const uint32_t blk = sb + L.pown + (uint32_t)(c0 >> 6) * (128 * 128);
          const uint32_t cc = (uint32_t)((c0 & 63) >> 3);
          tc::st_shared_v4(blk + tc::sw128_chunk(tid, cc), pk[0], pk[1], pk[2], pk[3]);
          tc::st_shared_v4(blk + tc::sw128_chunk(tid, cc + 1), pk[4], pk[5], pk[6], pk[7]);
        }
        tc::fence_before();
        tc::fence_proxy_async();
        __syncthreads();
        // ---- O_h = P_base V_base + P_own V_own  (V is the MN-major B operand)
        if (tid == 0) {
          tc::fence_after();
          const uint32_t idO = tc::make_idesc_bf16(128, dh) | (1u << 16);
          int first = 1;
          for (int k16 = 0; k16 < kb_base; k16 += 16) {
            const uint32_t kb = (uint32_t)(k16 >> 6), kk = (uint32_t)((k16 & 63) >> 4);
            tc::mma_bf16(tmem + TS_O + hh * dh,
                         tc::make_desc_sw128(sb + L.pbase + kb * 128 * 128 + kk * 32),
                         tc::make_desc_sw128(sb + L.vbase + (uint32_t)k16 * 128 + koff), idO,
                         first ? 0u : 1u);
            first = 0;
          }
          for (int k16 = 0; k16 < 128; k16 += 16) {
            const uint32_t kb = (uint32_t)(k16 >> 6), kk = (uint32_t)((k16 & 63) >> 4);
            tc::mma_bf16(tmem + TS_O + hh * dh,
                         tc::make_desc_sw128(sb + L.pown + kb * 128 * 128 + kk * 32),
                         tc::make_desc_sw128(sb + L.vown + (uint32_t)k16 * 128 + koff), idO,
                         first ? 0u : 1u);
            first = 0;
          }
          tc::mma_commit(&mbar[1]);
        }
        // next head's scores overwrite S only after everyone read it (barrier
        // above); P is rewritten only after O has consumed it
        tc::mbar_wait(&mbar[1], ph_o);
        ph_o ^= 1;
        tc::fence_after();
      }
      // ---- drain the group's O (64 cols) to the fp32 attention output
      for (int c0 = 0; c0 < 64; c0 += 16) {
        float v[16];
        tc::tmem_ld16(trow + TS_O + c0, v);
        tc::tmem_wait_ld();
        if (live) {
          float4* o = reinterpret_cast<float4*>(att + myloc * d + gi * 64 + c0);
          o[0] = make_float4(v[0], v[1], v[2], v[3]);
          o[1] = make_float4(v[4], v[5], v[6], v[7]);
          o[2] = make_float4(v[8], v[9], v[10], v[11]);
          o[3] = make_float4(v[12], v[13], v[14], v[15]);
        }
      }
      tc::fence_before();
      __syncthreads();
    }
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

inline bool tc_attn_ok(int prec, int d, int dh, int T) {
  return prec == 1 && d % 64 == 0 && (dh == 16 || dh == 32 || dh == 64) && T <= 128;
}

}  // namespace vqb

// (b) Gathered causal attention on tcgen05 (multihead_attention /
// masked_attention, proj/src/tensor.cpp:199-262, over the compressed stream,
// proj/src/dedup.cpp:128-134), for the bf16 configurations.
//
// Work unit: a TILE of up to 128 active query locations made of whole
// connected rows of ONE sample (k_build_tiles packs rows greedily). For a
// query at (row k, position p >= a_k) the keys are the base row's at
// positions t < a_k and row k's own active locations a_k <= t <= p. The own
// keys of every row in the tile are the tile's own locations, so per head:
//   S_base = Q K_base^T   (M=128, N=16*ceil(max a/16))   base row's keys
//   S_own  = Q K_tile^T   (M=128, N=128)                 the tile's own keys
//   softmax per query over S_base[:, :a_k] and S_own[:, seg_k .. i]
//   O      = P_base V_base + P_own V_tile                (M=128, N=dh)
// Scores are scaled after the product and the normalised probabilities are
// rounded to bf16 before the value product, exactly where the reference's
// product boundary rounds under bf16 emulation.
//
// All operands are staged with cp.async per 64-wide head group as SW128
// tiles [rows x 64]: Q/K are K-major operands; V, staged the same way
// (key rows, 64 head-dims contiguous), is the MN-major B operand of the value
// product, so nothing is transposed. Softmax: ONE TMEM pass loads the warp's
// live score columns into registers (4 x 16 per thread); max, exp2 + sum and
// the normalised bf16 P tiles are computed from registers, and the next
// head's score MMA is issued as soon as every warp has loaded its scores.
// TMEM: S_base | S_own | O(group) = T_pad + 128 + 64 <= 512 columns.
//
// Outputs per active location: the attention row x as its two-term bf16
// split xh = bf16(x), xl = bf16(x - xh) (the VQ distance GEMM operands; x is
// represented to 2^-18 relative), |x|^2 and |x - xh - xl|^2 (the certified
// argmin error bound, tc_vq.cuh). 512 threads: warp w owns TMEM lanes
// 32(w%4).. (its query rows); the four warpgroups split the score columns.
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
                              const int32_t* __restrict__ row_perm,
                              const int64_t* __restrict__ act_off, AttnTile* __restrict__ tiles,
                              int32_t* __restrict__ n_tiles) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const int Ks = K[s];
  int cur = 0;
  int64_t start = act_off[s];
  for (int i = 0; i < Ks; ++i) {  // rows in active-layout order (k_connected)
    const int k = row_perm[(int64_t)s * R1 + i];
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
  uint32_t q, kown, vown, kbase, vbase, pbase, pown, rows, bar, total;
  __host__ __device__ AttnSmem(int T) {
    const uint32_t KBb = (uint32_t)attn_kb_base(T);
    q = 0;                             // 128 x 64
    kown = q + 128 * 128;              // 128 x 64
    vown = kown + 128 * 128;           // 128 x 64 (MN-major B)
    kbase = vown + 128 * 128;          // (64*KBb) x 64
    vbase = kbase + 64 * KBb * 128;    // (64*KBb) x 64
    pbase = vbase + 64 * KBb * 128;    // P base: 128 x (64*KBb) in KBb blocks
    pown = pbase + KBb * 128 * 128;    // P own: 128 x 128 in 2 blocks
    rows = pown + 2 * 128 * 128;       // int64 row offsets: 128 tile + 128 base
    bar = rows + 256 * 8;
    total = bar + 64;
  }
};

__device__ __forceinline__ int warp_max_i(int v) { return __reduce_max_sync(0xffffffffu, v); }
__device__ __forceinline__ int warp_min_i(int v) { return __reduce_min_sync(0xffffffffu, v); }

constexpr int TCA_THREADS = 512;

__global__ void __launch_bounds__(TCA_THREADS, 1) k_tc_attention(
    const AttnTile* __restrict__ tiles, const int32_t* __restrict__ n_tiles_p, int R1, int T,
    int d, int dh, float scale, const int32_t* __restrict__ row_t1,
    const int64_t* __restrict__ act_off, const int32_t* __restrict__ lrow,
    const int16_t* __restrict__ lpos, const int32_t* __restrict__ I,
    const int64_t* __restrict__ Uoff, const bf16* __restrict__ qkv, bf16* __restrict__ xh_out,
    bf16* __restrict__ xl_out, float* __restrict__ xn2_out, float* __restrict__ rr2_out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const AttnSmem L(T);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 2);
  int64_t* rowq = reinterpret_cast<int64_t*>(smem + L.rows);  // qkv offsets of tile rows
  int64_t* rowb = rowq + 128;                                 // ... of base rows
  __shared__ float red[4][128];
  __shared__ float red2[4][128];
  __shared__ int s_amax;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & 127, part = tid >> 7;  // warp w drains TMEM lanes 32(w%4)..
  const int KBb = attn_kb_base(T);
  const int n_tiles = *n_tiles_p;
  const int TP = attn_tpad(T);
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
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
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
    // this thread's query (tile row `row`): base keys [0, a), own keys [own_lo, own_hi]
    const bool live = row < tile.nloc;
    int a = 0, own_lo = 1 << 20, own_hi = -1;
    int64_t myloc = 0;
    if (tid == 0) s_amax = 0;
    if (part == 0) {
      rowq[row] = live ? (uo + I[tile.loc0 + row]) * ld : -1;
      rowb[row] = row < T ? (uo + I[base + row]) * ld : -1;
    }
    if (live) {
      myloc = tile.loc0 + row;
      const int r = lrow[myloc];
      const int p = lpos[myloc];
      a = (r % R1) == 0 ? 0 : row_t1[r] + 1;
      own_lo = row - (p - a);
      own_hi = row;
    }
    __syncthreads();
    if (part == 0) atomicMax(&s_amax, a);
    // warp-uniform live column ranges (16-column chunks)
    const int wb_end = (warp_max_i(a) + 15) & ~15;
    const int w_olo = warp_min_i(own_lo), w_ohi = warp_max_i(own_hi);
    const int wo_beg = w_olo >= 128 ? 128 : (w_olo & ~15);
    const int wo_end = w_ohi < 0 ? 0 : ((w_ohi + 16) & ~15);
    float xn2 = 0.f, rr2 = 0.f;
    for (int gi = 0; gi < G; ++gi) {
      // ---- stage the group's operands (cp.async, zero-filled tails)
      for (int e = tid; e < 128 * 8; e += TCA_THREADS) {
        const int r = e >> 3, c = e & 7;
        const int64_t off = rowq[r];
        const bool ok = off >= 0;
        const bf16* src = qkv + (ok ? off : 0) + gi * 64 + c * 8;
        const uint32_t o = tc::sw128_chunk(r, c);
        tc::cp_async16_zfill(sb + L.q + o, src, ok);
        tc::cp_async16_zfill(sb + L.kown + o, src + d, ok);
        tc::cp_async16_zfill(sb + L.vown + o, src + 2 * d, ok);
      }
      for (int e = tid; e < 64 * KBb * 8; e += TCA_THREADS) {
        const int t = e >> 3, c = e & 7;
        const int64_t off = t < 128 ? rowb[t] : -1;
        const bool ok = off >= 0;
        const bf16* src = qkv + (ok ? off : 0) + d + gi * 64 + c * 8;
        const uint32_t o = tc::sw128_chunk(t, c);
        tc::cp_async16_zfill(sb + L.kbase + o, src, ok);
        tc::cp_async16_zfill(sb + L.vbase + o, src + d, ok);
      }
      tc::cp_async_commit();
      tc::cp_async_wait<0>();
      tc::fence_proxy_async();
      __syncthreads();
      const int kb_base = (s_amax + 15) & ~15;  // base keys any row of the tile uses
      auto issue_scores = [&](int hq) {
        const uint32_t qoff = (uint32_t)(hq * dh * 2);  // head offset inside the 128-B row
        const uint32_t idS_b = tc::make_idesc_bf16(128, kb_base > 0 ? kb_base : 16);
        const uint32_t idS_o = tc::make_idesc_bf16(128, 128);
        for (int k = 0; k < dh / 16; ++k) {
          if (kb_base > 0)
            tc::mma_bf16(tmem + TS_BASE, tc::make_desc_sw128(sb + L.q + qoff + k * 32),
                         tc::make_desc_sw128(sb + L.kbase + qoff + k * 32), idS_b, k != 0);
          tc::mma_bf16(tmem + TS_OWN, tc::make_desc_sw128(sb + L.q + qoff + k * 32),
                       tc::make_desc_sw128(sb + L.kown + qoff + k * 32), idS_o, k != 0);
        }
        tc::mma_commit(&mbar[0]);
      };
      if (tid == 0) {
        tc::fence_after();
        issue_scores(0);
      }
      for (int hh = 0; hh < hpg; ++hh) {
        const uint32_t koff = (uint32_t)(hh * dh * 2);  // head offset inside the 128-B row
        tc::mbar_wait(&mbar[0], ph_s);
        ph_s ^= 1;
        tc::fence_after();
        // ---- the warp's live score chunks go to registers in ONE TMEM pass:
        // warpgroup `part` owns 16-column chunks c = 16 part + 64 i (i = 0, 1)
        // of S_base and of S_own (T_pad <= 128), so the S columns are free for
        // the next head's score MMA as soon as every warp has loaded them.
        float vb[2][16], vo[2][16];
        const int cb0 = part * 16, cb1 = part * 16 + 64;
        const bool lb0 = cb0 < wb_end, lb1 = cb1 < wb_end;
        const bool lo0 = cb0 >= wo_beg && cb0 < wo_end, lo1 = cb1 >= wo_beg && cb1 < wo_end;
        if (lb0) tc::tmem_ld16(trow + TS_BASE + cb0, vb[0]);
        if (lb1) tc::tmem_ld16(trow + TS_BASE + cb1, vb[1]);
        if (lo0) tc::tmem_ld16(trow + TS_OWN + cb0, vo[0]);
        if (lo1) tc::tmem_ld16(trow + TS_OWN + cb1, vo[1]);
        tc::tmem_wait_ld();
        float m = -INFINITY;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (lb0 && cb0 + j < a) m = fmaxf(m, vb[0][j]);
          if (lb1 && cb1 + j < a) m = fmaxf(m, vb[1][j]);
          if (lo0 && cb0 + j >= own_lo && cb0 + j <= own_hi) m = fmaxf(m, vo[0][j]);
          if (lo1 && cb1 + j >= own_lo && cb1 + j <= own_hi) m = fmaxf(m, vo[1][j]);
        }
        red[part][row] = m;
        tc::fence_before();
        __syncthreads();
        if (tid == 0 && hh + 1 < hpg) {
          // S is in registers everywhere: the next head's scores overlap this
          // head's softmax and value MMA
          tc::fence_after();
          issue_scores(hh + 1);
        }
        m = fmaxf(fmaxf(red[0][row], red[1][row]), fmaxf(red[2][row], red[3][row])) * sl2;
        // ---- e = exp2(s*scale*log2e - m) on live entries, 0 elsewhere
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          vb[0][j] = (lb0 && cb0 + j < a) ? exp2f(fmaf(vb[0][j], sl2, -m)) : 0.f;
          vb[1][j] = (lb1 && cb1 + j < a) ? exp2f(fmaf(vb[1][j], sl2, -m)) : 0.f;
          sum += vb[0][j];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) sum += vb[1][j];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          vo[0][j] = (lo0 && cb0 + j >= own_lo && cb0 + j <= own_hi)
                         ? exp2f(fmaf(vo[0][j], sl2, -m)) : 0.f;
          vo[1][j] = (lo1 && cb1 + j >= own_lo && cb1 + j <= own_hi)
                         ? exp2f(fmaf(vo[1][j], sl2, -m)) : 0.f;
          sum += vo[0][j];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) sum += vo[1][j];
        red2[part][row] = sum;
        __syncthreads();
        const float inv = 1.f / (((red2[0][row] + red2[1][row]) + red2[2][row]) + red2[3][row]);
        // P is rewritten only after the previous head's value MMA consumed it
        if (hh > 0) {
          tc::mbar_wait(&mbar[1], ph_o);
          ph_o ^= 1;
        }
        // ---- normalised bf16 probabilities into the P tiles
        auto put_p = [&](uint32_t blk0, int c0, const float* v) {
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 2) pk[j / 2] = tc::pack_bf16(v[j] * inv, v[j + 1] * inv);
          const uint32_t blk = blk0 + (uint32_t)(c0 >> 6) * (128 * 128);
          const uint32_t cc = (uint32_t)((c0 & 63) >> 3);
          tc::st_shared_v4(blk + tc::sw128_chunk(row, cc), pk[0], pk[1], pk[2], pk[3]);
          tc::st_shared_v4(blk + tc::sw128_chunk(row, cc + 1), pk[4], pk[5], pk[6], pk[7]);
        };
        if (cb0 < kb_base) put_p(sb + L.pbase, cb0, vb[0]);
        if (cb1 < kb_base) put_p(sb + L.pbase, cb1, vb[1]);
        put_p(sb + L.pown, cb0, vo[0]);
        put_p(sb + L.pown, cb1, vo[1]);
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
      }
      tc::mbar_wait(&mbar[1], ph_o);  // the group's last value MMA
      ph_o ^= 1;
      tc::fence_after();
      // ---- drain the group's O: warpgroup `part` takes columns [16 part, 16 part + 16)
      {
        float v[16];
        tc::tmem_ld16(trow + TS_O + part * 16, v);  // warp-collective: every lane loads
        tc::tmem_wait_ld();
        if (live) {
          uint32_t ph[8], pl[8];
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            ph[j / 2] = tc::pack_bf16(v[j], v[j + 1]);
            const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&ph[j / 2]);
            const float d0 = v[j] - __low2float(h), d1 = v[j + 1] - __high2float(h);
            pl[j / 2] = tc::pack_bf16(d0, d1);
            const __nv_bfloat162 l = *reinterpret_cast<const __nv_bfloat162*>(&pl[j / 2]);
            const float r0 = __low2float(l), r1 = __high2float(l);  // |xl|^2 (tc_vq.cuh)
            xn2 = fmaf(v[j], v[j], fmaf(v[j + 1], v[j + 1], xn2));
            rr2 = fmaf(r0, r0, fmaf(r1, r1, rr2));
          }
          uint4* oh = reinterpret_cast<uint4*>(xh_out + myloc * d + gi * 64 + part * 16);
          uint4* ol = reinterpret_cast<uint4*>(xl_out + myloc * d + gi * 64 + part * 16);
          oh[0] = make_uint4(ph[0], ph[1], ph[2], ph[3]);
          oh[1] = make_uint4(ph[4], ph[5], ph[6], ph[7]);
          ol[0] = make_uint4(pl[0], pl[1], pl[2], pl[3]);
          ol[1] = make_uint4(pl[4], pl[5], pl[6], pl[7]);
        }
      }
      tc::fence_before();
      __syncthreads();
    }
    // row norms: |x|^2 and |x - xh - xl|^2, reduced over the four warpgroups
    red[part][row] = xn2;
    red2[part][row] = rr2;
    __syncthreads();
    if (part == 0 && live) {
      xn2_out[myloc] = ((red[0][row] + red[1][row]) + red[2][row]) + red[3][row];
      rr2_out[myloc] = ((red2[0][row] + red2[1][row]) + red2[2][row]) + red2[3][row];
    }
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

inline bool tc_attn_ok(int prec, int d, int dh, int T) {
  return prec == 1 && d % 64 == 0 && (dh == 16 || dh == 32 || dh == 64) && T <= 128;
}

}  // namespace vqb

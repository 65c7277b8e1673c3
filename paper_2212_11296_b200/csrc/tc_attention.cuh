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
// Work items are (tile, 64-wide head group) pairs, persistent over the grid.
// The operands of item i+1 are staged with cp.async into the second of two
// SW128 buffers while item i computes: Q/K are K-major operands; V, staged
// the same way (key rows, 64 head-dims contiguous), is the MN-major B operand
// of the value product, so nothing is transposed. Per head ONE TMEM pass
// loads each warp's live score chunks into registers (the chunks are dealt
// round-robin to the four warpgroups that share a row quadrant); the
// warpgroups exchange (local max, local sum) once, write the normalised bf16
// probabilities straight back to TMEM, and the value product takes P as its
// TMEM A operand (no shared-memory round trip). The next head's score MMA is
// issued as soon as every warp holds its scores; the next item's first score
// MMA runs while this item's O drains.
// TMEM: S_base | S_own | P (bf16 pairs) | O(group) = 1.5 (T_pad + 128) + 64 <= 512.
//
// Outputs per active location: the attention row x as its two-term bf16
// split xh = bf16(x), xl = bf16(x - xh) (the VQ distance GEMM operands; x is
// represented to 2^-18 relative), |x|^2 and |x - xh - xl|^2 (the certified
// argmin error bound, tc_vq.cuh). 512 threads: warp w owns TMEM lanes
// 32(w%4).. (its query rows).
#pragma once

#include "common.cuh"
#include "tc_common.cuh"
#include "tma.cuh"

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

// shared memory carve (bytes; stages 1024-aligned). Two staging buffers, each
// q | k_own | v_own (128 x 64) | k_base | v_base (64 KBb x 64), so the operands
// of the next (tile, head group) item load while the current one computes.
struct AttnSmem {
  uint32_t stage, q, kown, vown, kbase, vbase, rows, info, bar, total;
  __host__ __device__ AttnSmem(int T) {
    const uint32_t KBb = (uint32_t)attn_kb_base(T);
    q = 0;
    kown = 128 * 128;
    vown = 2 * 128 * 128;
    kbase = 3 * 128 * 128;
    vbase = kbase + 64 * KBb * 128;
    stage = vbase + 64 * KBb * 128;
    rows = 2 * stage;    // int64 rowq[2][128], rowb[2][128]
    info = rows + 4096;  // int32 a[2][128], own_lo[2][128], wmax[2][4]
    bar = info + 2048 + 32;
    total = bar + 64;
  }
};

__device__ __forceinline__ int warp_max_i(int v) { return __reduce_max_sync(0xffffffffu, v); }
__device__ __forceinline__ int warp_min_i(int v) { return __reduce_min_sync(0xffffffffu, v); }

constexpr int TCA_THREADS = 512;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

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
  int64_t* rowq = reinterpret_cast<int64_t*>(smem + L.rows);  // [2][128] qkv offsets, tile rows
  int64_t* rowb = rowq + 256;                                 // [2][128] ... base rows
  int32_t* inf_a = reinterpret_cast<int32_t*>(smem + L.info);  // [2][128]
  int32_t* inf_lo = inf_a + 256;                               // [2][128]
  int32_t* wmax = inf_lo + 256;                                // [2][4]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.bar);  // S full, PV done, P ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 3);
  // exchange buffers alternate by head: a fast warp may publish head h+1
  // before a slow one has read head h (no block barrier in between)
  __shared__ float2 red[2][4][128];  // (local max, local sum)
  __shared__ float nrm[2][4][128];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row = tid & 127, part = tid >> 7;  // warp w owns TMEM lanes 32(w%4)..
  const int KBb = attn_kb_base(T);
  const int n_tiles = *n_tiles_p;
  const int TP = attn_tpad(T);
  const int G = d / 64;
  const int hpg = 64 / dh;  // heads per 64-wide group
  const int ld = 3 * d;
  const int my_tiles =
      (int)blockIdx.x < n_tiles ? (n_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x
                                : 0;
  const int nit = my_tiles * G;  // work items: (tile, head group)
  if (tid == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    tc::mbar_init(&mbar[2], TCA_THREADS / 32);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sb = tc::smem_u32(smem);
  // TMEM columns: S_base | S_own | P (bf16 pairs) | O(group)
  const uint32_t TS_BASE = 0, TS_OWN = (uint32_t)TP, TS_P = (uint32_t)TP + 128,
                 TS_O = TS_P + (uint32_t)(TP + 128) / 2;
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const float sl2 = scale * 1.4426950408889634f;
  uint32_t ph_s = 0, ph_o = 0, ph_p = 0, hc = 0;

  // item it = (tile j of this CTA, head group gi), it = j G + gi; counters
  // advance incrementally (no integer division in the loop)
  auto tile_of = [&](int j) { return tiles[blockIdx.x + j * gridDim.x]; };
  auto kb_of = [&](int tp) {
    const int m = max(max(wmax[tp * 4 + 0], wmax[tp * 4 + 1]),
                      max(wmax[tp * 4 + 2], wmax[tp * 4 + 3]));
    return (m + 15) & ~15;  // base keys any row of the tile uses
  };
  // stage the operands of item `it` (cp.async, zero-filled tails); the first
  // item of a tile first lays out the tile's row table
  auto prefetch = [&](int it, int j, int gi) {
    if (it >= nit) return;
    const int tp = j & 1;
    if (gi == 0) {
      const AttnTile tl = tile_of(j);
      if (part == 0) {
        const int64_t uo = Uoff[tl.sample], base = act_off[tl.sample];
        const bool lv = row < tl.nloc;
        int a = 0, lo = 1 << 20;
        if (lv) {
          const int64_t loc = tl.loc0 + row;
          const int r = lrow[loc];
          const int p = lpos[loc];
          a = (r % R1) == 0 ? 0 : row_t1[r] + 1;
          lo = row - (p - a);
        }
        rowq[tp * 128 + row] = lv ? (uo + I[tl.loc0 + row]) * ld : -1;
        rowb[tp * 128 + row] = row < T ? (uo + I[base + row]) * ld : -1;
        inf_a[tp * 128 + row] = a;
        inf_lo[tp * 128 + row] = lo;
        const int wm = warp_max_i(a);
        if (lane == 0) wmax[tp * 4 + warp] = wm;
      }
      __syncthreads();
    }
    const uint32_t st = sb + (uint32_t)(it & 1) * L.stage;
    const int64_t* rq = rowq + tp * 128;
    const int64_t* rb = rowb + tp * 128;
    for (int e = tid; e < 128 * 8; e += TCA_THREADS) {
      const int r = e >> 3, c = e & 7;
      const int64_t off = rq[r];
      const bool ok = off >= 0;
      const bf16* src = qkv + (ok ? off : 0) + gi * 64 + c * 8;
      const uint32_t o = tc::sw128_chunk(r, c);
      tc::cp_async16_zfill(st + L.q + o, src, ok);
      tc::cp_async16_zfill(st + L.kown + o, src + d, ok);
      tc::cp_async16_zfill(st + L.vown + o, src + 2 * d, ok);
    }
    for (int e = tid; e < 64 * KBb * 8; e += TCA_THREADS) {
      const int t = e >> 3, c = e & 7;
      const int64_t off = t < 128 ? rb[t] : -1;
      const bool ok = off >= 0;
      const bf16* src = qkv + (ok ? off : 0) + d + gi * 64 + c * 8;
      const uint32_t o = tc::sw128_chunk(t, c);
      tc::cp_async16_zfill(st + L.kbase + o, src, ok);
      tc::cp_async16_zfill(st + L.vbase + o, src + d, ok);
    }
    tc::cp_async_commit();
  };
  // S_base = Q K_base^T, S_own = Q K_own^T for head hq of item it (one thread)
  auto issue_scores = [&](int it, int hq, int kb_base) {
    const uint32_t st = sb + (uint32_t)(it & 1) * L.stage;
    const uint32_t qoff = (uint32_t)(hq * dh * 2);  // head offset inside the 128-B row
    const uint32_t idS_b = tc::make_idesc_bf16(128, kb_base > 0 ? kb_base : 16);
    const uint32_t idS_o = tc::make_idesc_bf16(128, 128);
    for (int k = 0; k < dh / 16; ++k) {
      if (kb_base > 0)
        tc::mma_bf16(tmem + TS_BASE, tc::make_desc_sw128(st + L.q + qoff + k * 32),
                     tc::make_desc_sw128(st + L.kbase + qoff + k * 32), idS_b, k != 0);
      tc::mma_bf16(tmem + TS_OWN, tc::make_desc_sw128(st + L.q + qoff + k * 32),
                   tc::make_desc_sw128(st + L.kown + qoff + k * 32), idS_o, k != 0);
    }
    tc::mma_commit(&mbar[0]);
  };

  prefetch(0, 0, 0);
  prefetch(1, G == 1 ? 1 : 0, G == 1 ? 0 : 1);
  tc::cp_async_wait<1>();
  tc::fence_proxy_async();
  __syncthreads();
  if (tid == 0 && nit > 0) {
    tc::fence_after();
    issue_scores(0, 0, kb_of(0));
  }

  // per-tile thread state
  bool live = false;
  int64_t myloc = 0;
  int kb_base = 0;
  int nb = 0, nq = 0, wo_beg = 0;  // warp's live chunks: nb base + (nq - nb) own from wo_beg
  int nbf = 0;                     // base chunks every live row of the warp uses entirely
  int a = 0, own_lo = 0, own_cnt = 0;
  float xn2 = 0.f, rr2 = 0.f;
  int j = 0, gi = 0;  // item it = (j, gi)
  for (int it = 0; it < nit; ++it) {
    const int tp = j & 1;
    const int j1 = gi + 1 == G ? j + 1 : j, g1 = gi + 1 == G ? 0 : gi + 1;  // item it + 1
    const uint32_t st = sb + (uint32_t)(it & 1) * L.stage;
    if (gi == 0) {
      const AttnTile tl = tile_of(j);
      live = row < tl.nloc;
      myloc = tl.loc0 + row;
      a = inf_a[tp * 128 + row];
      own_lo = inf_lo[tp * 128 + row];
      own_cnt = live ? row - own_lo + 1 : 0;
      kb_base = kb_of(tp);
      const int wb_end = (warp_max_i(a) + 15) & ~15;
      const int w_olo = warp_min_i(live ? own_lo : 1 << 20);
      const int w_ohi = warp_max_i(live ? row : -1);
      wo_beg = w_olo >= 128 ? 128 : (w_olo & ~15);
      const int wo_end = w_ohi < 0 ? 0 : ((w_ohi + 16) & ~15);
      nb = wb_end >> 4;
      nbf = warp_min_i(live ? a : 1 << 20) >> 4;
      nq = nb + max(0, (wo_end - wo_beg) >> 4);
      xn2 = 0.f;
      rr2 = 0.f;
      // P columns no warp writes this tile must read as zero
      const int pcols = (kb_base + 128) / 2;
      const uint32_t zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int c = part * 8; c < pcols; c += 32) tc::tmem_st8u(trow + TS_P + c, zero);
      tc::tmem_wait_st();
    }
    for (int hh = 0; hh < hpg; ++hh) {
      const uint32_t koff = (uint32_t)(hh * dh * 2);  // head offset inside the 128-B row
      tc::mbar_wait(&mbar[0], ph_s);
      ph_s ^= 1;
      tc::fence_after();
      // ---- the warp's live 16-column chunks (base chunks, then own chunks)
      // are dealt round-robin to the four warpgroups: slot i is chunk part + 4i.
      // ONE TMEM pass loads them into registers.
      float v[4][16];
      bool sl[4];
      int off[4], cnt[4];
      uint32_t pcol[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int q = part + 4 * i;
        sl[i] = q < nq;
        const bool isb = q < nb;
        const int c0 = isb ? 16 * q : wo_beg + 16 * (q - nb);
        off[i] = isb ? c0 : c0 - own_lo;  // entry j is live iff 0 <= off + j < cnt
        cnt[i] = isb ? a : own_cnt;
        pcol[i] = (uint32_t)((isb ? c0 : kb_base + c0) >> 1);
        if (sl[i]) tc::tmem_ld16(trow + (isb ? TS_BASE : TS_OWN) + c0, v[i]);
      }
      tc::tmem_wait_ld();
      // ---- local max and sum of exp2((s - m_part) * scale * log2e)
      float mp = -INFINITY;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (!sl[i]) continue;
        if (part + 4 * i < nbf) {
#pragma unroll
          for (int j = 0; j < 16; ++j) mp = fmaxf(mp, v[i][j]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const bool ok = (unsigned)(off[i] + j) < (unsigned)cnt[i];
            v[i][j] = ok ? v[i][j] : -INFINITY;
            mp = fmaxf(mp, v[i][j]);
          }
        }
      }
      const float mref = mp == -INFINITY ? 0.f : mp * sl2;
      float sp = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (!sl[i]) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          v[i][j] = ex2_approx(fmaf(v[i][j], sl2, -mref));
          sp += v[i][j];
        }
      }
      const int xb = hc & 1;
      ++hc;
      red[xb][part][row] = make_float2(mp, sp);
      tc::fence_before();
      __syncthreads();
      if (tid == 0 && hh + 1 < hpg) {
        // every warp holds its scores in registers: the next head's score
        // MMA overlaps this head's softmax and value MMA
        tc::fence_after();
        issue_scores(it, hh + 1, kb_base);
      }
      float2 rq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) rq[q] = red[xb][q][row];
      const float m = fmaxf(fmaxf(rq[0].x, rq[1].x), fmaxf(rq[2].x, rq[3].x));
      float tot = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) tot += rq[q].y > 0.f ? rq[q].y * ex2_approx((rq[q].x - m) * sl2) : 0.f;
      const float f = sp > 0.f ? __fdividef(ex2_approx((mp - m) * sl2), tot) : 0.f;
      // P is rewritten only after the previous head's value MMA consumed it
      if (hh > 0) {
        tc::mbar_wait(&mbar[1], ph_o);
        ph_o ^= 1;
      }
      // ---- normalised bf16 probabilities into the TMEM P tile
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (!sl[i]) continue;
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 16; j += 2) pk[j / 2] = tc::pack_bf16(v[i][j] * f, v[i][j + 1] * f);
        tc::tmem_st8u(trow + TS_P + pcol[i], pk);
      }
      tc::tmem_wait_st();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&mbar[2]));
      // ---- O_h = P_base V_base + P_own V_own  (P from TMEM, V the MN-major B operand)
      if (tid == 0) {
        tc::mbar_wait(&mbar[2], ph_p);
        tc::fence_after();
        const uint32_t idO = tc::make_idesc_bf16(128, dh) | (1u << 16);
        int first = 1;
        for (int k16 = 0; k16 < kb_base; k16 += 16) {
          tc::mma_bf16_ts(tmem + TS_O + hh * dh, tmem + TS_P + (uint32_t)(k16 >> 1),
                          tc::make_desc_sw128(st + L.vbase + (uint32_t)k16 * 128 + koff), idO,
                          first ? 0u : 1u);
          first = 0;
        }
        for (int k16 = 0; k16 < 128; k16 += 16) {
          tc::mma_bf16_ts(tmem + TS_O + hh * dh, tmem + TS_P + (uint32_t)((kb_base + k16) >> 1),
                          tc::make_desc_sw128(st + L.vown + (uint32_t)k16 * 128 + koff), idO,
                          first ? 0u : 1u);
          first = 0;
        }
        tc::mma_commit(&mbar[1]);
      }
      ph_p ^= 1;
    }
    // ---- next item's operands landed -> its first score MMA runs while this
    // item's O drains
    if (it + 1 < nit) {
      tc::cp_async_wait<0>();
      tc::fence_proxy_async();
    }
    tc::fence_before();
    __syncthreads();
    if (tid == 0 && it + 1 < nit) {
      tc::fence_after();
      issue_scores(it + 1, 0, kb_of(j1 & 1));
    }
    tc::mbar_wait(&mbar[1], ph_o);  // the item's last value MMA
    ph_o ^= 1;
    tc::fence_after();
    // ---- drain O: warpgroup `part` takes columns [16 part, 16 part + 16)
    {
      float o[16];
      tc::tmem_ld16(trow + TS_O + part * 16, o);  // warp-collective: every lane loads
      tc::tmem_wait_ld();
      if (live) {
        uint32_t ph[8], pl[8];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          ph[j / 2] = tc::pack_bf16(o[j], o[j + 1]);
          const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&ph[j / 2]);
          const float d0 = o[j] - __low2float(h), d1 = o[j + 1] - __high2float(h);
          pl[j / 2] = tc::pack_bf16(d0, d1);
          const __nv_bfloat162 l = *reinterpret_cast<const __nv_bfloat162*>(&pl[j / 2]);
          const float r0 = __low2float(l), r1 = __high2float(l);  // |xl|^2 (tc_vq.cuh)
          xn2 = fmaf(o[j], o[j], fmaf(o[j + 1], o[j + 1], xn2));
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
    if (gi == G - 1) {
      // row norms |x|^2 and |x - xh - xl|^2, reduced over the four warpgroups
      nrm[0][part][row] = xn2;
      nrm[1][part][row] = rr2;
      __syncthreads();
      if (part == 0 && live) {
        xn2_out[myloc] = ((nrm[0][0][row] + nrm[0][1][row]) + nrm[0][2][row]) + nrm[0][3][row];
        rr2_out[myloc] = ((nrm[1][0][row] + nrm[1][1][row]) + nrm[1][2][row]) + nrm[1][3][row];
      }
    }
    // into this item's stage: every MMA reading it has completed
    prefetch(it + 2, g1 + 1 == G ? j1 + 1 : j1, g1 + 1 == G ? 0 : g1 + 1);
    j = j1;
    gi = g1;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

inline bool tc_attn_ok(int prec, int d, int dh, int T) {
  return prec == 1 && d % 64 == 0 && (dh == 16 || dh == 32 || dh == 64) && T <= 128;
}

}  // namespace vqb

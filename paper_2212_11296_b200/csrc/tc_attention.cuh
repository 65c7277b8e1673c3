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
// issued as soon as every warp holds its scores; dedicated drain warps empty
// an item's O while the softmax warps work on the next item.
// TMEM: S_base | S_own | P (bf16 pairs) | O(even item) | O(odd item)
//       = 1.5 (T_pad + 128) + 128 <= 512.
//
// Outputs per active location: the attention row x as its two-term bf16
// split xh = bf16(x), xl = bf16(x - xh) (the VQ distance GEMM operands; x is
// represented to 2^-18 relative), |x|^2 and |x - xh - xl|^2 (the certified
// argmin error bound, tc_vq.cuh). Warp w reads TMEM lanes 32(w%4).. (its
// query rows); the warp roles are listed above k_tc_attention.
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

// Packing of whole rows (consecutive in active-location order) into tiles of
// <= 128 locations: a tile ends where k_connected marked the next row as a
// tile start, or (unmarked orders: the no-reuse regime) where the next row
// no longer fits. One thread per sample, in two passes: pass 0
// counts each sample's tiles (tcnt), pass 1 writes them at the sample's
// exclusive-scan offset (toff, k_scan) so a sample's tiles are contiguous in
// the tile list. The persistent attention kernel deals tiles round-robin over
// the CTAs, so the CTAs then work on the same few samples at a time and the
// samples' shared base-row K/V stay in L2.
__global__ void k_build_tiles(int pass, int S, int R1, int T, int cap,
                              const int32_t* __restrict__ K,
                              const int32_t* __restrict__ row_t1,
                              const int32_t* __restrict__ row_perm,
                              const int64_t* __restrict__ act_off, int32_t* __restrict__ tcnt,
                              const int64_t* __restrict__ toff, const int64_t* __restrict__ ttot,
                              AttnTile* __restrict__ tiles, int32_t* __restrict__ n_tiles) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (pass == 1 && s == 0) *n_tiles = (int32_t)*ttot;
  if (s >= S) return;
  const int Ks = K[s];
  int cur = 0, nt = 0, amax = 0;
  bool cut = false;
  int64_t start = act_off[s];
  const int64_t base = pass == 1 ? toff[s] : 0;
  for (int i = 0; i < Ks; ++i) {  // rows in active-layout order (k_connected)
    const int kf = row_perm[(int64_t)s * R1 + i];  // bit 30: first row of a tile (k_connected)
    const int k = kf & ~(1 << 30);
    const int n = k == 0 ? T : T - (row_t1[(int64_t)s * R1 + k] + 1);
    cut |= kf != k;
    if (n <= 0) continue;
    // score columns of the tile: base keys up to the largest a, then own keys
    const int cols = ((max(amax, T - n) + 15) & ~15) + ((cur + n + 15) & ~15);
    if (cur > 0 && (cur + n > 128 || cols > cap || cut)) {
      if (pass == 1) tiles[base + nt] = AttnTile{s, cur, start};
      ++nt;
      start += cur;
      cur = 0;
      amax = 0;
    }
    cur += n;
    amax = max(amax, T - n);
    cut = false;
  }
  if (cur > 0) {
    if (pass == 1) tiles[base + nt] = AttnTile{s, cur, start};
    ++nt;
  }
  if (pass == 0) tcnt[s] = nt;
}

__host__ __device__ inline int attn_tpad(int T) { return ((T + 15) / 16) * 16; }
__host__ __device__ inline int attn_kb_base(int T) { return (attn_tpad(T) + 63) / 64; }

__device__ __forceinline__ int warp_max_i(int v) { return __reduce_max_sync(0xffffffffu, v); }
__device__ __forceinline__ int warp_min_i(int v) { return __reduce_min_sync(0xffffffffu, v); }

// Per-tile row table, rebuilt per layer (the qkv row of a location depends on
// the layer's dedup). 1552 bytes per tile, fetched by the attention kernel
// with plain 16-byte async copies one tile ahead:
//   [0, 512)     int32 qkv row of tile row r (-1 past the tile)
//   [512, 1024)  int32 qkv row of base-row position t (-1 for t >= T)
//   [1024, 1280) int16 a_r: base keys of row r
//   [1280, 1536) int16 own_lo_r: first own key (tile row) of row r
//   [1536, 1552) int64 loc0, int32 nloc, int32 kb_base (16 ceil(max a))
constexpr int TINFO_BYTES = 1552;

__global__ void __launch_bounds__(128) k_tile_info(
    const AttnTile* __restrict__ tiles, const int32_t* __restrict__ n_tiles_p, int R1, int T,
    const int32_t* __restrict__ row_t1, const int64_t* __restrict__ act_off,
    const int32_t* __restrict__ lrow, const int16_t* __restrict__ lpos,
    const int32_t* __restrict__ I, const int64_t* __restrict__ Uoff,
    uint8_t* __restrict__ tinfo) {
  __shared__ int wm[4];
  const int n_tiles = *n_tiles_p;
  const int r = threadIdx.x;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const AttnTile tl = tiles[t];
    uint8_t* blk = tinfo + (int64_t)t * TINFO_BYTES;
    const int64_t uo = Uoff[tl.sample], base = act_off[tl.sample];
    const bool lv = r < tl.nloc;
    int a = 0, lo = 0x7fff;
    if (lv) {
      const int64_t loc = tl.loc0 + r;
      const int rr = lrow[loc];
      const int p = lpos[loc];
      a = (rr % R1) == 0 ? 0 : row_t1[rr] + 1;
      lo = r - (p - a);
    }
    reinterpret_cast<int32_t*>(blk)[r] = lv ? (int32_t)(uo + I[tl.loc0 + r]) : -1;
    reinterpret_cast<int32_t*>(blk + 512)[r] = r < T ? (int32_t)(uo + I[base + r]) : -1;
    reinterpret_cast<int16_t*>(blk + 1024)[r] = (int16_t)a;
    reinterpret_cast<int16_t*>(blk + 1280)[r] = (int16_t)lo;
    const int m = warp_max_i(a);
    if ((r & 31) == 0) wm[r >> 5] = m;
    __syncthreads();
    if (r == 0) {
      *reinterpret_cast<int64_t*>(blk + 1536) = tl.loc0;
      reinterpret_cast<int32_t*>(blk + 1544)[0] = tl.nloc;
      reinterpret_cast<int32_t*>(blk + 1544)[1] =
          (max(max(wm[0], wm[1]), max(wm[2], wm[3])) + 15) & ~15;
    }
    __syncthreads();
  }
}

// shared memory carve (bytes; stages 1024-aligned). Two staging buffers, each
// q | k_own | v_own (128 x 64) | k_base | v_base (64 KBb x 64), so the operands
// of the next (tile, head group) item load while the current one computes;
// four tile-table slots (fetched one tile ahead); the O staging tile for
// coalesced stores (xh | xl, 128 rows x 144 B: conflict-free 16-B writes).
constexpr int ATT_OPITCH = 144;
struct AttnSmem {
  uint32_t stage, q, kown, vown, kbase, vbase, info, out, bar, total;
  __host__ __device__ AttnSmem(int T) {
    const uint32_t KBb = (uint32_t)attn_kb_base(T);
    q = 0;
    kown = 128 * 128;
    vown = 2 * 128 * 128;
    kbase = 3 * 128 * 128;
    vbase = kbase + 64 * KBb * 128;
    stage = vbase + 64 * KBb * 128;
    info = 2 * stage;
    out = info + 8 * TINFO_BYTES;
    bar = out + 2 * 128 * ATT_OPITCH;
    total = bar + 160;  // 18 mbarriers, TMEM base
  }
};

#if defined(VQNQS_ATTN_TL)
// timeline mode: raw clock() of every trace point for three consecutive heads
#define VQNQS_TL_H0 (200 + 24 * (int)blockIdx.x)
#define ATR_DECL int tl_h = -1;
#define ATR(k) { if ((unsigned)tl_h < 3u) tlog[warp][tl_h * 16 + (k)] = (unsigned)clock(); }
#define MTR_DECL int tl_h = -VQNQS_TL_H0 - 1;
#define MTR(k) ATR(k)
#elif defined(VQNQS_ATTN_TRACE)
#define ATR_DECL unsigned long long atr[16] = {0}; long long atr_t = clock64();
#define ATR(k) { const long long _n = clock64(); atr[k] += _n - atr_t; atr_t = _n; }
#define MTR_DECL unsigned mtr[8] = {0}; unsigned mtr_t = (unsigned)clock();
#define MTR(k) { const unsigned _n = (unsigned)clock(); mtr[k] += _n - mtr_t; mtr_t = _n; }
#else
#define ATR_DECL
#define ATR(k)
#define MTR_DECL
#define MTR(k)
#endif

// exp2 of a pair on the FMA pipe, for moving part of the softmax exponentials
// off the MUFU unit (16 lanes / clock / SM): 2^t = 2^n 2^f with n = rint(t),
// f = t - n in [-1/2, 1/2], 2^f by a degree-5 minimax polynomial (relative
// error 1.8e-7 in fp32 Horner, the accuracy of ex2.approx), 2^n added to the
// exponent field. t is clamped to -127, where the result is exactly +0 (the
// masked entries, t = -inf). VQNQS_ATTN_EMU_PAIRS of the 8 pairs per score
// chunk take this path; measured on c4 / c5 0 is as fast as 2
// and faster than 3 or 4: the softmax warps are latency-, not MUFU-bound.
#ifndef VQNQS_ATTN_SWP
#define VQNQS_ATTN_SWP 1
#endif
#ifndef VQNQS_ATTN_EMU_PAIRS
#define VQNQS_ATTN_EMU_PAIRS 0
#endif
__device__ __forceinline__ float2 ex2_poly2(float2 t) {
  constexpr float M = 12582912.0f;  // 1.5 * 2^23: t + M rounds t to an integer
  t.x = fmaxf(t.x, -127.f);
  t.y = fmaxf(t.y, -127.f);
  const float2 j = tc::fadd2(t, make_float2(M, M));
  const float2 n = tc::fadd2(j, make_float2(-M, -M));
  const float2 f = tc::ffma2(n, make_float2(-1.f, -1.f), t);
  float2 p = tc::ffma2(make_float2(1.3264698209241033e-3f, 1.3264698209241033e-3f), f,
                       make_float2(9.671509265899658e-3f, 9.671509265899658e-3f));
  p = tc::ffma2(p, f, make_float2(5.550733953714371e-2f, 5.550733953714371e-2f));
  p = tc::ffma2(p, f, make_float2(2.4022242426872253e-1f, 2.4022242426872253e-1f));
  p = tc::ffma2(p, f, make_float2(6.931470036506653e-1f, 6.931470036506653e-1f));
  p = tc::ffma2(p, f, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 16 softmax warps (warp w: TMEM lanes 32(w%4).., column slots of warpgroup
// w/4) + one MMA warp. All hand-offs are mbarriers or quadrant-local named
// barriers (the four warps that share a row quadrant), so no block barrier
// runs per head or per item:
//   s_full   (MMA commit)      S(g) in TMEM
//   s_free   (16 warp arrivals) every warp holds S(g) in registers
//   p_full   (16 warp arrivals) P(g) written to TMEM
//   pv_done  (MMA commit)      O += P(g) V done, P free
//   st_full[2]   (3 producer warps) the item's cp.async operands landed
//   stage_free[2] (MMA commit)     every MMA of the item done (operands free,
//                                   its O complete)
//   o_empty[2]   (4 drain warps)   the item's O buffer drained
//   info_ready[8] (3 producer warps) a tile table landed
// Warpgroups: four softmax warpgroups; two drain warpgroups (warp 16 + 4h + q
// drains half h of row quadrant q's O, double-buffered by item in TMEM, into
// xh / xl and the row norms, so no softmax warp waits for an item's last
// value MMA); and the MMA warpgroup (warp 24 issues every tcgen05.mma, warps
// 25-27 stage the operands with cp.async). setmaxnreg redistributes the
// 896 x 72 launch registers: softmax 96, drain 40, MMA / producers 32.
#ifndef VQNQS_TCA_PARTS
#define VQNQS_TCA_PARTS 4
#endif
constexpr int TCA_PARTS = VQNQS_TCA_PARTS;  // softmax warps per row quadrant (they split its score chunks)
constexpr int TCA_SLOTS = (16 + TCA_PARTS - 1) / TCA_PARTS;  // chunks per softmax warp
static_assert(TCA_PARTS == 4 || TCA_PARTS == 6, "softmax warps per quadrant");
constexpr int TCA_SOFTMAX_WARPS = 4 * TCA_PARTS;
constexpr int TCA_SOFTMAX_REGS = TCA_PARTS == 6 ? 72 : 96;
constexpr int TCA_DRAIN_WARP0 = TCA_SOFTMAX_WARPS;
// Drain warps per CTA (template parameter NDRAIN): 4 (one per row quadrant,
// 64 columns) when an item holds two or more heads (dh <= 32: an O buffer is
// drained once per hpg heads, and four fewer warps compete with the softmax
// warps: c4 +1.8%), 8 (two per quadrant, 32 columns each) when every head
// ends an item (dh = 64: c5 is 4% slower with 4).
constexpr int tca_threads(int ndrain) { return 32 * (TCA_DRAIN_WARP0 + ndrain + 4); }
inline int tca_drain_warps(int dh) { return dh <= 32 ? 4 : 8; }

template <int NDRAIN>
__global__ void __launch_bounds__(tca_threads(NDRAIN), 1) k_tc_attention(
    const uint8_t* __restrict__ tinfo, const int32_t* __restrict__ n_tiles_p, int T, int d,
    int dh, float scale, const bf16* __restrict__ qkv, bf16* __restrict__ xh_out,
    bf16* __restrict__ xl_out, float* __restrict__ xn2_out, float* __restrict__ rr2_out) {
  constexpr int TCA_DRAIN_WARPS = NDRAIN;
  constexpr int TCA_DRAIN_REGS = NDRAIN == 4 ? 48 : 40;
  constexpr int TCA_DRAIN_COLS = 64 * 4 / NDRAIN;
  constexpr int TCA_MMA_WARP = TCA_DRAIN_WARP0 + NDRAIN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const AttnSmem L(T);
  // 8 tile-table slots (k_tile_info layout): tile j + 8 is fetched at item
  // (j + 7, 0), after the MMAs of item (j + 7) G - 2 and hence after the drain
  // of item (j + 7) G - 4 >= j G read tile j's table
  const uint8_t* info = smem + L.info;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* s_full = mbar + 0;
  uint64_t* s_free = mbar + 1;
  uint64_t* p_full = mbar + 2;
  uint64_t* pv_done = mbar + 3;
  uint64_t* st_full = mbar + 4;     // [2]
  uint64_t* stage_free = mbar + 6;  // [2]
  uint64_t* o_empty = mbar + 8;     // [2]
  uint64_t* info_ready = mbar + 10;  // [8]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 18);
  // exchange buffers alternate by head: a fast warp may publish head h+1
  // before a slow one of its quadrant has read head h
  __shared__ float2 red[2][TCA_PARTS][128];  // (local max, local sum)
  __shared__ float2 dnrm[128];       // drain warps' partial row norms
#ifdef VQNQS_ATTN_TL
  __shared__ unsigned tlog[32][48];
  for (int i = threadIdx.x; i < 32 * 48; i += blockDim.x) (&tlog[0][0])[i] = 0;
#endif
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
    tc::mbar_init(s_full, 1);
    tc::mbar_init(s_free, TCA_SOFTMAX_WARPS);
    tc::mbar_init(p_full, TCA_SOFTMAX_WARPS);
    tc::mbar_init(pv_done, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&st_full[i], 3);  // the three producer warps
      tc::mbar_init(&stage_free[i], 1);
      tc::mbar_init(&o_empty[i], TCA_DRAIN_WARPS);
    }
    for (int i = 0; i < 8; ++i) tc::mbar_init(&info_ready[i], 3);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sb = tc::smem_u32(smem);
  // TMEM columns: S_base | S_own | P (bf16 pairs) | O(even items) | O(odd items)
  const uint32_t TS_BASE = 0, TS_OWN = (uint32_t)TP, TS_P = (uint32_t)TP + 128,
                 TS_O = TS_P + (uint32_t)(TP + 128) / 2;
  auto slot = [&](int j) { return info + (j & 7) * TINFO_BYTES; };
  auto kb_of = [&](int j) { return reinterpret_cast<const int32_t*>(slot(j) + 1548)[0]; };

  if (warp >= TCA_DRAIN_WARP0 && warp < TCA_MMA_WARP) {
    // ================= drain warps: item O -> xh | xl and the row norms.
    // Warp 16 + 4 h + q drains columns [h C, h C + C) of row quadrant q.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(TCA_DRAIN_REGS) : "memory");
    constexpr int C = TCA_DRAIN_COLS, NH = TCA_DRAIN_WARPS / 4;
    const int q = warp & 3, hf = (warp - TCA_DRAIN_WARP0) >> 2;
    const int row = q * 32 + lane;
    const uint32_t trq = tmem + ((uint32_t)(q * 32) << 16);
    float xn2 = 0.f, rr2 = 0.f;
    int dnloc = 0;
    int64_t dloc0 = 0;
    int j = 0, gi = 0;
    for (int it = 0; it < nit; ++it) {
      if (gi == 0) {
        tc::mbar_wait(&info_ready[j & 7], (j >> 3) & 1);
        const uint8_t* ti = slot(j);
        dnloc = reinterpret_cast<const int32_t*>(ti + 1544)[0];
        dloc0 = *reinterpret_cast<const int64_t*>(ti + 1536);
        xn2 = 0.f;
        rr2 = 0.f;
      }
      tc::mbar_wait(&stage_free[it & 1], (it >> 1) & 1);  // the item's O is complete
      tc::fence_after();
      const uint32_t ob = sb + L.out + (uint32_t)(row * ATT_OPITCH);
#pragma unroll 1
      for (int c16 = hf * C; c16 < hf * C + C; c16 += 16) {
        float o[16];
        tc::tmem_ld16(trq + TS_O + (uint32_t)((it & 1) * 64 + c16), o);
        tc::tmem_wait_ld();
        uint32_t ph[8], pl[8];
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          ph[k / 2] = tc::pack_bf16(o[k], o[k + 1]);
          const float h0 = __uint_as_float(ph[k / 2] << 16);
          const float h1 = __uint_as_float(ph[k / 2] & 0xffff0000u);
          pl[k / 2] = tc::pack_bf16(o[k] - h0, o[k + 1] - h1);
          const float r0 = __uint_as_float(pl[k / 2] << 16);
          const float r1 = __uint_as_float(pl[k / 2] & 0xffff0000u);  // |xl|^2 (tc_vq.cuh)
          xn2 = fmaf(o[k], o[k], fmaf(o[k + 1], o[k + 1], xn2));
          rr2 = fmaf(r0, r0, fmaf(r1, r1, rr2));
        }
        tc::st_shared_v4(ob + c16 * 2, ph[0], ph[1], ph[2], ph[3]);
        tc::st_shared_v4(ob + c16 * 2 + 16, ph[4], ph[5], ph[6], ph[7]);
        tc::st_shared_v4(ob + 128 * ATT_OPITCH + c16 * 2, pl[0], pl[1], pl[2], pl[3]);
        tc::st_shared_v4(ob + 128 * ATT_OPITCH + c16 * 2 + 16, pl[4], pl[5], pl[6], pl[7]);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&o_empty[it & 1]));  // O buffer free
      // the warp's 32 rows x C columns, xh then xl: 64 segments of 2C bytes,
      // C / 8 lanes per segment. With C = 32 a shared-memory phase (8 lanes)
      // reads two rows: rows 4 apart (16 banks apart at the 144-B pitch) so
      // the two 64-B halves never share a bank.
      constexpr int LPS = C / 8, SPI = 32 / LPS;
      const int sub = lane / LPS;
      const int subr = SPI == 8 ? (((sub & 1) << 2) | (sub >> 1)) : sub;
#pragma unroll 4
      for (int k = 0; k < 64 / SPI; ++k) {
        const int seg = k * SPI + subr;  // 0..63
        const int rr = q * 32 + (seg & 31);
        const int cc = hf * C + (lane % LPS) * 8;
        if (rr < dnloc) {
          const uint32_t src = sb + L.out + (uint32_t)((seg >> 5) * 128 * ATT_OPITCH +
                                                       rr * ATT_OPITCH + cc * 2);
          uint32_t w0, w1, w2, w3;
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                       : "r"(src));
          bf16* dst = ((seg >> 5) ? xl_out : xh_out) + (dloc0 + rr) * d + gi * 64 + cc;
          *reinterpret_cast<uint4*>(dst) = make_uint4(w0, w1, w2, w3);
        }
      }
      __syncwarp();
      if (gi == G - 1) {
        // row norms |x|^2 and |x - xh - xl|^2 over the tile's head groups
        if constexpr (NH == 2) {
          if (hf == 1) dnrm[row] = make_float2(xn2, rr2);
          asm volatile("bar.sync %0, 64;" ::"r"(7 + q) : "memory");
          if (hf == 0) {
            const float2 o2 = dnrm[row];
            xn2 += o2.x;
            rr2 += o2.y;
          }
          asm volatile("bar.sync %0, 64;" ::"r"(7 + q) : "memory");
        }
        if (hf == 0 && row < dnloc) {
          xn2_out[dloc0 + row] = xn2;
          rr2_out[dloc0 + row] = rr2;
        }
      }
      if (++gi == G) {
        gi = 0;
        ++j;
      }
    }
  } else if (warp >= TCA_MMA_WARP) {
    // ================= MMA warp (one thread issues every tcgen05.mma)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 32;" ::: "memory");
    if (warp == TCA_MMA_WARP && nit > 0) {
      // The whole warp runs the (warp-uniform) schedule and one elected lane
      // issues, so descriptors stay in uniform registers and the MMA loops
      // are unrolled: this thread's issue latency paces the tensor pipe
      // (scripts/mma_probe2.cu: a 12-step value chain completes in ~270
      // cycles when issued unrolled).
      const bool leader = tc::elect_one();
      auto own_of = [&](int j) {  // own key columns in use: 16 ceil(nloc / 16)
        return (reinterpret_cast<const int32_t*>(slot(j) + 1544)[0] + 15) & ~15;
      };
      auto issue_scores = [&](int it, int hq, int kb_base, int nown) {
        const uint32_t st = sb + (uint32_t)(it & 1) * L.stage;
        const uint32_t qoff = (uint32_t)(hq * dh * 2);  // head offset inside the 128-B row
        const uint32_t idS_b = tc::make_idesc_bf16(128, kb_base > 0 ? kb_base : 16);
        const uint32_t idS_o = tc::make_idesc_bf16(128, nown);
        const uint64_t dq = tc::make_desc_sw128(st + L.q + qoff);
        const uint64_t dkb = tc::make_desc_sw128(st + L.kbase + qoff);
        const uint64_t dko = tc::make_desc_sw128(st + L.kown + qoff);
        if (leader) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // +32 B along K = +2 in the descriptor
            if (k < dh / 16) {
              if (kb_base > 0) tc::mma_bf16(tmem + TS_BASE, dq + 2 * k, dkb + 2 * k, idS_b, k != 0);
              tc::mma_bf16(tmem + TS_OWN, dq + 2 * k, dko + 2 * k, idS_o, k != 0);
            }
          }
          tc::mma_commit(s_full);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int it, int hh, int kb_base, int nown) {
        const uint32_t st = sb + (uint32_t)(it & 1) * L.stage;
        const uint32_t koff = (uint32_t)(hh * dh * 2);
        const uint32_t idO = tc::make_idesc_bf16(128, dh) | (1u << 16);
        const uint32_t tO = tmem + TS_O + (uint32_t)((it & 1) * 64 + hh * dh), tA = tmem + TS_P;
        const uint64_t db = tc::make_desc_sw128(st + L.vbase + koff);
        const uint64_t dw = tc::make_desc_sw128(st + L.vown + koff);
        const int nb16 = kb_base >> 4, no16 = nown >> 4;
        if (leader) {
          // descriptor start field is address >> 4: 16 key rows = +128
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (i < nb16) tc::mma_bf16_ts(tO, tA + 8u * i, db + 128u * i, idO, i > 0 ? 1u : 0u);
          const uint32_t tAo = tA + (uint32_t)(kb_base >> 1);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (i < no16)
              tc::mma_bf16_ts(tO, tAo + 8u * i, dw + 128u * i, idO, (nb16 > 0 || i > 0) ? 1u : 0u);
          tc::mma_commit(pv_done);
        }
        __syncwarp();
      };
      uint32_t ph_free = 0, ph_p = 0;
      MTR_DECL
#ifdef VQNQS_ATTN_TRACE2
      uint32_t ph_sf = 1, ph_pv = 0;  // S(0)'s phase is not waited for here
#endif
      // S(0)
      tc::mbar_wait(&st_full[0], 0);
      tc::fence_after();
      int kb_cur = kb_of(0), no_cur = own_of(0);
      issue_scores(0, 0, kb_cur, no_cur);
      int it = 0, hh = 0, j = 0, gi = 0;  // head g = (it, hh), item it = (j, gi)
      for (;;) {
        // next head (it2, hh2)
        int it2 = it, hh2 = hh + 1, j2 = j, gi2 = gi;
        if (hh2 == hpg) {
          hh2 = 0;
          it2 = it + 1;
          if (++gi2 == G) {
            gi2 = 0;
            ++j2;
          }
        }
        int kb_next = kb_cur, no_next = no_cur;
        MTR(0)
#ifdef VQNQS_ATTN_TL
        ++tl_h;
        MTR(8)
#endif
        if (it2 < nit) {
          tc::mbar_wait(s_free, ph_free);  // every warp holds S(g)
          ph_free ^= 1;
          MTR(1)
          if (it2 != it) {
            tc::mbar_wait(&st_full[it2 & 1], (it2 >> 1) & 1);  // operands of item it2
            kb_next = kb_of(j2);
            no_next = own_of(j2);
          }
          tc::fence_after();
          MTR(2)
          issue_scores(it2, hh2, kb_next, no_next);
          MTR(3)
#ifdef VQNQS_ATTN_TRACE2
          tc::mbar_wait(s_full, ph_sf);
          ph_sf ^= 1;
          MTR(7)
#endif
        }
        if (hh == 0 && it >= 2) {
          tc::mbar_wait(&o_empty[it & 1], ((it - 2) >> 1) & 1);  // O buffer drained
        }
        MTR(4)
        tc::mbar_wait(p_full, ph_p);  // every warp wrote P(g)
        ph_p ^= 1;
        tc::fence_after();
        MTR(5)
        issue_pv(it, hh, kb_cur, no_cur);
        MTR(6)
#ifdef VQNQS_ATTN_TRACE2
        tc::mbar_wait(pv_done, ph_pv);
        ph_pv ^= 1;
        MTR(0)
#endif
        if (hh == hpg - 1) {  // item it's operands read
          if (leader) tc::mma_commit(&stage_free[it & 1]);
          __syncwarp();
        }
        if (it2 >= nit) break;
        it = it2;
        hh = hh2;
        j = j2;
        gi = gi2;
        kb_cur = kb_next;
        no_cur = no_next;
      }
#if defined(VQNQS_ATTN_TRACE) && !defined(VQNQS_ATTN_TL)
      if (blockIdx.x < 1 && lane == 0)
        printf("ATR-MMA b%d items %d: loop %u w_sfree %u w_stfull %u issueS %u w_oempty %u w_pfull %u issuePV %u S-latency %u\n",
               blockIdx.x, nit, mtr[0], mtr[1], mtr[2], mtr[3], mtr[4], mtr[5], mtr[6], mtr[7]);
#endif
    }
    if (warp > TCA_MMA_WARP && nit > 0) {
      // ================= producer warps: cp.async staging of every item into
      // its stage once the item two back has released it, tile tables one
      // tile ahead; three warps, 96 threads
      const int ptid = tid - 32 * (TCA_MMA_WARP + 1);
      auto pbar = [&]() { asm volatile("bar.sync 6, 96;" ::: "memory"); };
      auto fetch_info = [&](int j) {
        if (j < my_tiles)
          for (int c = ptid; c < TINFO_BYTES / 16; c += 96) {
            const uint8_t* src = tinfo + (int64_t)(blockIdx.x + j * gridDim.x) * TINFO_BYTES;
            tc::cp_async16(sb + L.info + (uint32_t)((j & 7) * TINFO_BYTES) + c * 16, src + c * 16);
          }
      };
      auto info_arrive = [&](int t) {
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tc::smem_u32(&info_ready[t & 7]));
      };
      fetch_info(0);
      fetch_info(1);
      tc::cp_async_commit();
      tc::cp_async_wait<0>();
      pbar();
      info_arrive(0);
      info_arrive(1);
      int j = 0, gi = 0;
      for (int it = 0; it < nit; ++it) {
        if (it >= 2) tc::mbar_wait(&stage_free[it & 1], ((it - 2) >> 1) & 1);
        if (gi == 0 && j >= 1) fetch_info(j + 1);
        const uint32_t st = sb + (uint32_t)(it & 1) * L.stage;
        const int32_t* rq = reinterpret_cast<const int32_t*>(slot(j));
        const int32_t* rb = rq + 128;
        for (int e = ptid; e < 128 * 8; e += 96) {
          const int r = e >> 3, c = e & 7;
          const int64_t off = (int64_t)rq[r] * ld;
          const bool ok = off >= 0;
          const bf16* src = qkv + (ok ? off : 0) + gi * 64 + c * 8;
          const uint32_t o = tc::sw128_chunk(r, c);
          tc::cp_async16_zfill(st + L.q + o, src, ok);
          tc::cp_async16_zfill(st + L.kown + o, src + d, ok);
          tc::cp_async16_zfill(st + L.vown + o, src + 2 * d, ok);
        }
        for (int e = ptid; e < 64 * KBb * 8; e += 96) {
          const int t = e >> 3, c = e & 7;
          const int64_t off = t < 128 ? (int64_t)rb[t] * ld : -1;
          const bool ok = off >= 0;
          const bf16* src = qkv + (ok ? off : 0) + d + gi * 64 + c * 8;
          const uint32_t o = tc::sw128_chunk(t, c);
          tc::cp_async16_zfill(st + L.kbase + o, src, ok);
          tc::cp_async16_zfill(st + L.vbase + o, src + d, ok);
        }
        tc::cp_async_commit();
        tc::cp_async_wait<0>();
        tc::fence_proxy_async();
        pbar();  // every producer thread's copies (and the next table) landed
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tc::smem_u32(&st_full[it & 1]));
        if (gi == 0 && j >= 1) info_arrive(j + 1);
        if (++gi == G) {
          gi = 0;
          ++j;
        }
      }
    }
  } else {
    // ================= softmax / epilogue warps
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(TCA_SOFTMAX_REGS) : "memory");
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const float sl2 = scale * 1.4426950408889634f;
    const uint32_t qbar = 1 + (warp & 3);  // named barrier of the row quadrant (128 threads)
    auto qsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(qbar), "n"(32 * TCA_PARTS) : "memory"); };
    auto arrive = [&](uint64_t* b) {  // one arrival per warp
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(b));
    };
    uint32_t ph_s = 0, ph_o = 0, hc = 0;
    ATR_DECL
    // per-tile thread state
    bool live = false;
    int kb_base = 0;
    // per-tile chunk slots (slot i = chunk part + 4i of the warp's live chunks:
    // base chunks, then own chunks), packed once per tile:
    //   sc_[i] = S column | P column << 9; mk_[i >> 1] bits 16 (i & 1) + j:
    //   entry j of the chunk is a key of the lane's row; sflags bit i: slot
    //   live, bit 4 + i: every live row uses the whole chunk
    uint32_t sc_[TCA_SLOTS], mk_[2] = {0, 0}, sflags = 0;
#pragma unroll
    for (int i = 0; i < TCA_SLOTS; ++i) sc_[i] = 0;
    int j = 0, gi = 0;  // item it = (j, gi)
    for (int it = 0; it < nit; ++it) {
      const int j1 = gi + 1 == G ? j + 1 : j, g1 = gi + 1 == G ? 0 : gi + 1;  // item it + 1
      if (gi == 0) {
        // the table landed before any warp signalled this item's operands
        ATR(13)
        tc::mbar_wait(&st_full[it & 1], (it >> 1) & 1);
        ATR(9)
        const uint8_t* ti = slot(j);
        live = row < reinterpret_cast<const int32_t*>(ti + 1544)[0];
        const int a = reinterpret_cast<const int16_t*>(ti + 1024)[row];
        const int own_lo = reinterpret_cast<const int16_t*>(ti + 1280)[row];
        const int own_cnt = live ? row - own_lo + 1 : 0;
        kb_base = kb_of(j);
        const int wb_end = (warp_max_i(a) + 15) & ~15;
        const int w_olo = warp_min_i(live ? own_lo : 1 << 20);
        const int w_ohi = warp_max_i(live ? row : -1);
        const int wo_beg = w_olo >= 128 ? 128 : (w_olo & ~15);
        const int wo_end = w_ohi < 0 ? 0 : ((w_ohi + 16) & ~15);
        const int nb = wb_end >> 4;
        const int nq = nb + max(0, (wo_end - wo_beg) >> 4);
        sflags = 0;
        mk_[0] = mk_[1] = 0;
#pragma unroll
        for (int i = 0; i < TCA_SLOTS; ++i) {
          const int q = part + TCA_PARTS * i;
          const bool isb = q < nb;
          const int c0 = isb ? 16 * q : wo_beg + 16 * (q - nb);
          const int off = isb ? c0 : c0 - own_lo;
          const int cnt = isb ? a : own_cnt;
          sc_[i] = (uint32_t)((isb ? TS_BASE : TS_OWN) + c0) |
                   ((uint32_t)((isb ? c0 : kb_base + c0) >> 1) << 9);
          const int lo = max(0, -off), hi = min(16, cnt - off);
          const uint32_t m16 = (live && hi > lo) ? ((1u << hi) - 1u) & ~((1u << lo) - 1u) : 0u;
          mk_[i >> 1] |= m16 << (16 * (i & 1));
          const bool full = __all_sync(0xffffffffu, !live || (off >= 0 && off + 16 <= cnt));
          sflags |= (q < nq ? 1u : 0u) << i;
          sflags |= (full ? 1u : 0u) << (4 + i);
        }
      }
      ATR(12)
      for (int hh = 0; hh < hpg; ++hh) {
#ifdef VQNQS_ATTN_TL
        tl_h = (int)hc - VQNQS_TL_H0;
        ATR(9)
#endif
        tc::mbar_wait(s_full, ph_s);
        ph_s ^= 1;
        tc::fence_after();
#if defined(VQNQS_ATTN_TL)
        ATR(0)
#elif defined(VQNQS_ATTN_TRACE)
        if (hh == 0) ATR(8) else ATR(0)
#endif
        // ---- the warp's live 16-column chunks (base chunks, then own chunks)
        // are dealt round-robin to the four warpgroups: slot i is chunk
        // part + 4i, live slots are a prefix. Each chunk is processed on its
        // own as soon as it is in registers -- mask, chunk max m_i,
        // e = exp2((s - m_i) scale log2e), chunk sum -- while the next chunk's
        // TMEM load is in flight, so the four warps of a sub-partition drift
        // into different phases and the ALU-bound masking of one overlaps the
        // MUFU-bound exponentials of another (with one max pass over all
        // chunks first, the four ran both phases in lockstep). The per-chunk
        // references are folded into the row's normaliser below, like the
        // per-warp ones.
        float v[TCA_SLOTS][16];
        float cm[TCA_SLOTS], cs[TCA_SLOTS];
        const int nl = __popc(sflags & 15u);
#ifdef VQNQS_ATTN_TL
        if ((unsigned)tl_h < 3u) tlog[warp][tl_h * 16 + 11] = 1000u + nl * 100 + (sflags >> 4);
#endif
#if VQNQS_ATTN_SWP
        // Software pipeline inside the warp: chunk i + 1 is masked and reduced
        // to its max (ALU pipe) in the same straight-line block as chunk i's
        // exponentials (MUFU) and chunk i + 2's TMEM load, one block per live
        // chunk count, so the two pipes overlap within a warp instead of the
        // quadrant's four warps saturating first one and then the other.
#pragma unroll
        for (int i = 0; i < TCA_SLOTS; ++i) {
          cm[i] = -INFINITY;
          cs[i] = 0.f;
        }
        auto maskmax = [&](auto ic) {
          constexpr int i = decltype(ic)::value;
          const uint32_t m16 = mk_[i >> 1] >> (16 * (i & 1));
          float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
          for (int q = 0; q < 16; q += 2) {
#ifndef VQNQS_ABL_NOMASK
            v[i][q] = (m16 >> q) & 1u ? v[i][q] : -INFINITY;
            v[i][q + 1] = (m16 >> (q + 1)) & 1u ? v[i][q + 1] : -INFINITY;
#endif
            m0 = fmaxf(m0, v[i][q]);
            m1 = fmaxf(m1, v[i][q + 1]);
          }
          cm[i] = fmaxf(m0, m1);
        };
        auto exps = [&](auto ic) {
          constexpr int i = decltype(ic)::value;
          const float mref = cm[i] == -INFINITY ? 0.f : cm[i] * sl2;
          float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < 16; q += 2) {
            const float2 t = tc::ffma2(make_float2(v[i][q], v[i][q + 1]), make_float2(sl2, sl2),
                                       make_float2(-mref, -mref));
            if (q / 2 < VQNQS_ATTN_EMU_PAIRS) {
              const float2 e = ex2_poly2(t);
              v[i][q] = e.x;
              v[i][q + 1] = e.y;
            } else {
#ifdef VQNQS_ABL_NOEXP
              v[i][q] = t.x;
              v[i][q + 1] = t.y;
#else
              v[i][q] = ex2_approx(t.x);
              v[i][q + 1] = ex2_approx(t.y);
#endif
            }
            s2 = tc::fadd2(s2, make_float2(v[i][q], v[i][q + 1]));
          }
          cs[i] = s2.x + s2.y;
        };
        auto s_loaded = [&]() {
          // every load of the head landed: the MMA warp may overwrite S with
          // the next head's scores
          tc::fence_before();
          arrive(s_free);
#ifdef VQNQS_ATTN_TL
          ATR(10)
#endif
        };
        auto run = [&](auto nlc) {
          constexpr int NL = decltype(nlc)::value;
          tc::tmem_ld16(trow + (sc_[0] & 511u), v[0]);
          if constexpr (NL > 1) tc::tmem_ld16(trow + (sc_[1] & 511u), v[1]);
          tc::tmem_wait_ld();
          if constexpr (NL <= 2) s_loaded();
          maskmax(std::integral_constant<int, 0>{});
          tc::static_for<NL>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            if constexpr (i + 2 < NL) tc::tmem_ld16(trow + (sc_[i + 2] & 511u), v[i + 2]);
            if constexpr (i + 1 < NL) maskmax(std::integral_constant<int, i + 1>{});
            exps(ic);
            if constexpr (i + 2 < NL) {
              tc::tmem_wait_ld();
              if constexpr (i + 2 == NL - 1) s_loaded();
            }
          });
        };
        switch (nl) {
          case 0: s_loaded(); break;
          case 1: run(std::integral_constant<int, 1>{}); break;
          case 2: run(std::integral_constant<int, 2>{}); break;
          case 3: run(std::integral_constant<int, 3>{}); break;
          default:
            if constexpr (TCA_SLOTS >= 4) run(std::integral_constant<int, TCA_SLOTS>{});
            break;
        }
#else
        if (nl > 0) tc::tmem_ld16(trow + (sc_[0] & 511u), v[0]);
        tc::tmem_wait_ld();
        if (nl == 0) {
          tc::fence_before();
          arrive(s_free);
        }
#pragma unroll
        for (int i = 0; i < TCA_SLOTS; ++i) {
          cm[i] = -INFINITY;
          cs[i] = 0.f;
          if (i < nl) {
            if (i + 1 < nl) {
              constexpr int L = TCA_SLOTS - 1;
              if (i < L) tc::tmem_ld16(trow + (sc_[i < L ? i + 1 : L] & 511u), v[i < L ? i + 1 : L]);
            } else {
              // every load of the head landed: the MMA warp may overwrite S
              // with the next head's scores
              tc::fence_before();
              arrive(s_free);
#ifdef VQNQS_ATTN_TL
              ATR(10)
#endif
            }
            float m0 = -INFINITY, m1 = -INFINITY;
            if ((sflags >> (4 + i)) & 1u) {
#pragma unroll
              for (int q = 0; q < 16; q += 2) {
                m0 = fmaxf(m0, v[i][q]);
                m1 = fmaxf(m1, v[i][q + 1]);
              }
            } else {
              const uint32_t m16 = mk_[i >> 1] >> (16 * (i & 1));
#pragma unroll
              for (int q = 0; q < 16; q += 2) {
                v[i][q] = (m16 >> q) & 1u ? v[i][q] : -INFINITY;
                v[i][q + 1] = (m16 >> (q + 1)) & 1u ? v[i][q + 1] : -INFINITY;
                m0 = fmaxf(m0, v[i][q]);
                m1 = fmaxf(m1, v[i][q + 1]);
              }
            }
            const float mi = fmaxf(m0, m1);
            const float mref = mi == -INFINITY ? 0.f : mi * sl2;
            float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int q = 0; q < 16; q += 2) {
              const float2 t = tc::ffma2(make_float2(v[i][q], v[i][q + 1]), make_float2(sl2, sl2),
                                         make_float2(-mref, -mref));
              if (q / 2 < VQNQS_ATTN_EMU_PAIRS) {
                const float2 e = ex2_poly2(t);
                v[i][q] = e.x;
                v[i][q + 1] = e.y;
              } else {
                v[i][q] = ex2_approx(t.x);
                v[i][q + 1] = ex2_approx(t.y);
              }
              s2 = tc::fadd2(s2, make_float2(v[i][q], v[i][q + 1]));
            }
            cm[i] = mi;
            cs[i] = s2.x + s2.y;
            if (i + 1 < nl) tc::tmem_wait_ld();
          }
        }
#endif
        ATR(1)
        // the thread's (max, sum) over its chunks; cm[i] becomes chunk i's
        // weight exp2((m_i - mp) scale log2e) (0 for a chunk without live keys)
        float mp = cm[0];
#pragma unroll
        for (int i = 1; i < TCA_SLOTS; ++i) mp = fmaxf(mp, cm[i]);
        float sp = 0.f;
#pragma unroll
        for (int i = 0; i < TCA_SLOTS; ++i) {
          cm[i] = cs[i] > 0.f ? ex2_approx((cm[i] - mp) * sl2) : 0.f;
          sp = fmaf(cs[i], cm[i], sp);
        }
        const int xb = hc & 1;
        ++hc;
        red[xb][part][row] = make_float2(mp, sp);
        ATR(2)
        const bool pv_early = hh == 0 && gi == 0 && it > 0;
        if (pv_early) {
          // the previous item's last value MMA read P
          tc::mbar_wait(pv_done, ph_o);
          ph_o ^= 1;
          tc::fence_after();
        }
        if (hh == 0 && gi == 0) {
          // P columns no warp writes this tile must read as zero (before the
          // quadrant barrier: another warpgroup may write these columns)
          const int pcols = (kb_base + 128) / 2;
          const uint32_t zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          for (int c = part * 8; c < pcols; c += 8 * TCA_PARTS) tc::tmem_st8u(trow + TS_P + c, zero);
          tc::tmem_wait_st();
        }
        qsync();
        ATR(3)
        float2 rq[TCA_PARTS];
#pragma unroll
        for (int q = 0; q < TCA_PARTS; ++q) rq[q] = red[xb][q][row];
#ifdef VQNQS_ATTN_TL
        if (rq[0].x == 12345.f) ATR(13)  // keeps the loads before the stamp
        ATR(12)
#endif
        float m = rq[0].x;
#pragma unroll
        for (int q = 1; q < TCA_PARTS; ++q) m = fmaxf(m, rq[q].x);
        float tot = 0.f;
#pragma unroll
        for (int q = 0; q < TCA_PARTS; ++q)
          tot += rq[q].y > 0.f ? rq[q].y * ex2_approx((rq[q].x - m) * sl2) : 0.f;
#ifdef VQNQS_ATTN_TL
        if (tot == 12345.f) ATR(14)
        ATR(13)
#endif
        const float f = sp > 0.f ? __fdividef(ex2_approx((mp - m) * sl2), tot) : 0.f;
        ATR(4)
        // P is rewritten only after the previous head's value MMA consumed it
        if ((hh > 0 || it > 0) && !pv_early) {
          tc::mbar_wait(pv_done, ph_o);
          ph_o ^= 1;
          tc::fence_after();
        }
        ATR(5)
        // ---- normalised bf16 probabilities into the TMEM P tile
#pragma unroll
        for (int i = 0; i < TCA_SLOTS; ++i) {
          if (i >= nl) continue;
          const float fi = f * cm[i];
          uint32_t pk[8];
#pragma unroll
          for (int q = 0; q < 16; q += 2) {
            const float2 p2 = tc::fmul2(make_float2(v[i][q], v[i][q + 1]), make_float2(fi, fi));
            pk[q / 2] = tc::pack_bf16(p2.x, p2.y);
          }
          tc::tmem_st8u(trow + TS_P + (sc_[i] >> 9), pk);
        }
        ATR(8)
        tc::tmem_wait_st();
        ATR(6)
        tc::fence_before();
        arrive(p_full);  // O_h = P_base V_base + P_own V_own, issued by the MMA warp
        ATR(7)
      }
      ATR(11)
      j = j1;
      gi = g1;
    }
#if defined(VQNQS_ATTN_TRACE) && !defined(VQNQS_ATTN_TL)
    if (blockIdx.x < 1 && lane == 0 && (warp == 0 || warp == 5 || warp == 10 || warp >= 12))
      printf("ATR b%d w%2d items %d: wS %llu ld %llu sm %llu bar %llu comb %llu wPV %llu P %llu arr %llu | end %llu setup %llu | wS(h0) %llu wST %llu\n",
             blockIdx.x, warp, nit, atr[0], atr[1], atr[2], atr[3], atr[4], atr[5], atr[6], atr[7],
             atr[11], atr[12], atr[8], atr[9]);
#endif
    }
  tc::fence_before();
  __syncthreads();
#ifdef VQNQS_ATTN_TL
  if (blockIdx.x < 8 && tid == 0 && nit * hpg > VQNQS_TL_H0 + 3) {
    unsigned t0 = 0xffffffffu;
    for (int w = 0; w < 32; ++w)
      for (int e = 0; e < 48; ++e)
        if ((e & 15) != 11 && tlog[w][e] && tlog[w][e] < t0) t0 = tlog[w][e];
    for (int w = 0; w < 32; ++w)
      for (int h = 0; h < 3; ++h) {
        unsigned e[16];
        for (int k = 0; k < 16; ++k) e[k] = tlog[w][h * 16 + k] ? tlog[w][h * 16 + k] - (k == 11 ? 0 : t0) : 0u;
        printf("TL %d %d %d %u %u %u %u %u %u %u %u %u %u %u %u %u %u %u %u\n", (int)blockIdx.x, w, h,
               e[0], e[1], e[2], e[3], e[4], e[5], e[6], e[7], e[8], e[9], e[10], e[11], e[12],
               e[13], e[14], e[15]);
      }
  }
#endif
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// launch with the drain-warp count of the head width
template <class... Args>
inline void launch_tc_attention(int dh, int grid, size_t smem, cudaStream_t st, Args... args) {
  if (tca_drain_warps(dh) == 4) {
    smem_optin(reinterpret_cast<const void*>(k_tc_attention<4>), smem);
    k_tc_attention<4><<<grid, tca_threads(4), smem, st>>>(args...);
  } else {
    smem_optin(reinterpret_cast<const void*>(k_tc_attention<8>), smem);
    k_tc_attention<8><<<grid, tca_threads(8), smem, st>>>(args...);
  }
}

inline bool tc_attn_ok(int prec, int d, int dh, int T) {
  return prec == 1 && d % 64 == 0 && (dh == 16 || dh == 32 || dh == 64) && T <= 128;
}

}  // namespace vqb

// Integer / byte-bound stages of the local-energy pipeline:
//   (a) connected configurations          k_connected, k_enumerate
//   (d) unique-row dedup + gather build   k_dedup, k_build_gather, k_embed
//   (e) head + segmented E_loc reduction  k_head, k_eloc
// plus per-sample scans and the LayerNorm row kernel.
//
// Row/location layout. A micro-batch holds S samples. Rows of
// sample s (its connected set, proj/src/hamiltonian.cpp:41-74) live at fixed
// capacity slots r = s*R1 + k, R1 = n_bonds + 1, k = 0 the diagonal row. Row
// k >= 1 flips bond row_bond[r]; t1 = its first changed token position. A
// location (k, p) is ACTIVE when its hidden state can differ from the base
// row's: p >= a_k = t1 + 1 (a_0 = 0). Inactive locations provably carry the
// base row's state at every layer (causal attention, identical inputs), so
// they are never stored: they map to the base location (0, p). Active
// locations of a sample are compact from act_off[s]: the base row's T
// locations first, then each row's suffix in row order.
#pragma once

#include <algorithm>

#include "common.cuh"

namespace vqb {

// Target token at position p of row r (little-endian groups of g spins,
// proj/src/model.cpp:236-248): base token with the flipped bond's bits toggled.
__device__ __forceinline__ int row_token(const int32_t* tok0, const int32_t* bonds, int bond,
                                         int g, int p) {
  int t = tok0[p];
  if (bond >= 0) {
    const int i = bonds[2 * bond], j = bonds[2 * bond + 1];
    if (i / g == p) t ^= 1 << (i % g);
    if (j / g == p) t ^= 1 << (j % g);
  }
  return t;
}

// ---------------------------------------------------------------- (a)
// connected_set (proj/src/hamiltonian.cpp:41-74), one warp per sample:
// diagonal 1/4 sum z_i z_j (exact in double: multiples of 1/4), and one row
// per antiparallel bond in bond order (ballot + popc keeps the order).
// dense != 0 is the no-reuse regime (proj/src/bench.cpp:19-36): every row is
// active from position 0 (t1 := -1), rows stay in bond order.
__global__ void k_connected(int S, int N, int g, int T, int nb, int dense, int cap,
                            const uint8_t* __restrict__ cfg,
                            const int32_t* __restrict__ bonds, int32_t* __restrict__ K,
                            double* __restrict__ diag, int32_t* __restrict__ row_bond,
                            int32_t* __restrict__ row_t1, int64_t* __restrict__ row_aoff,
                            int32_t* __restrict__ Mact, int32_t* __restrict__ tok0,
                            int64_t* __restrict__ attw, int32_t* __restrict__ row_perm) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= S) return;
  const int s = warp;
  const uint8_t* c = cfg + (int64_t)s * N;
  const int R1 = nb + 1;
  for (int p = lane; p < T; p += 32) {
    int t = 0;
    for (int j = 0; j < g; ++j)
      if (p * g + j < N) t |= int(c[p * g + j] & 1) << j;
    tok0[(int64_t)s * T + p] = t;
  }
  int zz = 0;
  int nrows = 1;
  int64_t aoff = T;  // base row's T locations come first
  // sum over active locations of (p + 1): the causal attention work
  int64_t aw = (int64_t)T * (T + 1) / 2;
  if (lane == 0) {
    row_bond[(int64_t)s * R1] = -1;
    row_t1[(int64_t)s * R1] = -1;
    row_aoff[(int64_t)s * R1] = 0;
  }
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int b = b0 + lane;
    bool anti = false;
    int cnt = 0, t1 = 0;
    if (b < nb) {
      const int i = bonds[2 * b], j = bonds[2 * b + 1];
      const int zi = 2 * int(c[i]) - 1, zj = 2 * int(c[j]) - 1;
      zz += zi * zj;
      anti = c[i] != c[j];
      t1 = dense ? -1 : min(i / g, j / g);
      cnt = T - (t1 + 1);
    }
    const unsigned m = __ballot_sync(0xffffffffu, anti);
    const int before = __popc(m & ((1u << lane) - 1u));
    // inclusive scan of active counts among anti lanes
    int v = anti ? cnt : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (anti) {
      const int64_t r = (int64_t)s * R1 + nrows + before;
      row_bond[r] = b;
      row_t1[r] = t1;
      row_aoff[r] = aoff + v - cnt;
    }
    nrows += __popc(m);
    aoff += __shfl_sync(0xffffffffu, v, 31);
    int64_t w = anti ? ((int64_t)T * (T + 1) / 2 - (int64_t)(t1 + 1) * (t1 + 2) / 2) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    aw += w;
  }
  zz = warp_sum_i(zz);
  if (lane == 0) {
    K[s] = nrows;
    diag[s] = 0.25 * (double)zz;
    Mact[s] = (int32_t)aoff;
    attw[s] = aw;
  }
  if (dense) {  // rows keep bond order: row_aoff from the scan above
    for (int k = lane; k < nrows; k += 32) row_perm[(int64_t)s * R1 + k] = k;
    return;
  }
  // Re-lay the rows' active regions in order of first changed token (stable
  // counting sort by t1): rows that share t1 share their base-key range and
  // suffix length, so attention tiles built in this order (row_perm) have
  // tight live score ranges. Values are unaffected: unique rows are
  // order-independent and U counts are order-invariant.
  // per-warp scratch of max(T, nb + 1) ints each (dynamic: a lattice may have
  // more connected rows than tokens; k_connected_smem sizes it)
  extern __shared__ int kc_smem[];
  const int W = max(T, R1);
  int* hist = kc_smem + ((threadIdx.x >> 5) & 3) * 2 * W;
  int* sloc = hist + W;
  for (int t = lane; t < T; t += 32) hist[t] = 0;
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  for (int k0 = 1; k0 < nrows; k0 += 32) {
    const int k = k0 + lane;
    const bool valid = k < nrows;
    const int t1 = valid ? row_t1[(int64_t)s * R1 + k] : T + lane;
    const unsigned mk = __match_any_sync(0xffffffffu, t1);
    const int rank_in = __popc(mk & lt);
    const int basec = valid ? hist[t1] : 0;
    __syncwarp();
    if (valid && rank_in == 0) hist[t1] += __popc(mk);
    __syncwarp();
    if (valid) row_aoff[(int64_t)s * R1 + k] = basec + rank_in;  // rank, finalised below
  }
  __syncwarp();
  // exclusive prefix over t1 buckets of (locations, rows)
  {
    const int per = (T + 31) / 32;
    const int b = lane * per, e = min(T, b + per);
    int locs = 0, rows = 0;
    for (int t = b; t < e; ++t) {
      locs += hist[t] * (T - t - 1);
      rows += hist[t];
    }
    int il = locs, ir = rows;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int nl = __shfl_up_sync(0xffffffffu, il, o);
      const int nr = __shfl_up_sync(0xffffffffu, ir, o);
      if (lane >= o) {
        il += nl;
        ir += nr;
      }
    }
    int rl = il - locs, rr = ir - rows;
    for (int t = b; t < e; ++t) {
      const int h = hist[t];
      sloc[t] = rl;
      hist[t] = rr;  // now: first layout row index (minus the base row) of bucket t
      rl += h * (T - t - 1);
      rr += h;
    }
  }
  __syncwarp();
  for (int k = 1 + lane; k < nrows; k += 32) {
    const int64_t r = (int64_t)s * R1 + k;
    const int t1 = row_t1[r];
    const int rank = (int)row_aoff[r];
    row_perm[(int64_t)s * R1 + 1 + hist[t1] + rank] = k;  // sorted by t1
  }
  __syncwarp();
  // Tiles of <= 128 active locations by a two-pointer sweep over the sorted
  // rows (the longest left first, then the next longest while they fit, then
  // the shortest while they fit): ~19% fewer attention tiles than a greedy
  // sweep of the sorted order at c4. Inside a tile the SHORT rows come first
  // and the long ones last: a short row has many base keys and few own keys,
  // a long row's causal own range grows with the tile row, so this order
  // evens the live score chunks of the tile's four row quadrants (the
  // attention softmax waits for the slowest quadrant; scripts/tile_sim.py:
  // the maximum over quadrants drops 11% at c4, 18% at c5). The tile that
  // holds the base row keeps it first: the base row stays at the sample's
  // layout offset 0. Bit 30 of a row_perm entry marks the first row of a tile
  // (k_build_tiles cuts there).
  if (lane == 0) {
    int* srt = sloc;  // rows sorted by t1, base row first
    int* ord = hist;  // layout order
    const int64_t pb = (int64_t)s * R1;
    srt[0] = 0;
    for (int i = 1; i < nrows; ++i) srt[i] = row_perm[pb + i];
    auto len = [&](int k) { return k == 0 ? T : T - (row_t1[pb + k] + 1); };
    auto rev = [&](int b, int e) {  // reverse ord[b, e)
      for (--e; b < e; ++b, --e) {
        const int t = ord[b];
        ord[b] = ord[e];
        ord[e] = t;
      }
    };
    // a tile's score columns: 16 ceil(max a / 16) base keys + 16 ceil(n / 16)
    // own keys, at most cap (the attention kernel's TMEM score buffer)
    auto fits = [&](int c, int amax, int k) {
      const int n = c + len(k), a = max(amax, T - len(k));
      return n <= 128 && ((a + 15) & ~15) + ((n + 15) & ~15) <= cap;
    };
    int i = 0, j = nrows - 1, o = 0;
    while (i <= j) {
      const int o0 = o;
      int c = len(srt[i]), amax = T - c;
      ord[o++] = srt[i++];
      while (i <= j && fits(c, amax, srt[i])) {
        c += len(srt[i]);
        amax = max(amax, T - len(srt[i]));
        ord[o++] = srt[i++];
      }
      const int om = o;
      while (j >= i && fits(c, amax, srt[j])) {
        c += len(srt[j]);
        amax = max(amax, T - len(srt[j]));
        ord[o++] = srt[j--];
      }
      if (o0 > 0) {  // [long..., short...] -> [short..., long...], each group's order kept
        rev(o0, om);
        rev(om, o);
        rev(o0, o);
      }
      ord[o0] |= 1 << 30;
    }
    int64_t off = 0;
    for (int q = 0; q < nrows; ++q) {
      const int k = ord[q] & ~(1 << 30);
      row_aoff[pb + k] = off;
      off += len(k);
      row_perm[pb + q] = ord[q];
    }
  }
}

// dynamic shared memory of a 128-thread k_connected block
inline size_t k_connected_smem(int T, int nb) {
  return size_t(4) * 2 * size_t(std::max(T, nb + 1)) * sizeof(int);
}

// Exclusive scan of per-sample counts (single CTA). mode 1 scans hash-table
// capacities (next power of two >= 2*count + 2) instead of the counts.
__global__ void k_scan(int n, const int32_t* __restrict__ in, int64_t* __restrict__ off,
                       int64_t* __restrict__ total, int mode) {
  __shared__ int64_t wsum[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int b = tid * per, e = min(n, b + per);
  auto val = [&](int i) -> int64_t {
    int64_t v = in[i];
    if (mode == 1) {
      int64_t c = 16;
      while (c < 2 * v + 2) c <<= 1;
      v = c;
    }
    return v;
  };
  int64_t loc = 0;
  for (int i = b; i < e; ++i) loc += val(i);
  // block exclusive scan of loc
  int64_t x = loc;
  const int lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t y = lane < (nt >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += z;
    }
    wsum[lane] = y;
  }
  __syncthreads();
  int64_t run = x - loc + (w > 0 ? wsum[w - 1] : 0);
  for (int i = b; i < e; ++i) {
    off[i] = run;
    run += val(i);
  }
  if (tid == nt - 1) *total = run;
}

// Location -> (row slot, position) for every active location.
__global__ void k_enumerate(int S, int R1, int T, const int32_t* __restrict__ K,
                            const int32_t* __restrict__ row_t1,
                            const int64_t* __restrict__ row_aoff,
                            const int64_t* __restrict__ act_off, int32_t* __restrict__ lrow,
                            int16_t* __restrict__ lpos) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = idx / T;
  const int p = int(idx % T);
  if (r >= (int64_t)S * R1) return;
  const int s = int(r / R1), k = int(r % R1);
  if (k >= K[s]) return;
  const int a = k == 0 ? 0 : row_t1[r] + 1;
  if (p < a) return;
  const int64_t loc = act_off[s] + row_aoff[r] + (p - a);
  lrow[loc] = int32_t(r);
  lpos[loc] = int16_t(p);
}

// ---------------------------------------------------------------- (d)
// Exact-key unique rows of one sample's active locations, numbered in first
// occurrence order exactly like the reference's unordered_map emplace loops
// (compress_inputs, proj/src/dedup.cpp:52-76; requantize, :151-175).
//   MODE 0 (input layer): key = (p, BOS-shifted token)      dedup.cpp:61-63
//   MODE 1 (after VQ):    key = (residual row, VQ code)     dedup.cpp:156-159
//                         (H > 1: the code tuple packed or numbered, k_pack_codes)
//   MODE 2 (H > 1, wide tuples): key = the packed code tuple itself; the ids
//                         number the distinct tuples of the sample for MODE 1
// One CTA per sample; open-addressing table (atomicCAS claims a slot,
// atomicMin keeps the first location), then a block scan over locations in
// order assigns ids. The table lives in shared memory (k_dedup below); the
// global-memory variant (dedup_global, L2-resident, slots reset before exit
// so the table is clean for the next layer) takes the samples that do not
// fit it.
template <int MODE>
__device__ void dedup_global(
    const int32_t* __restrict__ Mact, const int64_t* __restrict__ act_off,
    const int64_t* __restrict__ tab_off, unsigned long long* __restrict__ tkey,
    int32_t* __restrict__ trep, int32_t* __restrict__ tuid, int32_t* __restrict__ slot,
    // MODE 0 inputs
    const int32_t* __restrict__ lrow, const int16_t* __restrict__ lpos,
    const int32_t* __restrict__ tok0, const int32_t* __restrict__ row_bond,
    const int32_t* __restrict__ bonds, int R1, int T, int g, int V,
    // MODE 1 inputs
    const int32_t* __restrict__ I_in, const int32_t* __restrict__ code,
    // no-reuse regime: every location is its own unique row
    int dense,
    // outputs
    int32_t* __restrict__ I_out, int32_t* __restrict__ rep_of, int32_t* __restrict__ Ucnt,
    // MODE 2 input
    const unsigned long long* __restrict__ tup, int* sh_wtot, int* sh_run) {
  int* wtot = sh_wtot;
  int& run_s = *sh_run;
  const int s = blockIdx.x;
  const int M = Mact[s];
  const int64_t base = act_off[s];
  const int64_t tb = tab_off[s];
  int64_t cap = 16;
  while (cap < 2 * (int64_t)M + 2) cap <<= 1;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
  // phase 1: insert
  for (int i = tid; i < M; i += nt) {
    const int64_t loc = base + i;
    unsigned long long key;
    if (dense) {
      key = (unsigned long long)i;
    } else if (MODE == 0) {
      const int r = lrow[loc];
      const int p = lpos[loc];
      const int sidx = r / R1;
      const int tok = p == 0 ? V : row_token(tok0 + (int64_t)sidx * T, bonds, row_bond[r], g, p - 1);
      key = (unsigned long long)p * (unsigned long long)(V + 1) + (unsigned long long)tok;
    } else if (MODE == 1) {
      key = ((unsigned long long)(uint32_t)I_in[loc] << 32) | (uint32_t)code[loc];
    } else {
      key = tup[loc];
    }
    int64_t h = (int64_t)(hash64(key) & (uint64_t)(cap - 1));
    for (;;) {
      const unsigned long long prev = atomicCAS(&tkey[tb + h], VQB_EMPTY_KEY, key);
      if (prev == VQB_EMPTY_KEY || prev == key) {
        atomicMin(&trep[tb + h], i);
        slot[loc] = (int32_t)h;
        break;
      }
      h = (h + 1) & (cap - 1);
    }
  }
  __syncthreads();
  // phase 2: ids in first-occurrence order. Warp w owns the contiguous
  // location segment [w L, (w + 1) L): it counts its first occurrences, one
  // block scan of the warp counts gives each warp its first id, and the warp
  // numbers its segment in order with ballots (two block barriers in all).
  const int nw = nt >> 5;
  const int L = (M + nw - 1) / nw;
  const int seg0 = min(M, w * L), seg1 = min(M, seg0 + L);
  int mine = 0;
  for (int i0 = seg0; i0 < seg1; i0 += 32) {
    const int i = i0 + lane;
    const bool flag = i < seg1 && trep[tb + slot[base + i]] == i;
    mine += __popc(__ballot_sync(0xffffffffu, flag));
  }
  if (lane == 0) wtot[w] = mine;
  __syncthreads();
  if (w == 0) {
    int v = lane < nw ? wtot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < nw) wtot[lane] = v;  // inclusive
    if (lane == 31) run_s = v;      // total
  }
  __syncthreads();
  int next = w > 0 ? wtot[w - 1] : 0;
  for (int i0 = seg0; i0 < seg1; i0 += 32) {
    const int i = i0 + lane;
    int64_t h = 0;
    bool flag = false;
    if (i < seg1) {
      h = slot[base + i];
      flag = trep[tb + h] == i;
    }
    const unsigned m = __ballot_sync(0xffffffffu, flag);
    if (flag) {
      const int id = next + __popc(m & ((1u << lane) - 1u));
      tuid[tb + h] = id;
      rep_of[base + id] = i;
    }
    next += __popc(m);
  }
  __syncthreads();
  // phase 3: scatter ids to locations
  for (int i = tid; i < M; i += nt) I_out[base + i] = tuid[tb + slot[base + i]];
  if (tid == 0) Ucnt[s] = run_s;
  __syncthreads();
  // phase 4: reset touched slots
  for (int i = tid; i < M; i += nt) {
    const int64_t h = slot[base + i];
    tkey[tb + h] = VQB_EMPTY_KEY;
    trep[tb + h] = VQB_INT_MAX;
  }
}

// Key of location i of sample s (MODE 0: (p, BOS-shifted token); MODE 1:
// (residual row, code); MODE 2: the packed code tuple).
template <int MODE>
__device__ __forceinline__ unsigned long long dedup_key(
    int64_t loc, const int32_t* __restrict__ lrow, const int16_t* __restrict__ lpos,
    const int32_t* __restrict__ tok0, const int32_t* __restrict__ row_bond,
    const int32_t* __restrict__ bonds, int R1, int T, int g, int V,
    const int32_t* __restrict__ I_in, const int32_t* __restrict__ code,
    const unsigned long long* __restrict__ tup) {
  if (MODE == 0) {
    const int r = lrow[loc];
    const int p = lpos[loc];
    const int sidx = r / R1;
    const int tok = p == 0 ? V : row_token(tok0 + (int64_t)sidx * T, bonds, row_bond[r], g, p - 1);
    return (unsigned long long)p * (unsigned long long)(V + 1) + (unsigned long long)tok;
  } else if (MODE == 1) {
    return ((unsigned long long)(uint32_t)I_in[loc] << 32) | (uint32_t)code[loc];
  } else {
    return tup[loc];
  }
}

// Shared-memory table: DEDUP_SC slots (key; first location, later -(id + 1))
// and a 16-bit slot per location, so a sample's dedup touches HBM only for
// its keys in and its ids out (~12 B per location instead of ~8 dependent
// L2 round trips per location through a global table); 176 KB, one CTA of
// 1024 threads per SM. A sample whose unique keys exceed half the slots, or whose locations
// exceed DEDUP_SMAX, takes the global table path (dedup_global) instead;
// MODE 0 keys index the table directly when the key space (T (V + 1)) fits.
constexpr int DEDUP_SC = 8192;
constexpr int DEDUP_SMAX = 40960;
constexpr int DEDUP_THREADS = 1024;
inline size_t dedup_smem_bytes() { return size_t(DEDUP_SC) * 12 + size_t(DEDUP_SMAX) * 2; }

template <int MODE>
__global__ void __launch_bounds__(DEDUP_THREADS, 1) k_dedup(
    const int32_t* __restrict__ Mact, const int64_t* __restrict__ act_off,
    const int64_t* __restrict__ tab_off, unsigned long long* __restrict__ tkey,
    int32_t* __restrict__ trep, int32_t* __restrict__ tuid, int32_t* __restrict__ slot,
    const int32_t* __restrict__ lrow, const int16_t* __restrict__ lpos,
    const int32_t* __restrict__ tok0, const int32_t* __restrict__ row_bond,
    const int32_t* __restrict__ bonds, int R1, int T, int g, int V,
    const int32_t* __restrict__ I_in, const int32_t* __restrict__ code, int dense,
    int32_t* __restrict__ I_out, int32_t* __restrict__ rep_of, int32_t* __restrict__ Ucnt,
    const unsigned long long* __restrict__ tup) {
  extern __shared__ __align__(16) uint8_t dd_smem[];
  __shared__ int wtot[32];
  __shared__ int run_s, n_new;
  unsigned long long* skey = reinterpret_cast<unsigned long long*>(dd_smem);
  int32_t* srep = reinterpret_cast<int32_t*>(skey + DEDUP_SC);
  uint16_t* sslot = reinterpret_cast<uint16_t*>(srep + DEDUP_SC);
  const int s = blockIdx.x;
  const int M = Mact[s];
  const int64_t base = act_off[s];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
  if (dense) {  // no-reuse regime: every location is its own unique row
    for (int i = tid; i < M; i += nt) {
      I_out[base + i] = i;
      rep_of[base + i] = i;
    }
    if (tid == 0) Ucnt[s] = M;
    return;
  }
  const bool direct = MODE == 0 && T * (V + 1) <= DEDUP_SC;
  if (M > DEDUP_SMAX) {
    dedup_global<MODE>(Mact, act_off, tab_off, tkey, trep, tuid, slot, lrow, lpos, tok0,
                       row_bond, bonds, R1, T, g, V, I_in, code, 0, I_out, rep_of, Ucnt, tup,
                       wtot, &run_s);
    return;
  }
  for (int h = tid; h < DEDUP_SC; h += nt) {
    skey[h] = VQB_EMPTY_KEY;
    srep[h] = VQB_INT_MAX;
  }
  if (tid == 0) n_new = 0;
  __syncthreads();
  // phase 1: insert (probing stops once the table is half full). Keys are
  // loaded four locations ahead of their inserts so the global loads overlap.
  constexpr int PF = 4;
  for (int i0 = tid; i0 < M; i0 += PF * nt) {
    unsigned long long keys[PF];
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int i = i0 + k * nt;
      keys[k] = i < M ? dedup_key<MODE>(base + i, lrow, lpos, tok0, row_bond, bonds, R1, T, g, V,
                                        I_in, code, tup)
                      : 0ull;
    }
#pragma unroll
    for (int k = 0; k < PF; ++k) {
    const int i = i0 + k * nt;
    if (i >= M) break;
    const unsigned long long key = keys[k];
    int h;
    if (direct) {
      h = (int)key;
    } else {
      // 32-bit multiplicative hash of the two key halves (cheap; the
      // table is small and probing is linear)
      uint32_t hh = (uint32_t)key * 0x9E3779B1u ^ (uint32_t)(key >> 32) * 0x85EBCA6Bu;
      h = (int)((hh ^ (hh >> 15)) & (DEDUP_SC - 1));
      for (;;) {
        const unsigned long long cur = skey[h];  // settled slots need no atomic
        if (cur == key) break;
        if (cur != VQB_EMPTY_KEY) {
          h = (h + 1) & (DEDUP_SC - 1);
          continue;
        }
        const unsigned long long prev = atomicCAS(&skey[h], VQB_EMPTY_KEY, key);
        if (prev == key) break;
        if (prev == VQB_EMPTY_KEY) {
          atomicAdd(&n_new, 1);
          break;
        }
        h = (h + 1) & (DEDUP_SC - 1);
      }
    }
    if (srep[h] > i) atomicMin(&srep[h], i);  // later locations of a seen key skip it
    sslot[i] = (uint16_t)h;
    }
    if (*reinterpret_cast<volatile int*>(&n_new) > DEDUP_SC / 2) break;
  }
  __syncthreads();
  if (n_new > DEDUP_SC / 2) {  // too many distinct keys for the table
    dedup_global<MODE>(Mact, act_off, tab_off, tkey, trep, tuid, slot, lrow, lpos, tok0,
                       row_bond, bonds, R1, T, g, V, I_in, code, 0, I_out, rep_of, Ucnt, tup,
                       wtot, &run_s);
    return;
  }
  // phase 2: ids in first-occurrence order (warp w numbers the contiguous
  // location segment [w L, (w + 1) L) after one block scan of warp counts)
  const int nw = nt >> 5;
  const int L = (M + nw - 1) / nw;
  const int seg0 = min(M, w * L), seg1 = min(M, seg0 + L);
  int mine = 0;
  for (int i0 = seg0; i0 < seg1; i0 += 32) {
    const int i = i0 + lane;
    const bool flag = i < seg1 && srep[sslot[i]] == i;
    mine += __popc(__ballot_sync(0xffffffffu, flag));
  }
  if (lane == 0) wtot[w] = mine;
  __syncthreads();
  if (w == 0) {
    int v = lane < nw ? wtot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < nw) wtot[lane] = v;  // inclusive
    if (lane == 31) run_s = v;      // total
  }
  __syncthreads();
  int next = w > 0 ? wtot[w - 1] : 0;
  // a key's entry is written only by its first location, and no other
  // location's test (srep[h] == i >= 0) can match the negative id
  for (int i0 = seg0; i0 < seg1; i0 += 32) {
    const int i = i0 + lane;
    int h = 0;
    bool flag = false;
    if (i < seg1) {
      h = sslot[i];
      flag = srep[h] == i;
    }
    const unsigned m = __ballot_sync(0xffffffffu, flag);
    if (flag) {
      const int id = next + __popc(m & ((1u << lane) - 1u));
      srep[h] = -(id + 1);
      rep_of[base + id] = i;
    }
    next += __popc(m);
  }
  __syncthreads();
  // phase 3: ids to locations
  for (int i = tid; i < M; i += nt) I_out[base + i] = -srep[sslot[i]] - 1;
  if (tid == 0) Ucnt[s] = run_s;
}

// Input embeddings of the unique input rows: tok_embed[tok] + pos_embed[p]
// (proj/src/dedup.cpp:79-89).
__global__ void k_embed(int d, int R1, int T, int g, int V, const int32_t* __restrict__ Ucnt,
                        const int64_t* __restrict__ Uoff, const int64_t* __restrict__ act_off,
                        const int32_t* __restrict__ rep_of, const int32_t* __restrict__ lrow,
                        const int16_t* __restrict__ lpos, const int32_t* __restrict__ tok0,
                        const int32_t* __restrict__ row_bond, const int32_t* __restrict__ bonds,
                        const float* __restrict__ tok_embed, const float* __restrict__ pos_embed,
                        float* __restrict__ x) {
  // one warp per unique input row: its (position, token) once, then the row
  // written as float4 (d % 4 == 0)
  const int s = blockIdx.x;
  const int U = Ucnt[s];
  const int64_t base = act_off[s], uo = Uoff[s];
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int d4 = d >> 2;
  for (int uid = threadIdx.x >> 5; uid < U; uid += nw) {
    const int64_t loc = base + rep_of[base + uid];
    const int r = lrow[loc], p = lpos[loc];
    const int tok = p == 0 ? V : row_token(tok0 + (int64_t)s * T, bonds, row_bond[r], g, p - 1);
    if ((d & 3) == 0) {
      const float4* te = reinterpret_cast<const float4*>(tok_embed + (int64_t)tok * d);
      const float4* pe = reinterpret_cast<const float4*>(pos_embed + (int64_t)p * d);
      float4* xr = reinterpret_cast<float4*>(x + (uo + uid) * d);
      for (int c = lane; c < d4; c += 32) {
        const float4 a = te[c], b = pe[c];
        xr[c] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
      }
    } else {
      for (int c = lane; c < d; c += 32)
        x[(uo + uid) * d + c] = tok_embed[(int64_t)tok * d + c] + pos_embed[(int64_t)p * d + c];
    }
  }
}

constexpr int LN_REG = 8;  // row elements per lane kept in registers (d <= 256)

// kernels::layer_norm (proj/src/tensor.cpp:57-83): two-pass biased variance,
// eps 1e-5, statistics in double; one warp per row over *Mp rows.
template <typename TA>
__global__ void k_layernorm(const int64_t* __restrict__ Mp, int d, const float* __restrict__ x,
                            const float* __restrict__ gam, const float* __restrict__ bet,
                            TA* __restrict__ out) {
  const int64_t M = *Mp;
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  const int64_t r0 = blockIdx.x * wpb + (threadIdx.x >> 5), rstep = (int64_t)gridDim.x * wpb;
  if (d <= 32 * LN_REG) {
    // rows read once into registers (element lane + 32 k), the warp's next
    // row loaded before this row's reductions; same sums
    float nx[LN_REG];
#pragma unroll
    for (int k = 0; k < LN_REG; ++k) {
      const int c = lane + 32 * k;
      nx[k] = (r0 < M && c < d) ? x[r0 * d + c] : 0.f;
    }
    for (int64_t r = r0; r < M; r += rstep) {
      float xv[LN_REG];
#pragma unroll
      for (int k = 0; k < LN_REG; ++k) xv[k] = nx[k];
      const int64_t rn = r + rstep;
#pragma unroll
      for (int k = 0; k < LN_REG; ++k) {
        const int c = lane + 32 * k;
        nx[k] = (rn < M && c < d) ? x[rn * d + c] : 0.f;
      }
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < LN_REG; ++k)
        if (lane + 32 * k < d) s += xv[k];
      const double mean = warp_sum(s) / d;
      double v = 0.0;
#pragma unroll
      for (int k = 0; k < LN_REG; ++k)
        if (lane + 32 * k < d) {
          const double t = xv[k] - mean;
          v += t * t;
        }
      const double var = warp_sum(v) / d;
      const double rstd = 1.0 / sqrt(var + 1e-5);
#pragma unroll
      for (int k = 0; k < LN_REG; ++k) {
        const int c = lane + 32 * k;
        if (c < d) out[r * d + c] = from_f<TA>((float)((xv[k] - mean) * rstd * gam[c] + bet[c]));
      }
    }
    return;
  }
  for (int64_t r = r0; r < M; r += rstep) {
    const float* xr = x + r * d;
    double s = 0.0;
    for (int c = lane; c < d; c += 32) s += xr[c];
    const double mean = warp_sum(s) / d;
    double v = 0.0;
    for (int c = lane; c < d; c += 32) {
      const double t = xr[c] - mean;
      v += t * t;
    }
    const double var = warp_sum(v) / d;
    const double rstd = 1.0 / sqrt(var + 1e-5);
    for (int c = lane; c < d; c += 32)
      out[r * d + c] = from_f<TA>((float)((xr[c] - mean) * rstd * gam[c] + bet[c]));
  }
}

// d = 128 NV: the row as NV float4 per lane (element 4 lane + 128 k ..), read
// once with 512-byte warp loads, the warp's next row in flight; statistics in
// double as above ((double)x - mean is the deviation of both later passes), the
// affine output (t rstd) gamma + beta in fp32 from the double t rstd: two
// conversions per element instead of six, which bound the scalar kernel.
template <typename TA>
__device__ __forceinline__ void store4(TA* p, float a, float b, float c, float e);
template <>
__device__ __forceinline__ void store4<float>(float* p, float a, float b, float c, float e) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, e);
}
template <>
__device__ __forceinline__ void store4<bf16>(bf16* p, float a, float b, float c, float e) {
  const __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, e);
  uint2 w;
  w.x = *reinterpret_cast<const uint32_t*>(&lo);
  w.y = *reinterpret_cast<const uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = w;
}

// statistics and output of one row held as NV float4 per lane
template <typename TA, int NV>
__device__ __forceinline__ void ln_row_v(const float4* xv, int lane, const float* __restrict__ gam,
                                         const float* __restrict__ bet, TA* __restrict__ orow) {
  constexpr int d = 128 * NV;
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k)
    s += ((double)xv[k].x + (double)xv[k].y) + ((double)xv[k].z + (double)xv[k].w);
  const double mean = warp_sum(s) / d;
  double q = 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double t0 = xv[k].x - mean, t1 = xv[k].y - mean, t2 = xv[k].z - mean,
                 t3 = xv[k].w - mean;
    q += (t0 * t0 + t1 * t1) + (t2 * t2 + t3 * t3);
  }
  const double var = warp_sum(q) / d;
  const double rstd = 1.0 / sqrt(var + 1e-5);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int c = 4 * lane + 128 * k;
    const float4 g = *reinterpret_cast<const float4*>(gam + c);
    const float4 b = *reinterpret_cast<const float4*>(bet + c);
    store4<TA>(orow + c, fmaf((float)((xv[k].x - mean) * rstd), g.x, b.x),
               fmaf((float)((xv[k].y - mean) * rstd), g.y, b.y),
               fmaf((float)((xv[k].z - mean) * rstd), g.z, b.z),
               fmaf((float)((xv[k].w - mean) * rstd), g.w, b.w));
  }
}

template <typename TA, int NV>
__global__ void __launch_bounds__(256) k_layernorm_v(const int64_t* __restrict__ Mp,
                                                     const float* __restrict__ x,
                                                     const float* __restrict__ gam,
                                                     const float* __restrict__ bet,
                                                     TA* __restrict__ out) {
  constexpr int d = 128 * NV;
  const int64_t M = *Mp;
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  const int64_t r0 = blockIdx.x * wpb + (threadIdx.x >> 5), rstep = (int64_t)gridDim.x * wpb;
  float4 nx[NV];
  auto load = [&](int64_t r) {
    const float4* xr = reinterpret_cast<const float4*>(x + (r < M ? r : 0) * d);
#pragma unroll
    for (int k = 0; k < NV; ++k) nx[k] = xr[lane + 32 * k];
  };
  load(r0);
  for (int64_t r = r0; r < M; r += rstep) {
    float4 xv[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) xv[k] = nx[k];
    load(r + rstep);
    ln_row_v<TA, NV>(xv, lane, gam, bet, out + r * d);
  }
}

// k_cont_ln for one VQ head and d = 128 NV (see k_cont_ln below)
template <typename TA, int NV>
__global__ void __launch_bounds__(256) k_cont_ln_v(
    const int64_t* __restrict__ Mp, const float* __restrict__ x,
    const int64_t* __restrict__ g_res, const int32_t* __restrict__ g_code,
    const float* __restrict__ pwo, const float* __restrict__ gam, const float* __restrict__ bet,
    float* __restrict__ y, TA* __restrict__ out) {
  constexpr int d = 128 * NV;
  const int64_t M = *Mp;
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  const int64_t r0 = blockIdx.x * wpb + (threadIdx.x >> 5), rstep = (int64_t)gridDim.x * wpb;
  float4 nx[NV], np[NV];
  auto gather = [&](int64_t r) {
    const bool ok = r < M;
    const float4* xr = reinterpret_cast<const float4*>(x + (ok ? g_res[r] : 0) * d);
    const float4* pr = reinterpret_cast<const float4*>(pwo + (int64_t)(ok ? g_code[r] : 0) * d);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      nx[k] = xr[lane + 32 * k];
      np[k] = pr[lane + 32 * k];
    }
  };
  gather(r0);
  for (int64_t r = r0; r < M; r += rstep) {
    float4 yv[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k)
      yv[k] = make_float4(nx[k].x + np[k].x, nx[k].y + np[k].y, nx[k].z + np[k].z,
                          nx[k].w + np[k].w);
    gather(r + rstep);
    float4* yr = reinterpret_cast<float4*>(y + r * d);
#pragma unroll
    for (int k = 0; k < NV; ++k) yr[lane + 32 * k] = yv[k];
    ln_row_v<TA, NV>(yv, lane, gam, bet, out + r * d);
  }
}

// Continuation head (proj/src/dedup.cpp:255-262) on the U_{b+1} new unique
// rows: y = r + o with r the block-input residual row and o = code_row Wo + bo
// read from the per-code table pwo (computed once per model by the same GEMM,
// so each row's o is bit-identical to a per-row product), then LN2(y).
// One warp per row; y is kept for the W2 residual.
template <typename TA>
__global__ void k_cont_ln(const int64_t* __restrict__ Mp, int d, int H, int Q,
                          const float* __restrict__ x,
                          const int64_t* __restrict__ g_res, const int32_t* __restrict__ g_code,
                          const float* __restrict__ pwo, const float* __restrict__ gam,
                          const float* __restrict__ bet, float* __restrict__ y,
                          TA* __restrict__ out) {
  const int64_t M = *Mp;
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  const int64_t r0 = blockIdx.x * wpb + (threadIdx.x >> 5), rstep = (int64_t)gridDim.x * wpb;
  if (H == 1 && d <= 32 * LN_REG) {
    // y = x[g_res] + P[g_code] in registers between the passes, the warp's
    // next row gathered before this row's reductions; same sums
    float nxv[LN_REG], npv[LN_REG];
    auto gather = [&](int64_t r, float* xv, float* pv) {
      const bool ok = r < M;
      const float* xr = x + (ok ? g_res[r] : 0) * d;
      const float* pr = pwo + (int64_t)(ok ? g_code[r] : 0) * d;
#pragma unroll
      for (int k = 0; k < LN_REG; ++k) {
        const int c = lane + 32 * k;
        xv[k] = (ok && c < d) ? xr[c] : 0.f;
        pv[k] = (ok && c < d) ? pr[c] : 0.f;
      }
    };
    gather(r0, nxv, npv);
    for (int64_t r = r0; r < M; r += rstep) {
      float yv[LN_REG];
#pragma unroll
      for (int k = 0; k < LN_REG; ++k) yv[k] = nxv[k] + npv[k];
      gather(r + rstep, nxv, npv);
      float* yr = y + r * d;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < LN_REG; ++k) {
        const int c = lane + 32 * k;
        if (c < d) {
          yr[c] = yv[k];
          s += yv[k];
        }
      }
      const double mean = warp_sum(s) / d;
      double q = 0.0;
#pragma unroll
      for (int k = 0; k < LN_REG; ++k)
        if (lane + 32 * k < d) {
          const double t = yv[k] - mean;
          q += t * t;
        }
      const double var = warp_sum(q) / d;
      const double rstd = 1.0 / sqrt(var + 1e-5);
#pragma unroll
      for (int k = 0; k < LN_REG; ++k) {
        const int c = lane + 32 * k;
        if (c < d) out[r * d + c] = from_f<TA>((float)((yv[k] - mean) * rstd * gam[c] + bet[c]));
      }
    }
    return;
  }
  for (int64_t r = r0; r < M; r += rstep) {
    const float* xr = x + g_res[r] * d;
    const float* pr = pwo + (int64_t)g_code[r * H] * d;
    float* yr = y + r * d;
    if (H > 1) {
      // H VQ heads: o = sum_h table_h[code_h] (head 0's table carries bo)
      double s = 0.0;
      for (int c = lane; c < d; c += 32) {
        float o = pr[c];
        for (int hh = 1; hh < H; ++hh)
          o += pwo[((int64_t)hh * Q + g_code[r * H + hh]) * d + c];
        const float v = xr[c] + o;
        yr[c] = v;
        s += v;
      }
      const double mean = warp_sum(s) / d;
      double q = 0.0;
      for (int c = lane; c < d; c += 32) {
        const double t = yr[c] - mean;
        q += t * t;
      }
      const double var = warp_sum(q) / d;
      const double rstd = 1.0 / sqrt(var + 1e-5);
      for (int c = lane; c < d; c += 32)
        out[r * d + c] = from_f<TA>((float)((yr[c] - mean) * rstd * gam[c] + bet[c]));
      continue;
    }
    double s = 0.0;
    for (int c = lane; c < d; c += 32) {
      const float v = xr[c] + pr[c];
      yr[c] = v;
      s += v;
    }
    const double mean = warp_sum(s) / d;
    double q = 0.0;
    for (int c = lane; c < d; c += 32) {
      const double t = yr[c] - mean;
      q += t * t;
    }
    const double var = warp_sum(q) / d;
    const double rstd = 1.0 / sqrt(var + 1e-5);
    for (int c = lane; c < d; c += 32)
      out[r * d + c] = from_f<TA>((float)((yr[c] - mean) * rstd * gam[c] + bet[c]));
  }
}

// LayerNorm / continuation launchers: the vector kernels for d = 128 NV,
// NV in {1, 2, 3, 4, 6, 8}; the scalar ones otherwise.
template <typename TA>
inline void launch_layernorm(int grid, cudaStream_t st, const int64_t* Mp, int d, const float* x,
                             const float* gam, const float* bet, TA* out) {
  switch (d % 128 == 0 ? d / 128 : 0) {
    case 1: k_layernorm_v<TA, 1><<<grid, 256, 0, st>>>(Mp, x, gam, bet, out); break;
    case 2: k_layernorm_v<TA, 2><<<grid, 256, 0, st>>>(Mp, x, gam, bet, out); break;
    case 3: k_layernorm_v<TA, 3><<<grid, 256, 0, st>>>(Mp, x, gam, bet, out); break;
    case 4: k_layernorm_v<TA, 4><<<grid, 256, 0, st>>>(Mp, x, gam, bet, out); break;
    case 6: k_layernorm_v<TA, 6><<<grid, 256, 0, st>>>(Mp, x, gam, bet, out); break;
    case 8: k_layernorm_v<TA, 8><<<grid, 256, 0, st>>>(Mp, x, gam, bet, out); break;
    default: k_layernorm<TA><<<grid, 256, 0, st>>>(Mp, d, x, gam, bet, out);
  }
}
template <typename TA>
inline void launch_cont_ln(int grid, cudaStream_t st, const int64_t* Mp, int d, int H, int Q,
                           const float* x, const int64_t* g_res, const int32_t* g_code,
                           const float* pwo, const float* gam, const float* bet, float* y,
                           TA* out) {
  switch (H == 1 && d % 128 == 0 ? d / 128 : 0) {
    case 1: k_cont_ln_v<TA, 1><<<grid, 256, 0, st>>>(Mp, x, g_res, g_code, pwo, gam, bet, y, out); break;
    case 2: k_cont_ln_v<TA, 2><<<grid, 256, 0, st>>>(Mp, x, g_res, g_code, pwo, gam, bet, y, out); break;
    case 3: k_cont_ln_v<TA, 3><<<grid, 256, 0, st>>>(Mp, x, g_res, g_code, pwo, gam, bet, y, out); break;
    case 4: k_cont_ln_v<TA, 4><<<grid, 256, 0, st>>>(Mp, x, g_res, g_code, pwo, gam, bet, y, out); break;
    case 6: k_cont_ln_v<TA, 6><<<grid, 256, 0, st>>>(Mp, x, g_res, g_code, pwo, gam, bet, y, out); break;
    case 8: k_cont_ln_v<TA, 8><<<grid, 256, 0, st>>>(Mp, x, g_res, g_code, pwo, gam, bet, y, out); break;
    default:
      k_cont_ln<TA><<<grid, 256, 0, st>>>(Mp, d, H, Q, x, g_res, g_code, pwo, gam, bet, y, out);
  }
}

// For each new unique row (global id g): which codebook row and which
// residual row it concatenates (requantize's V' = [code row || residual row],
// proj/src/dedup.cpp:176-184), and its token position.
__global__ void k_build_gather(int H, const int32_t* __restrict__ Ucnt_next,
                               const int64_t* __restrict__ Uoff_next,
                               const int64_t* __restrict__ Uoff_cur,
                               const int64_t* __restrict__ act_off,
                               const int32_t* __restrict__ rep_of,
                               const int32_t* __restrict__ code, const int32_t* __restrict__ I_cur,
                               const int16_t* __restrict__ lpos, int32_t* __restrict__ g_code,
                               int64_t* __restrict__ g_res, int16_t* __restrict__ upos) {
  const int s = blockIdx.x;
  const int U = Ucnt_next[s];
  const int64_t base = act_off[s];
  for (int uid = threadIdx.x; uid < U; uid += blockDim.x) {
    const int64_t loc = base + rep_of[base + uid];
    const int64_t gi = Uoff_next[s] + uid;
    for (int h = 0; h < H; ++h) g_code[gi * H + h] = code[loc * H + h];
    g_res[gi] = Uoff_cur[s] + I_cur[loc];
    upos[gi] = lpos[loc];
  }
}

// Blocks without a VQ (the trailing half block; every block when VQ is
// off): densify_attention (proj/src/dedup.cpp:187-211) makes every location
// its own unique row, with the residual row it concatenates. Over the
// active locations that is the identity; the new rows' global ids equal the
// location index (Uoff_next = act_off). One CTA per sample.
__global__ void k_densify(const int32_t* __restrict__ Mact, const int64_t* __restrict__ act_off,
                          const int64_t* __restrict__ Uoff_cur, const int32_t* __restrict__ I_cur,
                          const int16_t* __restrict__ lpos, int32_t* __restrict__ I_next,
                          int64_t* __restrict__ g_res, int16_t* __restrict__ upos,
                          int32_t* __restrict__ Ucnt_next) {
  const int s = blockIdx.x;
  const int M = Mact[s];
  const int64_t base = act_off[s];
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    I_next[base + i] = i;
    g_res[base + i] = Uoff_cur[s] + I_cur[base + i];
    upos[base + i] = lpos[base + i];
  }
  if (threadIdx.x == 0) Ucnt_next[s] = M;
}

// out[r] = x[g[r]] for r < *Mp rows of d floats (the residual rows of a
// densified block, contiguous for the Wo GEMM's residual epilogue).
__global__ void k_gather_rows(const int64_t* __restrict__ Mp, int d, const float* __restrict__ x,
                              const int64_t* __restrict__ g, float* __restrict__ out) {
  const int64_t M = *Mp;
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * wpb + (threadIdx.x >> 5); r < M; r += (int64_t)gridDim.x * wpb) {
    const float* src = x + g[r] * d;
    for (int c = lane; c < d; c += 32) out[r * d + c] = src[c];
  }
}

// bf16 copy of *Mp fp32 rows of d (a bf16 engine's Wo operand when the
// attention ran on CUDA cores).
__global__ void k_to_bf16(const int64_t* __restrict__ Mp, int d, const float* __restrict__ x,
                          bf16* __restrict__ out) {
  const int64_t n = *Mp * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(x[i]);
}

// x = xh + xl (the tcgen05 attention's two-term split) as fp32 rows, for the
// CUDA-core quantizer (vq_heads > 1).
__global__ void k_join_split(const int64_t* __restrict__ Mp, int d, const bf16* __restrict__ xh,
                             const bf16* __restrict__ xl, float* __restrict__ out) {
  const int64_t n = *Mp * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __bfloat162float(xh[i]) + __bfloat162float(xl[i]);
}

// The H codes of a location as one exact key: code_h << (h * qbits), either
// as 32 bits (key32, the MODE 1 code operand directly) or 64 bits (tup, to be
// numbered by k_dedup<2> first).
// Test hook (Engine::set_code_override): code of active location loc of
// layer b := ovr[((s0 + s) L + b) R1 + k][p] unless that entry is -1.
__global__ void k_code_override(const int64_t* __restrict__ Mp, const int32_t* __restrict__ lrow,
                                const int16_t* __restrict__ lpos, int R1, int T, int L, int b,
                                int64_t s0, const int16_t* __restrict__ ovr,
                                int32_t* __restrict__ code) {
  const int64_t M = *Mp;
  for (int64_t loc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; loc < M;
       loc += (int64_t)gridDim.x * blockDim.x) {
    const int r = lrow[loc];
    const int s = r / R1, k = r - s * R1;
    const int16_t v = ovr[(((s0 + s) * L + b) * R1 + k) * T + lpos[loc]];
    if (v >= 0) code[loc] = v;
  }
}

__global__ void k_pack_codes(const int64_t* __restrict__ Mp, int H, int qbits,
                             const int32_t* __restrict__ code, unsigned long long* __restrict__ tup,
                             int32_t* __restrict__ key32) {
  const int64_t M = *Mp;
  const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l >= M) return;
  unsigned long long k = 0;
  for (int h = 0; h < H; ++h) k |= (unsigned long long)(uint32_t)code[l * H + h] << (h * qbits);
  if (tup) tup[l] = k;
  if (key32) key32[l] = (int32_t)(uint32_t)k;
}

// ---------------------------------------------------------------- (e)
// LN_f output -> head linear -> (pad mask) -> log_softmax in double
// (proj/src/dedup.cpp:284-308, tensor.cpp:107-124). One warp per unique row.
template <typename TA>
__global__ void k_head(const int64_t* __restrict__ Mp, int d, int V, int lastV, int T,
                       const TA* __restrict__ h, const TA* __restrict__ W,
                       const float* __restrict__ b, const int16_t* __restrict__ upos,
                       double* __restrict__ lpV) {
  const int64_t M = *Mp;
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  double logit[16];
  for (int64_t r = blockIdx.x * wpb + (threadIdx.x >> 5); r < M; r += (int64_t)gridDim.x * wpb) {
    // one pass over the row for all V logits; products of fp32 / bf16
    // operands are exact in double
    double acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = 0.0;
    for (int e = lane; e < d; e += 32) {
      const double he = (double)to_f<TA>(h[r * d + e]);
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < V) acc[c] += he * (double)to_f<TA>(W[(int64_t)e * V + c]);
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if (c >= V) break;
      logit[c] = warp_sum(acc[c]) + (double)b[c];
      if (lastV < V && c >= lastV && upos[r] == T - 1) logit[c] = -1e30;
    }
    double mx = logit[0];
    for (int c = 1; c < V; ++c) mx = fmax(mx, logit[c]);
    double sum = 0.0;
    for (int c = 0; c < V; ++c) sum += exp(logit[c] - mx);
    const double lse = mx + log(sum);
    if (lane < V) {
      double v = 0.0;
      for (int c = 0; c < V; ++c)
        if (c == lane) v = logit[c] - lse;
      lpV[r * V + lane] = v;
    }
  }
}

// Segmented psi-ratio sum, one warp per sample (proj/src/dedup.cpp:310-321,
// 410-417). lp_k - lp_0 is accumulated only over positions p >= t1_k, where
// row k's target token or hidden state can differ from the base row's; the
// shared prefix cancels exactly. E = diag + sum_{k>=1} c * exp(0.5 (lp_k - lp_0)).
// One CTA (256 threads) per sample: warp w takes rows k = 1 + w, 1 + w + 8,
// ..., its lanes the positions of a row (sum in a fixed shuffle tree); the
// row terms land in shared memory and warp 0 adds them in row order, so a
// sample's energy does not depend on the micro-batch it ran in.
constexpr int ELOC_THREADS = 256;
__global__ void __launch_bounds__(ELOC_THREADS) k_eloc(
    int S, int R1, int T, int g, int V, double coeff, const int32_t* __restrict__ K,
    const double* __restrict__ diag, const int32_t* __restrict__ row_bond,
    const int32_t* __restrict__ row_t1, const int64_t* __restrict__ row_aoff,
    const int64_t* __restrict__ act_off, const int32_t* __restrict__ tok0,
    const int32_t* __restrict__ bonds, const int32_t* __restrict__ I_L,
    const int64_t* __restrict__ Uoff_L, const double* __restrict__ lpV,
    double* __restrict__ e_out, double* __restrict__ logpsi, double* __restrict__ lp_rows) {
  extern __shared__ double el_term[];  // [R1]
  __shared__ double lp0_s;
  const int s = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int32_t* t0 = tok0 + (int64_t)s * T;
  const int64_t base = act_off[s];
  const int64_t uo = Uoff_L[s];
  if (w == 0) {
    double lp0 = 0.0;
    for (int p = lane; p < T; p += 32) lp0 += lpV[(uo + I_L[base + p]) * V + t0[p]];
    lp0 = warp_sum(lp0);
    if (lane == 0) lp0_s = lp0;
  }
  const int Ks = K[s];
  __syncthreads();
  const double lp0 = lp0_s;
  for (int k = 1 + w; k < Ks; k += nw) {
    const int64_t r = (int64_t)s * R1 + k;
    const int bond = row_bond[r], t1 = row_t1[r], a = t1 + 1;
    const int64_t rloc = base + row_aoff[r];
    double diff = 0.0;
    for (int p = max(t1, 0) + lane; p < T; p += 32) {  // t1 = -1 in the no-reuse regime
      const int64_t u0 = uo + I_L[base + p];
      const int64_t uk = p < a ? u0 : uo + I_L[rloc + (p - a)];
      diff += lpV[uk * V + row_token(t0, bonds, bond, g, p)] - lpV[u0 * V + t0[p]];
    }
    diff = warp_sum(diff);
    if (lane == 0) {
      el_term[k] = coeff * exp(0.5 * diff);
      if (lp_rows) lp_rows[r] = lp0 + diff;
    }
  }
  __syncthreads();
  if (w == 0) {
    double acc = 0.0;
    for (int k = 1 + lane; k < Ks; k += 32) acc += el_term[k];
    acc = warp_sum(acc);
    if (lane == 0) {
      e_out[s] = diag[s] + acc;
      logpsi[s] = 0.5 * lp0;
      if (lp_rows) lp_rows[(int64_t)s * R1] = lp0;
    }
  }
}

// fill_stats (proj/src/trainer.cpp:184-198) over a device-resident shard of
// local energies, in a fixed summation order (deterministic). One CTA of
// 1024 threads; each thread sums a contiguous slice, then a fixed tree.
//   mode 0: red[0] = n, red[1] = sum Re E, red[2] = #non-finite
//   mode 1: red[3] = sum (Re E - red[1] / red[0])^2, after red[0..2] have
//           been summed over the ranks (the reference's two-pass variance)
__global__ void __launch_bounds__(1024) k_stats(int64_t n, const double* __restrict__ e,
                                                double* __restrict__ red, int mode) {
  __shared__ double sh[1024];
  __shared__ double bad[1024];
  const int tid = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t b = tid * per, en = min(n, b + per);
  const double mean = mode == 1 ? red[1] / red[0] : 0.0;
  double acc = 0.0, nf = 0.0;
  for (int64_t i = b; i < en; ++i) {
    const double v = e[i];
    if (mode == 0) {
      if (isfinite(v)) acc += v;
      else nf += 1.0;
    } else if (isfinite(v)) {
      acc += (v - mean) * (v - mean);
    }
  }
  sh[tid] = acc;
  bad[tid] = nf;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (tid < o) {
      sh[tid] += sh[tid + o];
      bad[tid] += bad[tid + o];
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (mode == 0) {
      red[0] = double(n);
      red[1] = sh[0];
      red[2] = bad[0];
    } else {
      red[3] = sh[0];
    }
  }
}

}  // namespace vqb

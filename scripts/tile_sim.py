"""Developer tool (CPU only): attention tile packing / row-order policies under
the softmax cost model of k_tc_attention (csrc/tc_attention.cuh).

A tile's head takes time ~ c0 + c1 * max over row quadrants of
ceil(live 16-column score chunks of the quadrant / 4): the four warps of a
quadrant (one SM sub-partition) split its live chunks, and every quadrant
waits for the slowest one at the MMA hand-off. This script draws seeded
zero-Sz samples of a workload, builds the connected rows' (a, len) lists and
compares policies by that cost.

    python scripts/tile_sim.py [L] [n_samples]
"""
import sys

import numpy as np


def rows_of(L, rng, g=2):
    N = L * L
    cfg = np.zeros(N, np.int8)
    cfg[rng.permutation(N)[: N // 2]] = 1
    T = N // g
    out = []
    for y in range(L):
        for x in range(L):
            i = y * L + x
            for j in (y * L + (x + 1) % L, ((y + 1) % L) * L + x):
                if cfg[i] != cfg[j]:
                    t1 = min(i // g, j // g)
                    if T - (t1 + 1) > 0:
                        out.append(t1 + 1)  # a
    return T, sorted(out)  # ascending a = descending length


def quad_chunks(tile, T):
    """tile: list of (a, len) in lane order. Returns live chunk count per quadrant."""
    a_r, lo_r = [], []
    r = 0
    for a, n in tile:
        for p in range(n):
            a_r.append(a)
            lo_r.append(r)
        r += n
    nloc = len(a_r)
    res = []
    for q in range(4):
        rows = range(32 * q, min(32 * q + 32, nloc))
        if len(rows) == 0:
            res.append(0)
            continue
        wb_end = (max(a_r[i] for i in rows) + 15) // 16
        olo = min(lo_r[i] for i in rows)
        ohi = max(rows)
        nown = (ohi + 16) // 16 - olo // 16
        res.append(wb_end + nown)
    return res


def pack_two_pointer(rows, T, order="long_first"):
    """rows: list of a ascending, base row (a=0) first. Returns tiles."""
    srt = [(0, T)] + [(a, T - a) for a in rows]
    i, j = 0, len(srt) - 1
    tiles = []
    while i <= j:
        first = [srt[i]]
        c = srt[i][1]
        i += 1
        while i <= j and c + srt[i][1] <= 128:
            first.append(srt[i])
            c += srt[i][1]
            i += 1
        tail = []
        while j >= i and c + srt[j][1] <= 128:
            tail.append(srt[j])
            c += srt[j][1]
            j -= 1
        if order == "long_first":
            tiles.append(first + tail)
        elif order == "short_first":
            tiles.append(tail[::-1] + first[::-1])
        elif order == "short_first_b":
            tiles.append(tail + first)
        elif order == "best":
            cands = [first + tail, tail[::-1] + first[::-1], tail + first, first[::-1] + tail,
                     tail[::-1] + first]
            tiles.append(min(cands, key=lambda t: cost(quad_chunks(t, T))))
    return tiles


def pack_sorted(rows, T):
    srt = [(0, T)] + [(a, T - a) for a in rows]
    tiles, cur, c = [], [], 0
    for r in srt:
        if c + r[1] > 128:
            tiles.append(cur)
            cur, c = [], 0
        cur.append(r)
        c += r[1]
    if cur:
        tiles.append(cur)
    return tiles


def cost(qc):
    return max((n + 3) // 4 for n in qc)


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    rng = np.random.default_rng(1)
    pols = {
        "two_pointer long_first (current)": lambda r, T: pack_two_pointer(r, T, "long_first"),
        "two_pointer short_first(rev)": lambda r, T: pack_two_pointer(r, T, "short_first"),
        "two_pointer short_first": lambda r, T: pack_two_pointer(r, T, "short_first_b"),
        "two_pointer best-of-5": lambda r, T: pack_two_pointer(r, T, "best"),
        "sorted greedy": pack_sorted,
    }
    agg = {k: [0, 0, 0, 0, np.zeros(6)] for k in pols}
    for s in range(ns):
        T, rows = rows_of(L, rng)
        for k, f in pols.items():
            tiles = f(rows, T)
            a = agg[k]
            for t in tiles:
                qc = quad_chunks(t, T)
                a[0] += 1
                a[1] += cost(qc)
                a[2] += sum((n + 3) // 4 for n in qc) / 4
                a[3] += sum(n for _, n in t)
                a[4][cost(qc)] += 1
    for k, a in agg.items():
        print(f"{k:36s} tiles {a[0]:6d} fill {a[3] / a[0]:6.1f} sum_max_slots {a[1]:6d} "
              f"({a[1] / a[0]:.2f}/tile; mean-quadrant {a[2] / a[0]:.2f}) hist {a[4].astype(int)}")


if __name__ == "__main__":
    main()


def efficiency(L=16, ns=4, order="short_first_b", cw=16):
    """live (query, key) pairs / lanes x columns of the live chunks (chunk width cw)."""
    rng = np.random.default_rng(1)
    live = tot = tot_q = 0
    for s in range(ns):
        T, rows = rows_of(L, rng)
        for tile in pack_two_pointer(rows, T, order):
            a_r, lo_r = [], []
            r = 0
            for a, n in tile:
                a_r += [a] * n
                lo_r += [r] * n
                r += n
            for q in range(4):
                rr = range(32 * q, min(32 * q + 32, len(a_r)))
                if not len(rr):
                    continue
                live += sum(a_r[i] + (i - lo_r[i] + 1) for i in rr)
                nb = (max(a_r[i] for i in rr) + cw - 1) // cw
                nown = (max(rr) + cw) // cw - min(lo_r[i] for i in rr) // cw
                tot += (nb + nown) * cw * 32
    return live / tot


def full_fraction(L=16, ns=4, order="short_first_b"):
    """fraction of a quadrant's live chunks that need no mask (every live row uses all 16)."""
    rng = np.random.default_rng(1)
    full = tot = 0
    for s in range(ns):
        T, rows = rows_of(L, rng)
        for tile in pack_two_pointer(rows, T, order):
            a_r, lo_r = [], []
            r = 0
            for a, n in tile:
                a_r += [a] * n
                lo_r += [r] * n
                r += n
            for q in range(4):
                rr = list(range(32 * q, min(32 * q + 32, len(a_r))))
                if not rr:
                    continue
                nb = (max(a_r[i] for i in rr) + 15) // 16
                for c in range(nb):
                    tot += 1
                    full += all(a_r[i] >= 16 * c + 16 for i in rr)
                c0 = min(lo_r[i] for i in rr) // 16
                c1 = (max(rr) + 16) // 16
                for c in range(c0, c1):
                    tot += 1
                    full += all(lo_r[i] <= 16 * c and i >= 16 * c + 15 for i in rr)
    return full / tot

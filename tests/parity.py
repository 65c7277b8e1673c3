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


@dataclass
class ParityReport:
    window: float = GAP_FLAG
    logpsi_tol: float = LOGPSI_TOL
    eloc_rtol: float = ELOC_RTOL
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
    max_dlp: float = 0.0
    max_dlogpsi: float = 0.0
    max_rel_de: float = 0.0
    notes: list = field(default_factory=list)

    def ok(self) -> bool:
        return (self.flips_beyond == 0 and self.u_fail == 0 and self.lp_fail == 0
                and self.logpsi_fail == 0 and self.eloc_fail == 0)

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
                f"flagged_locations={self.flagged_locations}/{self.locations}")


def compare(rep: ParityReport, taps, ref_e, ref_lpsi, gpu_codes, gpu_U, gpu_e, gpu_lpsi,
            gpu_lp_rows, T):
    """One sample. taps: oracle Taps (codes [L, K*T, 1], gaps [L, K*T], lp [K],
    U [L+1]); gpu_codes [L, K*T]; gpu_U [L+1]; gpu_lp_rows [K]."""
    rep.samples += 1
    K = int(taps.K)
    rc = taps.codes[..., 0].reshape(-1, K, T)
    gc = np.asarray(gpu_codes).reshape(-1, K, T)
    gaps = taps.gaps.reshape(-1, K, T)
    L = rc.shape[0]
    rep.locations += rc.size
    rep.flagged_locations += int((gaps < GAP_FLAG).sum())
    mm = rc != gc
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
        rep.lp_fail += int((dlp > 2 * rep.logpsi_tol).sum())
    if clean[0]:
        rep.logpsi_checked += 1
        dl = abs(float(ref_lpsi) - float(gpu_lpsi))
        rep.max_dlogpsi = max(rep.max_dlogpsi, dl)
        rep.logpsi_fail += int(dl > rep.logpsi_tol)
    if clean.all():
        rep.clean_samples += 1
        rep.eloc_checked += 1
        re = abs(float(ref_e) - float(gpu_e)) / max(abs(float(ref_e)), 1e-12)
        rep.max_rel_de = max(rep.max_rel_de, re)
        rep.eloc_fail += int(re > rep.eloc_rtol)

"""Generate the c3/c4/c5 parity fixtures from the REFERENCE ITSELF.

The reference's hot-path sources (oracle/_ref/libvqnqs_ref.so: proj/src/
{flops,tensor,hamiltonian,model,dedup}.cpp compiled unmodified with the Eigen
shim) evaluate a few seeded samples of each BASELINE workload, in plain
double and in bf16-emulation mode (weights snapped to bf16 on both sides,
both operands of every product rounded to bf16). A c4 sample
costs the reference ~110 s and a c5 sample several minutes, which is why the
GPU tests read these fixtures instead of running the CPU checker live.

Per case (parity_<case>.npz):
  samples [n, N] u8, idx [n] (sample indices of the workload's seeded batch),
  e_re [n], logpsi [n]             local_energies (proj/src/trainer.cpp:150-180)
  K [n], U [n, L+1]                connected-set sizes, unique-row counts
  lp_<i> [K_i]                     per-row dedup_log_prob (proj/src/dedup.cpp:272-323)
  codes_<i> [L, K_i*T] int16       per-location VQ codes (vq_apply_rows picks)
  gidx_<i>, gval_<i>               the locations whose top-2 relative distance
                                   gap is below SPARSE_GAP (flat [L*K_i*T]
                                   index, float32 gap); every other location's
                                   gap is >= SPARSE_GAP, which is all the
                                   parity rules need (they only ask < 1e-5 /
                                   < 1e-4)
  ledger [7]                       the reference's FLOP ledger over the n samples

Needs /root/reference (dev container only). Usage:
  python tests/golden/make_golden_large.py [case ...]   (default: all)
"""
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

SPARSE_GAP = 1e-3

# case -> (workload, bf16, sample indices)
CASES = {
    "c3_fp64": ("c3", False, list(range(16))),
    "c3_bf16e": ("c3", True, list(range(16))),
    "c4_fp64": ("c4", False, list(range(8))),
    "c4_bf16e": ("c4", True, list(range(8))),
    "c5_fp64": ("c5", False, list(range(8))),
    "c5_bf16e": ("c5", True, list(range(8))),
}


def _one(args):
    case, i = args
    from oracle import RefLib
    from paper_2212_11296_b200.config import workload
    wl, bf, idx = CASES[case]
    w = workload(wl)
    R = RefLib()
    R.set_bf16(bf)
    m = R.model(w.model, w.weight_seed, snap_bf16=bf)
    h = R.hamiltonian("grid_periodic", w.L, w.L)
    s = R.zero_sz_samples(w.n_sites, idx[i], 1, w.sample_seed)
    t0 = time.time()
    e_re, e_im, lpsi, led = m.local_energies(h, s, workers=1)
    tp = m.taps(h, s[0])
    g = tp.gaps.reshape(-1)
    sel = np.nonzero(g < SPARSE_GAP)[0].astype(np.int32)
    assert tp.codes.shape[-1] == 1 and tp.codes.max() < 32768
    print(f"{case}[{i}] K={tp.K} {time.time() - t0:.0f}s", flush=True)
    return dict(case=case, i=i, sample=s[0], e_re=e_re[0], e_im=e_im[0], logpsi=lpsi[0],
                led=led, K=tp.K, U=tp.U, lp=tp.lp, codes=tp.codes[..., 0].astype(np.int16),
                gidx=sel, gval=g[sel].astype(np.float32))


def main():
    cases = sys.argv[1:] or list(CASES)
    jobs = [(c, i) for c in cases for i in range(len(CASES[c][2]))]
    # the big cases first so the pool's tail is short
    jobs.sort(key=lambda j: {"c5": 0, "c4": 1, "c3": 2}[CASES[j[0]][0]])
    nproc = int(os.environ.get("GOLDEN_PROCS", max(1, (os.cpu_count() or 2) - 1)))
    with mp.get_context("spawn").Pool(nproc) as pool:
        res = pool.map(_one, jobs, chunksize=1)
    for c in cases:
        rs = sorted([r for r in res if r["case"] == c], key=lambda r: r["i"])
        wl, bf, idx = CASES[c]
        out = dict(workload=np.array(wl), bf16=np.array(bf), idx=np.array(idx),
                   samples=np.stack([r["sample"] for r in rs]),
                   e_re=np.array([r["e_re"] for r in rs]),
                   e_im=np.array([r["e_im"] for r in rs]),
                   logpsi=np.array([r["logpsi"] for r in rs]),
                   K=np.array([r["K"] for r in rs]),
                   U=np.stack([r["U"] for r in rs]),
                   ledger=np.sum([r["led"] for r in rs], axis=0),
                   sparse_gap=np.array(SPARSE_GAP))
        for r in rs:
            out[f"lp_{r['i']}"] = r["lp"]
            out[f"codes_{r['i']}"] = r["codes"]
            out[f"gidx_{r['i']}"] = r["gidx"]
            out[f"gval_{r['i']}"] = r["gval"]
        path = os.path.join(HERE, f"parity_{c}.npz")
        np.savez_compressed(path, **out)
        print(c, "->", path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()

"""Diagnostics: gap distribution of GPU-vs-oracle code mismatches."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2212_11296_b200 as P
from oracle import PortLib
from parity import ParityReport, compare
name = sys.argv[1]; n = int(sys.argv[2])
w = P.workload(name); bf = w.precision == "bf16"
port = PortLib(); port.set_bf16(bf)
model = P.VqTransformer.init(w.model, 0, snap_bf16=bf)
eng = P.LocalEnergyEngine(model, P.HamiltonianModel(P.build_lattice("grid2d", (w.L, w.L), True)), w.precision)
om = port.model(w.model, 0, bf); oh = port.hamiltonian("grid_periodic", w.L, w.L)
S = P.zero_sz_samples(w.n_sites, 0, n)
t = time.time(); ref_e, _, ref_l, _ = om.local_energies(oh, S, workers=os.cpu_count()); print("oracle", time.time()-t)
e, l = eng.local_energies(S); K, U, codes = eng.taps(S)
rep = ParityReport(); T = w.model.seq_len
first_gaps = []
for i in range(n):
    tp = om.taps(oh, S[i]); rc = tp.codes[..., 0]
    compare(rep, tp, ref_e[i], ref_l[i], codes[i], U[i], e[i].real, l[i], T)
    mm = rc != codes[i]
    if mm.any():
        b = int(np.argmax(mm.any(axis=1)))
        first_gaps += list(tp.gaps[b][mm[b]])
        print(f"s{i} first mismatch layer {b}: n={int(mm[b].sum())} gaps={np.sort(tp.gaps[b][mm[b]])[:6]} dlogpsi={l[i]-ref_l[i]:.2e} dE_rel={(e[i].real-ref_e[i])/abs(ref_e[i]):.2e} U_ref={tp.U.tolist()} U_gpu={U[i].tolist()}")
    else:
        print(f"s{i} clean dlogpsi={l[i]-ref_l[i]:.2e} dE_rel={(e[i].real-ref_e[i])/abs(ref_e[i]):.2e}")
print(rep.summary())
g = np.array(first_gaps)
if g.size:
    for thr in [1e-6, 1e-5, 3e-5, 1e-4, 3e-4, 1e-3]:
        print(f"first-layer mismatches with gap < {thr:g}: {np.mean(g < thr):.2f}")

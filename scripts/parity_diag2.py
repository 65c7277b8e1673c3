import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2212_11296_b200 as P
from oracle import PortLib
name = sys.argv[1]; n = int(sys.argv[2])
w = P.workload(name); bf = w.precision == "bf16"
port = PortLib(); port.set_bf16(bf)
model = P.VqTransformer.init(w.model, 0, snap_bf16=bf)
eng = P.LocalEnergyEngine(model, P.HamiltonianModel(P.build_lattice("grid2d", (w.L, w.L), True)), w.precision)
om = port.model(w.model, 0, bf); oh = port.hamiltonian("grid_periodic", w.L, w.L)
S = P.zero_sz_samples(w.n_sites, 0, n)
K, U, codes = eng.taps(S); T = w.model.seq_len
for i in range(n):
    tp = om.taps(oh, S[i]); rc = tp.codes[..., 0]; Kk = tp.K
    mm = (rc != codes[i]).reshape(-1, Kk, T)
    L = mm.shape[0]
    for b in range(L):
        for k, p in zip(*np.nonzero(mm[b])):
            earlier = mm[:b, k, :].any()
            g = tp.gaps[b].reshape(Kk, T)[k, p]
            if g >= 1e-5 and not earlier:
                print(f"s{i} L{b} k={k} p={p} gap={g:.2e} ref={rc[b].reshape(Kk,T)[k,p]} gpu={codes[i][b].reshape(Kk,T)[k,p]} rowmm_this_layer={mm[b,k].sum()} base_mm_earlier={mm[:b,0,:].any()} base_mm_pos={np.nonzero(mm[:b,0,:])}")

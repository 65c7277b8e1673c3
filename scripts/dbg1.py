import sys, os, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/oracle")
import paper_2212_11296_b200 as P
from oracle import PortLib
w = P.workload("c1")
eng = P.LocalEnergyEngine(P.VqTransformer.init(w.model, 0), P.HamiltonianModel(P.build_lattice("grid2d", (4, 4), True)), "fp32")
S = P.zero_sz_samples(16, 0, 3)
e, l = eng.local_energies(S)
print("prof", eng.last_profile())
K, U, codes, lps = eng.taps(S)
port = PortLib(); om = port.model(w.model, 0); oh = port.hamiltonian("grid_periodic", 4, 4)
for i in range(3):
    t = om.taps(oh, S[i])
    print(K[i], "gpu", lps[i][:6], "\nref", t.lp[:6], "lpsi", l[i], 0.5 * t.lp[0])
print(eng.connected_log_probs(S[0])[:6])

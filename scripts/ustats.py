"""Developer probe: per-sample active locations M and unique rows U_b at each
layer (engine taps) for a seeded batch of each workload."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2212_11296_b200 as P  # noqa: E402

for name in sys.argv[1:] or ["c3", "c4", "c5"]:
    w = P.workload(name)
    model = P.VqTransformer.init(w.model, w.weight_seed, snap_bf16=True)
    lat = P.build_lattice("grid2d", (w.L, w.L), periodic=True)
    eng = P.LocalEnergyEngine(model, P.HamiltonianModel(lat), precision="bf16", device=0)
    S = P.zero_sz_samples(w.n_sites, 0, 64, w.sample_seed)
    K, U, codes, lps = eng.taps(S)
    U = np.array(U)
    print(name, "K max", int(np.max(K)), "U per layer: mean", np.round(U.mean(0)).astype(int).tolist(),
          "max", U.max(0).tolist(), flush=True)
    eng.close()

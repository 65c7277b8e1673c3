"""Developer timing probe: score-function gradient (LogProbGradient.grad) on
K samples, per workload."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2212_11296_b200 as P  # noqa: E402

for arg in sys.argv[1:] or ["c4_16x16:256"]:
    name, n = arg.split(":")
    w = P.workload(name)
    model = P.VqTransformer.init(w.model, w.weight_seed)
    g = P.LogProbGradient(model)
    S = P.zero_sz_samples(w.n_sites, 0, int(n), w.sample_seed)
    wts = np.linspace(-1, 1, int(n))
    g.grad(S[:8], wts[:8])
    torch.cuda.synchronize()
    dts = []
    for _ in range(3):
        t0 = time.perf_counter()
        g.grad(S, wts)
        dts.append(time.perf_counter() - t0)
    print(f"{name} samples={n} grad {min(dts):.3f}s ({int(n) / min(dts):.0f} samples/s)", flush=True)

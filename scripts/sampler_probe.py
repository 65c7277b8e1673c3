"""Developer timing probe: GPU sampler throughput (samples/s) per workload."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2212_11296_b200 as P  # noqa: E402

for arg in sys.argv[1:] or ["c4_16x16:8192"]:
    name, n = arg.split(":")
    w = P.workload(name)
    model = P.VqTransformer.init(w.model, w.weight_seed, snap_bf16=w.precision == "bf16")
    lat = P.build_lattice("grid2d", (w.L, w.L), periodic=True)
    eng = P.LocalEnergyEngine(model, P.HamiltonianModel(lat), precision=w.precision)
    eng.sample(64, 1)
    torch.cuda.synchronize()
    dts = []
    for rep in range(3):  # the first call also sizes the buffers
        t0 = time.perf_counter()
        cfg, lp = eng.sample(int(n), 2)
        dts.append(time.perf_counter() - t0)
    dt = min(dts)
    print(f"{name} samples={n} {dt:.2f}s (runs {', '.join(f'{x:.2f}' for x in dts)}) "
          f"{int(n) / dt:.0f} samples/s launches={eng.last_launch_count()} "
          f"mean lp {lp.mean():.3f} mean Sz {cfg.mean() - 0.5:+.4f}", flush=True)

"""Developer timing probe (not the bench contract): device-resident throughput
of one batch per workload plus the engine's stage profile.

    python scripts/quickbench.py c3_10x10:1024 c4_16x16:1024 c5_12x12:1024 [c4_16x16:256:fp32]
prints: workload evals/s ms/step attention_ms vq_ms rescored tile_fill (locations per tile)
"""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2212_11296_b200 as P  # noqa: E402


def run(name: str, batch: int, steps: int = 3, precision: str = "") -> None:
    w = P.workload(name)
    precision = precision or w.precision
    model = P.VqTransformer.init(w.model, w.weight_seed, snap_bf16=precision == "bf16")
    lat = P.build_lattice("grid2d", (w.L, w.L), periodic=True)
    eng = P.LocalEnergyEngine(model, P.HamiltonianModel(lat), precision=precision, device=0)
    S = P.zero_sz_samples(w.n_sites, 0, batch, w.sample_seed)
    dS = torch.from_numpy(S).cuda()
    dE = torch.empty(batch, dtype=torch.float64, device="cuda")
    dL = torch.empty(batch, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    led = eng.local_energies_device(dS, dE, dL, st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.local_energies_device(dS, dE, dL, st)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    prof = eng.last_profile()
    evals = led.other // w.model.seq_len  # connected configurations
    fill = prof[3] / prof[11] if len(prof) > 11 and prof[11] else 0.0
    print(f"{name}{'/' + precision if precision != w.precision else ''} {evals / ms * 1e3:.0f} "
          f"{ms:.1f} {prof[7]:.1f} {prof[6]:.1f} {prof[8]:.0f} "
          f"tile_fill={fill:.1f}", flush=True)


if __name__ == "__main__":
    for arg in sys.argv[1:] or ["c3_10x10:1024", "c4_16x16:1024", "c5_12x12:1024"]:
        n, b, *pr = arg.split(":")
        run(n, int(b), precision=pr[0] if pr else "")

"""Generate the committed golden fixtures from the REFERENCE ITSELF.

Runs the reference's own hot-path sources (oracle/_ref/libvqnqs_ref.so:
proj/src/{flops,tensor,hamiltonian,model,dedup}.cpp compiled unmodified with
the Eigen shim) on seeded inputs and writes small .npz fixtures:

  golden_<case>.npz : samples, per-sample E_loc / logpsi, the ledger, and for
                      the first few samples the taps (U counts, VQ codes,
                      top-2 gaps, per-row log-probs).
  golden_sample.npz : the reference sampler's configurations and log-probs
                      (VqTransformer::sample) for a few seeded cases.
  ckpt_c1.vqnqs, report_c1/report.{csv,json} : the reference's checkpoint
                      file and measurement report (the §8(f) wire formats).

Needs /root/reference (dev container only). The fixtures travel with the repo;
tests/test_oracle.py checks the C restatement (oracle/_port) against them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import RefLib  # noqa: E402
from paper_2212_11296_b200.config import ModelConfig, workload  # noqa: E402

CASES = {
    # name: (workload or explicit cfg, lattice, bf16, n_samples, n_taps)
    "c1_fp64": ("c1", None, False, 64, 8),
    "c2_fp64": ("c2", None, False, 16, 4),
    "c3_bf16": ("c3", None, True, 2, 2),
    # reference test-suite shapes (proj/tests/test_dedup.cpp small_cfg):
    # vq_heads=2, codebook 8, trailing half block, open 4x4 lattice
    "small_open4x4": (ModelConfig(n_sites=16, group_size=2, d_hidden=16, n_heads=2,
                                  n_blocks=1, trailing_half_block=True, vq_heads=2,
                                  vq_codebook=8), ("grid", 4, 4), False, 32, 4),
    "small_chain6_g3": (ModelConfig(n_sites=6, group_size=3, d_hidden=24, n_heads=2,
                                    n_blocks=2, trailing_half_block=False, vq_heads=2,
                                    vq_codebook=16), ("chain_periodic", 6, 0), False, 16, 4),
}


# the reference's autoregressive sampler (VqTransformer::sample,
# proj/src/model.cpp:485-525): name -> (cfg, bf16, count, seed)
SAMPLE_CASES = {
    "c1_fp64": ("c1", False, 32, 7),
    "c1_bf16": ("c1", True, 16, 11),
    "small_open4x4": ("small_open4x4", False, 16, 3),
}


def make_samples(R):
    out = {}
    for name, (wl, bf, count, seed) in SAMPLE_CASES.items():
        cfg = workload(wl).model if wl.startswith("c") else CASES[wl][0]
        R.set_bf16(bf)
        m = R.model(cfg, 0, snap_bf16=bf)
        configs, lp = m.sample(count, seed)
        out[f"{name}_configs"] = configs
        out[f"{name}_log_probs"] = lp
        out[f"{name}_seed"] = np.array(seed)
        print("sample", name, configs.sum(1)[:6], lp[:3])
    np.savez_compressed(os.path.join(HERE, "golden_sample.npz"), **out)


def make_wire(R):
    """The reference's checkpoint file for the c1 model (seed 0) and its
    measurement report (measure_flops, 8 x 2 samples, Rng(5), periodic 4x4)."""
    cfg = workload("c1").model
    R.set_bf16(False)
    m = R.model(cfg, 0)
    m.save_checkpoint(os.path.join(HERE, "ckpt_c1.vqnqs"))
    m.measure_and_emit(R.hamiltonian("grid_periodic", 4, 4), 8, 2, 5,
                       os.path.join(HERE, "report_c1"))


def main():
    R = RefLib()
    if "--sample-only" in sys.argv:
        make_samples(R)
        return
    if "--wire-only" in sys.argv:
        make_wire(R)
        return
    make_samples(R)
    make_wire(R)
    for name, (wl, lat, bf, ns, nt) in CASES.items():
        if isinstance(wl, str):
            w = workload(wl)
            cfg, L = w.model, w.L
            lat = ("grid_periodic", L, L)
        else:
            cfg = wl
        R.set_bf16(bf)
        m = R.model(cfg, 0, snap_bf16=bf)
        h = R.hamiltonian(lat[0], lat[1], lat[2])
        S = R.zero_sz_samples(cfg.n_sites, 0, ns, 1)
        e_re, e_im, lpsi, led = m.local_energies(h, S, workers=os.cpu_count() or 4)
        out = dict(samples=S, e_re=e_re, e_im=e_im, logpsi=lpsi, ledger=led,
                   bonds=h.bonds(), bf16=np.array(bf),
                   cfg=np.array([cfg.n_sites, cfg.group_size, cfg.d_hidden, cfg.n_heads,
                                 cfg.n_blocks, int(cfg.trailing_half_block),
                                 int(cfg.vq_enabled), cfg.vq_heads, cfg.vq_codebook]),
                   vq_init_scale=np.array(cfg.vq_init_scale),
                   lattice=np.array([{"grid": 1, "grid_periodic": 2, "chain": 0,
                                      "chain_periodic": 3}[lat[0]], lat[1], lat[2]]))
        params = m.params()
        out["param_checksums"] = np.array([np.float64(p.sum()) for _, p in params])
        out["param_first"] = np.array([p.reshape(-1)[0] for _, p in params])
        for i in range(nt):
            t = m.taps(h, S[i])
            out[f"taps{i}_U"] = t.U
            out[f"taps{i}_codes"] = t.codes
            out[f"taps{i}_gaps"] = t.gaps
            out[f"taps{i}_lp"] = t.lp
        np.savez_compressed(os.path.join(HERE, f"golden_{name}.npz"), **out)
        print(name, "E[:3]", e_re[:3], "ledger", led.tolist())


if __name__ == "__main__":
    main()

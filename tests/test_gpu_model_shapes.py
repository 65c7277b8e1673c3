"""GPU parity beyond the BASELINE shapes: the reference's own model variants.

* trailing half block (attention only, no VQ, no FFN) -> densify_attention
  (proj/src/dedup.cpp:187-211; proj/src/model.cpp:164-166);
* vq_heads > 1: per-head argmin over [H*Q x d/H] codebooks
  (proj/src/model.cpp:283-319) and the code-tuple dedup key
  (proj/src/dedup.cpp:156-159);
* vq_enabled = false (the paper's "Baseline" transformer);
* the reference's DEFAULT ModelConfig (proj/include/vqnqs/model.hpp:13-27);
* the paper's table-1 architecture: d = 256, 8 heads, three blocks plus a
  half block, VQ with 1/2/4/8 heads of 64 codes.

Against the reference-generated fixtures where they exist
(tests/golden/golden_small_*.npz, written by oracle/_ref), and otherwise
against the oracle's C restatement run live (itself pinned bit-for-bit to the
reference, tests/test_oracle.py).
"""
import os

import numpy as np
import pytest

import paper_2212_11296_b200 as P
from paper_2212_11296_b200.config import ModelConfig
from parity import (BF16_ELOC_RTOL, BF16_LOGPSI_TOL, BF16_WINDOW, ParityReport, compare,
                    heisenberg_coeffs)

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
LATTICES = {"chain": ("chain1d", False), "grid": ("grid2d", False),
            "grid_periodic": ("grid2d", True), "chain_periodic": ("chain1d", True)}
NAMES = {0: "chain", 1: "grid", 2: "grid_periodic", 3: "chain_periodic"}


def lattice(kind, lx, ly):
    k, per = LATTICES[kind]
    return P.build_lattice(k, (lx, ly) if k == "grid2d" else (lx,), periodic=per)


def run_gpu(cfg, lat, S, precision, snap):
    model = P.VqTransformer.init(cfg, 0, snap_bf16=snap)
    eng = P.LocalEnergyEngine(model, P.HamiltonianModel(lat), precision=precision)
    led = P.Ledger()
    e, lpsi = eng.local_energies(S, led)
    K, U, codes, lps = eng.taps(S)
    assert np.array_equal([0.5 * lp[0] for lp in lps], lpsi)
    return e, lpsi, led, K, U, codes, lps


@pytest.mark.parametrize("name", ["small_open4x4", "small_chain6_g3"])
def test_reference_fixture_models(name):
    """Half block + 2 VQ heads (open 4x4, codebook 8, d = 16) and 2 VQ heads
    with group_size 3 on a periodic chain (d = 24): against the reference's
    own outputs (local energies, logpsi, ledger, and per-location codes, U
    and row log-probs of the tapped samples)."""
    g = np.load(os.path.join(GOLDEN, f"golden_{name}.npz"))
    c = g["cfg"]
    cfg = ModelConfig(n_sites=int(c[0]), group_size=int(c[1]), d_hidden=int(c[2]),
                      n_heads=int(c[3]), n_blocks=int(c[4]), trailing_half_block=bool(c[5]),
                      vq_enabled=bool(c[6]), vq_heads=int(c[7]), vq_codebook=int(c[8]),
                      vq_init_scale=float(g["vq_init_scale"]))
    lk = g["lattice"]
    lat = lattice(NAMES[int(lk[0])], int(lk[1]), int(lk[2]))
    assert np.array_equal(lat.bonds, g["bonds"])
    S = g["samples"]
    e, lpsi, led, K, U, codes, lps = run_gpu(cfg, lat, S, "fp32", False)
    rep = ParityReport()
    i = 0
    while f"taps{i}_U" in g:
        class Taps:
            pass
        t = Taps()
        t.K, t.U, t.codes, t.gaps, t.lp = (int(K[i]), g[f"taps{i}_U"], g[f"taps{i}_codes"],
                                           g[f"taps{i}_gaps"], g[f"taps{i}_lp"])
        assert t.codes.shape[0] == cfg.n_layers and t.lp.shape[0] == K[i]
        compare(rep, t, g["e_re"][i], g["logpsi"][i], codes[i], U[i], e[i].real, lpsi[i], lps[i],
                cfg.seq_len, coeffs=heisenberg_coeffs(S[i], lat.bonds))
        i += 1
    print(f"\n[{name}] {rep.summary()}")
    assert i > 0 and rep.ok(), rep.summary() + "\n" + "\n".join(rep.notes[:10])
    # every sample's energy and logpsi (not only the tapped ones)
    np.testing.assert_allclose(lpsi, g["logpsi"], atol=1e-5, rtol=0)
    np.testing.assert_allclose(e.real, g["e_re"], rtol=1e-4, atol=1e-4 * np.abs(g["e_re"]).max())
    assert np.array_equal(led.as_array(), g["ledger"])


def port_parity(port, cfg, lat_kind, lx, ly, n, precision="fp32", min_clean=0.9):
    bf = precision == "bf16"
    lat = lattice(lat_kind, lx, ly)
    S = P.zero_sz_samples(cfg.n_sites, 0, n, 1)
    e, lpsi, led, K, U, codes, lps = run_gpu(cfg, lat, S, precision, bf)
    port.set_bf16(bf)
    om = port.model(cfg, 0, snap_bf16=bf)
    oh = port.hamiltonian(lat_kind, lx, ly)
    assert np.array_equal(oh.bonds(), lat.bonds)
    ref_e, _, ref_lpsi, ref_led = om.local_energies(oh, S, workers=os.cpu_count() or 4)
    rep = (ParityReport(window=BF16_WINDOW, logpsi_tol=BF16_LOGPSI_TOL, eloc_rtol=BF16_ELOC_RTOL)
           if bf else ParityReport())
    for i in range(n):
        compare(rep, om.taps(oh, S[i]), ref_e[i], ref_lpsi[i], codes[i], U[i], e[i].real,
                lpsi[i], lps[i], cfg.seq_len, coeffs=heisenberg_coeffs(S[i], lat.bonds))
    print(f"\n[{cfg} {precision}] {rep.summary()}")
    assert rep.ok(), rep.summary() + "\n" + "\n".join(rep.notes[:10])
    assert rep.clean_rows >= min_clean * rep.rows
    if rep.clean_samples == rep.samples:
        assert np.array_equal(led.as_array(), ref_led)
    return rep


def test_reference_default_model_config(port):
    """ModelConfig{} of the reference (n_sites 4, d 32, 4 heads, 2 blocks +
    the half block, one 64-code VQ head, init scale 0.05) on its 4-site chain."""
    port_parity(port, ModelConfig(), "chain", 4, 0, 6)


@pytest.mark.parametrize("vq_heads", [1, 2, 4, 8])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_paper_architecture(port, vq_heads, precision):
    """The paper's VQ-NQS (table 1): d = 256, 8 attention heads, three blocks
    plus an attention-only half block, VQ with H heads of 64 codes
    (6H bits), on the periodic 4x4 Heisenberg lattice."""
    cfg = ModelConfig(n_sites=16, group_size=2, d_hidden=256, n_heads=8, n_blocks=3,
                      trailing_half_block=True, vq_enabled=True, vq_heads=vq_heads,
                      vq_codebook=64, vq_init_scale=1.0 / 256)
    port_parity(port, cfg, "grid_periodic", 4, 4, 12, precision,
                min_clean=0.9 if precision == "fp32" else 0.6)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_baseline_transformer_without_vq(port, precision):
    """vq_enabled = false (the paper's baseline): every block densifies."""
    cfg = ModelConfig(n_sites=36, group_size=2, d_hidden=64, n_heads=4, n_blocks=2,
                      trailing_half_block=True, vq_enabled=False)
    port_parity(port, cfg, "grid_periodic", 6, 6, 8, precision)


def test_wide_code_tuples_take_the_numbering_pass(port):
    """8 VQ heads x 1024 codes = 80 bits of code tuple: refused (> 63 bits);
    6 heads x 1024 codes = 60 bits: numbered by the extra dedup pass."""
    cfg = ModelConfig(n_sites=16, group_size=2, d_hidden=48, n_heads=4, n_blocks=2,
                      trailing_half_block=False, vq_enabled=True, vq_heads=6,
                      vq_codebook=1024, vq_init_scale=1.0 / 48)
    port_parity(port, cfg, "grid_periodic", 4, 4, 8)
    bad = ModelConfig(n_sites=16, group_size=2, d_hidden=64, n_heads=4, n_blocks=1,
                      trailing_half_block=False, vq_heads=8, vq_codebook=1024)
    with pytest.raises(P.CapabilityError):
        P.LocalEnergyEngine(P.VqTransformer.init(bad, 0),
                            P.HamiltonianModel(lattice("grid_periodic", 4, 4)))

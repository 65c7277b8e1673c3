"""Edge-case inputs on the GPU path, against the oracle (tests/parity.py
contract): the configurations at the two ends of the Heisenberg connected set
(proj/src/hamiltonian.cpp:41-74) and degenerate batches.

- fully polarised (all up / all down): no antiparallel bond, K = 1, the
  diagonal term only, so the connected stage emits no rows at all;
- Néel (checkerboard): every bond antiparallel, K = n_bonds + 1, the largest
  connected set;
- a batch of one, a batch of identical samples, and an empty batch.
"""
import os

import numpy as np
import pytest

import paper_2212_11296_b200 as P
from parity import ParityReport, compare
from parity import BF16_ELOC_RTOL, BF16_LOGPSI_TOL, BF16_WINDOW

pytestmark = pytest.mark.gpu


def _setup(port, name):
    w = P.workload(name)
    bf = w.precision == "bf16"
    model = P.VqTransformer.init(w.model, w.weight_seed, snap_bf16=bf)
    lat = P.build_lattice("grid2d", (w.L, w.L), periodic=True)
    eng = P.LocalEnergyEngine(model, P.HamiltonianModel(lat), precision=w.precision)
    port.set_bf16(bf)
    om = port.model(w.model, w.weight_seed, snap_bf16=bf)
    oh = port.hamiltonian("grid_periodic", w.L, w.L)
    return w, eng, om, oh, lat


def _edge_configs(w):
    n = w.n_sites
    up = np.ones(n, np.uint8)
    down = np.zeros(n, np.uint8)
    x, y = np.meshgrid(np.arange(w.L), np.arange(w.L), indexing="xy")
    neel = ((x + y) % 2).reshape(-1).astype(np.uint8)
    return np.stack([up, down, neel, 1 - neel])


@pytest.mark.parametrize("name", ["c1_4x4", "c3_10x10"])
def test_edge_configurations(port, name):
    w, eng, om, oh, lat = _setup(port, name)
    S = _edge_configs(w)
    bf = w.precision == "bf16"
    ref_e, _, ref_lpsi, _ = om.local_energies(oh, S, workers=os.cpu_count() or 8)
    e, lpsi = eng.local_energies(S, None)
    K, U, codes, lps = eng.taps(S)
    nb = len(lat.bonds)
    assert list(K) == [1, 1, nb + 1, nb + 1]
    rep = (ParityReport(window=BF16_WINDOW, logpsi_tol=BF16_LOGPSI_TOL, eloc_rtol=BF16_ELOC_RTOL)
           if bf else ParityReport())
    for i in range(len(S)):
        compare(rep, om.taps(oh, S[i]), ref_e[i], ref_lpsi[i], codes[i], U[i], e[i].real,
                lpsi[i], lps[i], w.model.seq_len)
    print(f"\n[{name} edges] {rep.summary()}")
    assert rep.ok(), rep.summary() + "\n" + "\n".join(rep.notes[:10])
    # the polarised states are diagonal: E = (1/4) sum_bonds z_i z_j = n_bonds / 4
    assert np.allclose(e[:2].real, nb / 4.0, rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", ["c1_4x4", "c3_10x10"])
def test_degenerate_batches(port, name):
    w, eng, om, oh, lat = _setup(port, name)
    S = P.zero_sz_samples(w.n_sites, 0, 6, w.sample_seed)
    e_all, l_all = eng.local_energies(S, None)
    # a batch of one gives the same numbers as the same sample inside a batch
    for i in (0, 5):
        e1, l1 = eng.local_energies(S[i:i + 1], None)
        assert e1.shape == (1,) and np.array_equal(e1, e_all[i:i + 1])
        assert np.array_equal(l1, l_all[i:i + 1])
    # identical samples: identical outputs
    rep = np.repeat(S[2:3], 5, axis=0)
    e_r, l_r = eng.local_energies(rep, None)
    assert np.all(e_r == e_all[2]) and np.all(l_r == l_all[2])
    # an empty batch
    e0, l0 = eng.local_energies(S[:0], None)
    assert e0.shape == (0,) and l0.shape == (0,)


def test_more_bonds_than_scratch_rows(port):
    """A 24x24 periodic lattice has 1152 bonds, so a Néel configuration has
    1153 connected rows: more rows than tokens (T = 288) and more than the
    1025-row per-warp scratch of the first k_connected (sized since as
    max(T, n_bonds + 1)). fp32 engine against the oracle, strict contract."""
    L = 24
    cfg = P.ModelConfig(n_sites=L * L, group_size=2, d_hidden=32, n_heads=4, n_blocks=1,
                        trailing_half_block=False, vq_codebook=64, vq_init_scale=1.0 / 32)
    model = P.VqTransformer.init(cfg, 0)
    lat = P.build_lattice("grid2d", (L, L), periodic=True)
    eng = P.LocalEnergyEngine(model, P.HamiltonianModel(lat), precision="fp32")
    port.set_bf16(False)
    om = port.model(cfg, 0)
    oh = port.hamiltonian("grid_periodic", L, L)
    x, y = np.meshgrid(np.arange(L), np.arange(L), indexing="xy")
    neel = ((x + y) % 2).reshape(-1).astype(np.uint8)
    S = np.stack([neel, 1 - neel, P.zero_sz_samples(L * L, 0, 1, 7)[0]])
    ref_e, _, ref_lpsi, _ = om.local_energies(oh, S, workers=os.cpu_count() or 8)
    e, lpsi = eng.local_energies(S, None)
    K, U, codes, lps = eng.taps(S)
    assert int(K[0]) == len(lat.bonds) + 1 == 1153
    rep = ParityReport()
    for i in range(len(S)):
        compare(rep, om.taps(oh, S[i]), ref_e[i], ref_lpsi[i], codes[i], U[i], e[i].real,
                lpsi[i], lps[i], cfg.seq_len)
    print(f"\n[24x24 Néel] {rep.summary()}")
    assert rep.ok(), rep.summary() + "\n" + "\n".join(rep.notes[:10])

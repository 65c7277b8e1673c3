"""The no-reuse regime (dense_local_energy, proj/src/bench.cpp:19-36) on the
GPU: every connected configuration's full T-token forward, no shared prefix,
no unique-row merging. It must give the compressed path's outputs (the
reference's own KAT: dense == dedup to 1e-9 in double, proj/tests), and its
unique-row counts must be the dense ones (U_b = K*T at every layer).

fp32 configs are compared at the strict tolerances; bf16 configs at the bf16
accumulation tolerances of test_gpu_parity.py (the two regimes partition the
attention work differently, so fp32 accumulation order differs)."""
import numpy as np
import pytest

import paper_2212_11296_b200 as P

pytestmark = pytest.mark.gpu


def _engine(name, precision=None):
    w = P.workload(name)
    precision = precision or w.precision
    model = P.VqTransformer.init(w.model, w.weight_seed, snap_bf16=precision == "bf16")
    lat = P.build_lattice("grid2d", (w.L, w.L), periodic=True)
    return w, P.LocalEnergyEngine(model, P.HamiltonianModel(lat), precision=precision)


@pytest.mark.parametrize("name,n,ltol,etol", [
    ("c1_4x4", 64, 1e-6, 1e-6),
    ("c2_6x6", 32, 1e-5, 1e-5),
    ("c3_10x10", 16, 5e-3, 2e-3),
])
def test_dense_equals_compressed(name, n, ltol, etol):
    w, eng = _engine(name)
    S = P.zero_sz_samples(w.n_sites, 0, n, w.sample_seed)
    led_c = P.Ledger()
    e_c, l_c = eng.local_energies(S, led_c)
    eng.set_reuse(False)
    led_d = P.Ledger()
    e_d, l_d = eng.local_energies(S, led_d)
    K, U, _, _ = eng.taps(S)
    eng.set_reuse(True)
    e_c2, l_c2 = eng.local_energies(S, None)
    # the switch is stateless: the compressed path reproduces itself bit for bit
    assert np.array_equal(e_c, e_c2) and np.array_equal(l_c, l_c2)
    assert np.max(np.abs(l_d - l_c)) < ltol
    assert np.max(np.abs(e_d - e_c) / np.maximum(1.0, np.abs(e_c))) < etol
    # dense regime: every location is its own unique row at every layer
    T = w.model.seq_len
    assert np.array_equal(U, np.repeat((K.astype(np.int64) * T)[:, None], U.shape[1], axis=1))
    # and its ledger is the dense one (the reference's total_dense)
    assert led_d.total_dedup() == led_d.total_dense()
    assert led_c.total_dense() == led_d.total_dense()


@pytest.mark.parametrize("name,n", [("c1_4x4", 16), ("c2_6x6", 8)])
def test_dense_matches_oracle_dense_log_prob(port, name, n):
    """The GPU's no-reuse regime row by row against the oracle's own dense
    forward (dense_log_prob, proj/src/model.cpp:398-426): every connected
    configuration's log P within 2e-5 and E_loc within 1e-4 relative of the
    oracle's local energies. The oracle's VQ codes are forced at every
    location (LocalEnergyEngine.set_code_override), so flagged near-ties
    cannot make a row incomparable."""
    from parity import override_codes

    w, eng = _engine(name, "fp32")
    lat = P.build_lattice("grid2d", (w.L, w.L), periodic=True)
    port.set_bf16(False)
    om = port.model(w.model, w.weight_seed)
    oh = port.hamiltonian("grid_periodic", w.L, w.L)
    S = P.zero_sz_samples(w.n_sites, 0, n, w.sample_seed)
    taps = [om.taps(oh, s) for s in S]
    m = w.model
    eng.set_reuse(False)
    eng.set_code_override(override_codes(None, taps, m.n_layers, lat.bonds.shape[0] + 1,
                                         m.seq_len))
    try:
        e, lpsi = eng.local_energies(S)
        K, U, _, lps = eng.taps(S)
    finally:
        eng.set_code_override(None)
        eng.set_reuse(True)
    ref_e, _, ref_lpsi, _ = om.local_energies(oh, S, workers=4)
    for i, s in enumerate(S):
        cf, _ = oh.connected_set(s)
        ref_rows = om.dense_log_prob(cf)  # the reference's dense forward per configuration
        assert int(K[i]) == cf.shape[0]
        assert np.max(np.abs(np.asarray(lps[i]) - ref_rows)) < 2e-5
        assert abs(lpsi[i] - 0.5 * ref_rows[0]) < 1e-5
    assert np.max(np.abs(e.real - ref_e) / np.maximum(np.abs(ref_e), 1e-12)) < 1e-4

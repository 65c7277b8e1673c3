"""CPU: the oracle's C restatement (oracle/_port) pinned to the reference.

1. Golden fixtures (tests/golden/*.npz, generated from the reference's own
   sources by tests/golden/make_golden.py) must be reproduced BIT FOR BIT:
   E_loc, logpsi, the FLOP ledger, per-layer unique counts, VQ codes, top-2
   gaps and per-row log-probs — double arithmetic and bf16 emulation alike.
2. Where oracle/_ref is built (it travels with the repo), fresh seeded cases
   are compared live, again bit for bit.
3. The reference's own known-answer tests for this path, restated
   (proj/tests/test_dedup.cpp, test_hamiltonian.cpp, test_model.cpp).
"""
import glob
import itertools
import math
import os

import numpy as np
import pytest

from paper_2212_11296_b200.config import ModelConfig, workload

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(p for p in glob.glob(os.path.join(HERE, "golden", "golden_*.npz"))
                if not p.endswith("golden_sample.npz"))
SAMPLE_GOLDEN = os.path.join(HERE, "golden", "golden_sample.npz")
LATTICE_NAMES = {0: "chain", 1: "grid", 2: "grid_periodic", 3: "chain_periodic"}


def cfg_from(g):
    c = g["cfg"]
    return ModelConfig(n_sites=int(c[0]), group_size=int(c[1]), d_hidden=int(c[2]),
                       n_heads=int(c[3]), n_blocks=int(c[4]), trailing_half_block=bool(c[5]),
                       vq_enabled=bool(c[6]), vq_heads=int(c[7]), vq_codebook=int(c[8]),
                       vq_init_scale=float(g["vq_init_scale"]))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_port_reproduces_reference_golden_bitwise(port, path):
    g = np.load(path)
    cfg = cfg_from(g)
    bf = bool(g["bf16"])
    port.set_bf16(bf)
    m = port.model(cfg, 0, snap_bf16=bf)
    lat = g["lattice"]
    h = port.hamiltonian(LATTICE_NAMES[int(lat[0])], int(lat[1]), int(lat[2]))
    assert np.array_equal(h.bonds(), g["bonds"])
    S = g["samples"]
    assert np.array_equal(port.zero_sz_samples(cfg.n_sites, 0, S.shape[0], 1), S)
    params = m.params()
    assert np.array_equal(np.array([p.sum() for _, p in params]), g["param_checksums"])
    e_re, e_im, lpsi, led = m.local_energies(h, S, workers=4)
    assert np.array_equal(e_re, g["e_re"])
    assert np.array_equal(lpsi, g["logpsi"])
    assert np.array_equal(led, g["ledger"])
    i = 0
    while f"taps{i}_U" in g:
        t = m.taps(h, S[i])
        assert np.array_equal(t.U, g[f"taps{i}_U"])
        assert np.array_equal(t.codes, g[f"taps{i}_codes"])
        assert np.array_equal(t.gaps, g[f"taps{i}_gaps"])
        assert np.array_equal(t.lp, g[f"taps{i}_lp"])
        i += 1
    assert i > 0


@pytest.mark.parametrize("case", ["c1_fp64", "c1_bf16", "small_open4x4"])
def test_port_sampler_reproduces_reference_golden_bitwise(port, case):
    """VqTransformer::sample (proj/src/model.cpp:485-525): the C restatement
    draws the reference's configurations and log-probs bit for bit."""
    g = np.load(SAMPLE_GOLDEN)
    if case.startswith("c1"):
        cfg, bf = workload("c1").model, case.endswith("bf16")
    else:
        cfg, bf = ModelConfig(n_sites=16, group_size=2, d_hidden=16, n_heads=2, n_blocks=1,
                              trailing_half_block=True, vq_heads=2, vq_codebook=8), False
    port.set_bf16(bf)
    m = port.model(cfg, 0, snap_bf16=bf)
    configs, lp = m.sample(g[f"{case}_configs"].shape[0], int(g[f"{case}_seed"]))
    assert np.array_equal(configs, g[f"{case}_configs"])
    assert np.array_equal(lp, g[f"{case}_log_probs"])


def test_port_sampler_matches_live_reference(ref, port):
    w = workload("c2")
    for bf in (False, True):
        ref.set_bf16(bf)
        port.set_bf16(bf)
        a = ref.model(w.model, 5, snap_bf16=bf).sample(4, 21)
        b = port.model(w.model, 5, snap_bf16=bf).sample(4, 21)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("seed,lat,n,bf", [(3, ("grid_periodic", 4, 4), 16, False),
                                           (11, ("grid", 3, 4), 12, False),
                                           (5, ("grid_periodic", 6, 6), 36, True)])
def test_port_matches_live_reference(ref, port, seed, lat, n, bf):
    cfg = ModelConfig(n_sites=n, group_size=2, d_hidden=32, n_heads=4, n_blocks=2,
                      trailing_half_block=seed == 11, vq_heads=1 + (seed == 11),
                      vq_codebook=32, vq_init_scale=1 / 32)
    for lib in (ref, port):
        lib.set_bf16(bf)
    mr, mp = ref.model(cfg, seed, bf), port.model(cfg, seed, bf)
    hr, hp = ref.hamiltonian(*lat), port.hamiltonian(*lat)
    S = ref.zero_sz_samples(n, 7, 6, seed)
    a, b = mr.local_energies(hr, S, workers=2), mp.local_energies(hp, S, workers=3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    for i in range(2):
        cf, co = hr.connected_set(S[i])
        cf2, co2 = hp.connected_set(S[i])
        assert np.array_equal(cf, cf2) and np.array_equal(co, co2)
        assert np.array_equal(mr.dense_log_prob(cf), mp.dense_log_prob(cf))
        assert np.array_equal(mr.dedup_log_prob(cf, S[i]), mp.dedup_log_prob(cf, S[i]))


# ---- restated reference known-answer tests ---------------------------------

def small_cfg(n, g=2):
    """proj/tests/test_dedup.cpp:13-23"""
    return ModelConfig(n_sites=n, group_size=g, d_hidden=16, n_heads=2, n_blocks=1,
                       vq_heads=2, vq_codebook=8)


def test_single_flip_unique_count_bound(port):
    """test_dedup.cpp:93-115: single-flip set, g=1, N=16 -> U0 = 2N - 1 = 31,
    and U0 <= (K-1) + T. The TFIM connected set IS the single-flip set."""
    cfg = small_cfg(16, g=1)
    m = port.model(cfg, 3)
    h = port.hamiltonian("chain", 16, 0, kind="tfim", Gamma=1.0)
    rng = np.random.default_rng(3)
    for _ in range(4):
        s = rng.integers(0, 2, 16).astype(np.uint8)
        t = m.taps(h, s)
        assert t.K == 17
        assert t.U[0] == 31
        assert t.U[0] <= (t.K - 1) + 16
    cfg2 = small_cfg(16, g=2)
    m2 = port.model(cfg2, 4)
    t2 = m2.taps(h, s)
    assert t2.U[0] <= (t2.K - 1) + 8


def test_two_site_difference_bound_rejected(port):
    """test_dedup.cpp:117-124: rows differing from base in > 2 sites -> UsageError."""
    from oracle import OracleError
    m = port.model(small_cfg(6), 5)
    base = np.zeros(6, np.uint8)
    bad = np.array([1, 1, 1, 0, 0, 0], np.uint8)
    with pytest.raises(OracleError) as ei:
        m.dedup_log_prob(np.stack([base, bad]), base)
    assert ei.value.kind == "UsageError"


def test_dense_equals_dedup_random_models(port):
    """test_dedup.cpp:320-349: compressed == dense log-probs within 1e-9,
    random models on a 4x4 Heisenberg lattice and a 16-chain TFIM."""
    heis = port.hamiltonian("grid", 4, 4)
    tfim = port.hamiltonian("chain", 16, 0, kind="tfim")
    rng = np.random.default_rng(1000)
    for draw in range(8):
        cfg = ModelConfig(n_sites=16, group_size=2, d_hidden=24 if draw % 3 == 0 else 16,
                          n_heads=2, n_blocks=1, vq_heads=2,
                          vq_codebook=8 if draw % 2 == 0 else 16)
        m = port.model(cfg, 1000 + draw)
        for h in (heis, tfim):
            s = rng.integers(0, 2, 16).astype(np.uint8)
            cf, _ = h.connected_set(s)
            np.testing.assert_allclose(m.dedup_log_prob(cf, s), m.dense_log_prob(cf),
                                       atol=1e-9, rtol=0)


def test_diagonal_only_local_energy(port):
    """test_dedup.cpp:433-447: Gamma = 0 -> E_loc equals the diagonal coefficient."""
    h = port.hamiltonian("chain", 6, 0, kind="tfim", J=1.3, Gamma=0.0)
    m = port.model(small_cfg(6), 13)
    s = np.array([[1, 1, 0, 1, 0, 0]], np.uint8)
    e, e_im, _, _ = m.local_energies(h, s)
    _, co = h.connected_set(s[0])
    assert abs(e[0] - co[0]) <= 1e-14 * abs(co[0])
    assert e_im[0] == 0.0


def test_uniform_wavefunction_local_energy(port):
    """test_dedup.cpp:449-464: all-zero weights -> log P({1,1}) = log 1/4 and
    E_loc = -3 for the 2-site TFIM chain."""
    m = port.model(small_cfg(2), 14)
    for i, (_, p) in enumerate(m.params()):
        m.set_param(i, np.zeros_like(p))
    lp = m.dense_log_prob(np.array([[1, 1]], np.uint8))
    assert abs(lp[0] - math.log(0.25)) < 1e-12
    h = port.hamiltonian("chain", 2, 0, kind="tfim")
    e, e_im, _, led = m.local_energies(h, np.array([[1, 1]], np.uint8))
    assert abs(e[0] + 3.0) < 1e-12
    assert e_im[0] == 0.0
    total_dense = led[0] + led[2] + led[3] + led[4]
    total_dedup = led[1] + led[2] + led[3] + led[4]
    assert total_dedup > 0 and total_dense >= total_dedup


def test_dedup_local_energy_equals_dense(port):
    """test_dedup.cpp:466-498: Heisenberg 2x3, dedup E_loc == dense E_loc (1e-9)."""
    h = port.hamiltonian("grid", 2, 3)
    m = port.model(small_cfg(6), 15)
    rng = np.random.default_rng(15)
    S = rng.integers(0, 2, (8, 6)).astype(np.uint8)
    e, _, _, _ = m.local_energies(h, S)
    for i in range(8):
        cf, co = h.connected_set(S[i])
        lp = m.dense_log_prob(cf)
        want = float(np.sum(co * np.exp(0.5 * (lp - lp[0]))))
        assert abs(e[i] - want) <= 1e-9 * max(1.0, abs(want))


def test_heisenberg_connected_set_coefficients(port):
    """test_hamiltonian.cpp:132-170: diagonal 1/4 sum z z, off-diagonals -1/2
    (Marshall) in bond order, entry count = 1 + #antiparallel bonds — on the
    periodic lattices the BASELINE configs use."""
    rng = np.random.default_rng(7)
    for L in (3, 4, 6):
        h = port.hamiltonian("grid_periodic", L, L)
        bonds = h.bonds()
        assert bonds.shape[0] == 2 * L * L
        for _ in range(5):
            s = rng.integers(0, 2, L * L).astype(np.uint8)
            cf, co = h.connected_set(s)
            z = 2 * s.astype(int) - 1
            anti = [b for b in range(len(bonds)) if s[bonds[b, 0]] != s[bonds[b, 1]]]
            assert cf.shape[0] == 1 + len(anti)
            assert co[0] == 0.25 * sum(z[i] * z[j] for i, j in bonds)
            assert np.all(co[1:] == -0.5)
            for r, b in enumerate(anti, start=1):
                f = s.copy()
                f[bonds[b]] ^= 1
                assert np.array_equal(cf[r], f)


def test_periodic_heisenberg_matches_kronecker_oracle(port):
    """Generalises test_hamiltonian.cpp:52-73,184-220 to a periodic 3x3
    lattice: the matrix assembled from connected sets equals the Kronecker
    construction sum_bonds 1/4 (sz sz) - 1/2 (s+ s- + s- s+) (Marshall-rotated),
    and every off-diagonal element is <= 0."""
    L = 3
    n = L * L
    h = port.hamiltonian("grid_periodic", L, L)
    dim = 1 << n
    H = np.zeros((dim, dim))
    for idx in range(dim):
        s = np.array([(idx >> i) & 1 for i in range(n)], np.uint8)
        cf, co = h.connected_set(s)
        for row, c in zip(cf, co):
            j = int(sum(int(v) << i for i, v in enumerate(row)))
            H[idx, j] += c
    sz = np.diag([-0.5, 0.5])
    sp = np.array([[0, 0], [1, 0.]])  # |1><0|: raises down(0) -> up(1)
    sm = sp.T

    def op(single, site):
        out = np.array([[1.0]])
        for i in reversed(range(n)):
            out = np.kron(out, single if i == site else np.eye(2))
        return out
    K = np.zeros((dim, dim))
    for i, j in h.bonds():
        K += op(sz, i) @ op(sz, j) - 0.5 * (op(sp, i) @ op(sm, j) + op(sm, i) @ op(sp, j))
    assert np.allclose(H, K, atol=1e-12)
    off = H - np.diag(np.diag(H))
    assert np.all(off <= 0)


def test_normalisation_by_enumeration(port):
    """test_model.cpp:92-103: sum_s exp(log P(s)) = 1 within 1e-9."""
    cfg = ModelConfig(n_sites=8, group_size=2, d_hidden=16, n_heads=2, n_blocks=2,
                      vq_codebook=8, trailing_half_block=False, vq_init_scale=0.3)
    m = port.model(cfg, 21)
    allc = np.array(list(itertools.product([0, 1], repeat=8)), np.uint8)
    lp = m.dense_log_prob(allc)
    assert abs(np.exp(lp).sum() - 1.0) < 1e-9


def test_zero_sz_sampler_contract(port):
    """SURVEY §8d sampler: N/2 up spins, deterministic per (seed, index)."""
    S = port.zero_sz_samples(16, 0, 64, 1)
    assert np.all(S.sum(1) == 8)
    assert np.array_equal(port.zero_sz_samples(16, 10, 5, 1), S[10:15])
    assert len({bytes(r) for r in S}) > 50


def test_bf16_emulation_rounds_products(port):
    """bf16 emulation changes results, and snapping weights is idempotent."""
    w = workload("c1")
    port.set_bf16(False)
    m = port.model(w.model, 0, snap_bf16=True)
    h = port.hamiltonian("grid_periodic", 4, 4)
    S = port.zero_sz_samples(16, 0, 4, 1)
    a = m.local_energies(h, S)[0]
    port.set_bf16(True)
    b = m.local_energies(h, S)[0]
    port.set_bf16(False)
    assert not np.array_equal(a, b)
    assert np.allclose(a, b, rtol=1e-2)
    for _, p in m.params():
        f = p.astype(np.float32)
        assert np.array_equal(f.view(np.uint32) & 0xFFFF, np.zeros_like(f.view(np.uint32)))

"""CPU: host-side logic of the product library and the C ABI surface
(no GPU needed). The product must reproduce the reference's seeded model,
lattices and ledger exactly, and the C-ABI library must load and export every
symbol include/*.h declares."""
import ctypes as C
import glob
import os
import re

import numpy as np
import pytest

import paper_2212_11296_b200 as P
from paper_2212_11296_b200 import _native
from paper_2212_11296_b200.config import ConfigError, ModelConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        for m in re.finditer(r"\b(vqnqs_\w+)\s*\(", txt):
            names.add(m.group(1))
    return names


def test_abi_exports_every_declared_symbol():
    lib = C.CDLL(_native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in sorted(syms):
        assert hasattr(lib, s), s
    # and the Python binding declares signatures for every public one
    public = {s for s in syms if not s.startswith("vqnqs_debug")}
    assert public <= set(_native.SIGNATURES), public - set(_native.SIGNATURES)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_init_params_equal_reference(port, name):
    w = P.workload(name)
    for snap in (False, True):
        mine = P.VqTransformer.init(w.model, w.weight_seed, snap_bf16=snap)
        theirs = port.model(w.model, w.weight_seed, snap_bf16=snap).params()
        assert [p.name for p in mine.params] == [n for n, _ in theirs]
        for p, (_, v) in zip(mine.params, theirs):
            assert np.array_equal(p.value.reshape(-1), v)


def test_init_params_match_reference_golden():
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_c1_fp64.npz"))
    m = P.VqTransformer.init(P.workload("c1").model, 0)
    assert np.array_equal(np.array([p.value.sum() for p in m.params]), g["param_checksums"])


def test_lattices_and_sampler_equal_reference(port):
    for L in (4, 6, 10, 12, 16):
        lat = P.build_lattice("grid2d", (L, L), periodic=True)
        assert np.array_equal(lat.bonds, port.hamiltonian("grid_periodic", L, L).bonds())
        assert np.array_equal(P.zero_sz_samples(L * L, 3, 9),
                              port.zero_sz_samples(L * L, 3, 9, 1))
    assert np.array_equal(P.build_lattice("grid2d", (3, 5)).bonds,
                          port.hamiltonian("grid", 3, 5).bonds())
    assert np.array_equal(P.build_lattice("chain1d", (7,)).bonds,
                          port.hamiltonian("chain", 7, 0).bonds())
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_c1_fp64.npz"))
    assert np.array_equal(P.build_lattice("grid2d", (4, 4), True).bonds, g["bonds"])
    assert np.array_equal(P.zero_sz_samples(16, 0, 64), g["samples"])


def test_lattice_errors():
    with pytest.raises(ConfigError):
        P.build_lattice("grid2d", (2, 2), periodic=True)
    with pytest.raises(ConfigError):
        P.build_lattice("grid2d", (0, 3))
    with pytest.raises(ConfigError):
        P.build_lattice("ring", (3,))


@pytest.mark.parametrize("gold", ["c1_fp64", "c2_fp64", "small_open4x4", "small_chain6_g3"])
def test_host_ledger_equals_reference_ledger(port, gold):
    """The engine recomputes flops::Ledger host-side from K and the realised
    unique counts; summed over a batch it must equal the reference's own
    ledger exactly (integers)."""
    from test_oracle import LATTICE_NAMES, cfg_from
    g = np.load(os.path.join(ROOT, "tests", "golden", f"golden_{gold}.npz"))
    cfg = cfg_from(g)
    port.set_bf16(bool(g["bf16"]))
    m = port.model(cfg, 0, snap_bf16=bool(g["bf16"]))
    lat = g["lattice"]
    h = port.hamiltonian(LATTICE_NAMES[int(lat[0])], int(lat[1]), int(lat[2]))
    tot = P.Ledger()
    for s in g["samples"]:
        t = m.taps(h, s)
        tot += P.Ledger.from_counts(cfg, t.K, t.U)
    assert np.array_equal(tot.as_array(), g["ledger"])
    dense, dedup = tot.total_dense(), tot.total_dedup()
    assert dense > dedup > 0
    s_tot, s_q = tot.savings()
    assert s_tot > 1 and s_q > 1


def test_model_config_validation_messages():
    with pytest.raises(ConfigError, match="n_heads"):
        ModelConfig(d_hidden=10, n_heads=3).validate()
    with pytest.raises(ConfigError, match="at least one block"):
        ModelConfig(n_blocks=0, trailing_half_block=False).validate()
    with pytest.raises(ConfigError, match="vq_heads"):
        ModelConfig(d_hidden=8, n_heads=2, vq_heads=3).validate()


def test_workloads_record_survey_decisions():
    for name, w in P.WORKLOADS.items():
        r = w.record()
        assert r["n_bonds"] == 2 * w.L * w.L
        assert w.model.group_size == 2 and not w.model.trailing_half_block
        assert w.model.vq_heads == 1
        assert abs(w.model.vq_init_scale - 1.0 / w.model.d_hidden) < 1e-15
    assert P.n_params(P.workload("c5").model) > 80_000_000 if hasattr(P, "n_params") else True


def test_engine_creation_fails_loudly_without_gpu():
    """No CPU fallback: without a usable CUDA device the engine refuses."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    w = P.workload("c1")
    m = P.VqTransformer.init(w.model, 0)
    with pytest.raises(P.VqnqsError):
        P.LocalEnergyEngine(m, P.HamiltonianModel(P.build_lattice("grid2d", (4, 4), True)),
                            precision="fp32")


def test_engine_rejects_unsupported_capabilities():
    torch = pytest.importorskip("torch")
    w = P.workload("c1")
    m = P.VqTransformer.init(w.model, 0)
    with pytest.raises(P.CapabilityError):
        P.LocalEnergyEngine(m, P.HamiltonianModel(P.build_lattice("grid2d", (4, 4), True),
                                                  kind="tfim"))


def test_fill_stats_matches_reference_formula():
    e = np.array([-1.0, -2.0, -4.0, -3.5]) + 0j
    est = P.fill_stats(e)
    assert est.energy == pytest.approx(-2.625)
    assert est.variance == pytest.approx(np.var(e.real, ddof=1))
    assert est.std_err == pytest.approx(np.sqrt(np.var(e.real, ddof=1) / 4))

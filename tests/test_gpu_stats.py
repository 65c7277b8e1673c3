"""estimate_energy / fill_stats behind the C ABI (vqnqs_gpu_estimate_energy):
fp64 device reduction plus the NCCL allreduce (proj/src/trainer.cpp:184-211).
One GPU per box here, so the NCCL path runs as a one-rank communicator; the
multi-rank logic is covered by the gloo world-2 tests (tests/test_distributed.py)."""
import numpy as np
import pytest

import paper_2212_11296_b200 as P

pytestmark = pytest.mark.gpu


def _engine(name="c2", precision="fp32"):
    w = P.workload(name)
    model = P.VqTransformer.init(w.model, w.weight_seed, snap_bf16=precision == "bf16")
    lat = P.build_lattice("grid2d", (w.L, w.L), periodic=True)
    return w, lat, P.LocalEnergyEngine(model, P.HamiltonianModel(lat), precision=precision)


@pytest.mark.parametrize("name,precision", [("c2", "fp32"), ("c3", "bf16")])
def test_estimate_energy_matches_fill_stats(name, precision):
    w, lat, eng = _engine(name, precision)
    S = P.zero_sz_samples(w.n_sites, 0, 300, w.sample_seed)
    led_a = P.Ledger()
    e, lpsi = eng.local_energies(S, led_a)
    ref = P.fill_stats(e)
    led_b = P.Ledger()
    est = eng.estimate_energy(S, ledger=led_b)
    assert np.array_equal(est.local_energies.real, e.real)
    assert np.array_equal(est.logpsi, lpsi)
    assert est.k_total == 300
    assert est.energy == pytest.approx(ref.energy, rel=1e-13)
    assert est.variance == pytest.approx(ref.variance, rel=1e-12)
    assert est.std_err == pytest.approx(ref.std_err, rel=1e-12)
    assert np.array_equal(led_a.as_array(), led_b.as_array())


def test_estimate_energy_through_a_one_rank_nccl_communicator():
    from paper_2212_11296_b200.distributed import NcclComm
    w, lat, eng = _engine("c2", "fp32")
    S = P.zero_sz_samples(w.n_sites, 0, 257, w.sample_seed)
    alone = eng.estimate_energy(S)
    comm = NcclComm(rank=0, world=1, device=0)
    led = P.Ledger()
    est = eng.estimate_energy(S, comm=comm, ledger=led)
    comm.close()
    assert (est.energy, est.variance, est.std_err, est.k_total) == \
        (alone.energy, alone.variance, alone.std_err, alone.k_total)
    led_ref = P.Ledger()
    eng.local_energies(S, led_ref)
    assert np.array_equal(led.as_array(), led_ref.as_array())


def test_estimate_energy_balanced_shards_reassemble():
    """Shards dealt by vqnqs_balanced_shards, evaluated one after another on
    this GPU, give the batch's per-sample energies back exactly."""
    from paper_2212_11296_b200.distributed import balanced_shards
    w, lat, eng = _engine("c2", "fp32")
    S = P.zero_sz_samples(w.n_sites, 0, 200, w.sample_seed)
    e_all, _ = eng.local_energies(S)
    owner = balanced_shards(S, lat.bonds, 4)
    for r in range(4):
        mine = np.nonzero(owner == r)[0]
        est = eng.estimate_energy(S[mine])
        assert np.array_equal(est.local_energies.real, e_all.real[mine])


def test_fill_stats_device_matches_host_estimate():
    import torch
    w, lat, eng = _engine("c2", "fp32")
    S = P.zero_sz_samples(w.n_sites, 0, 129, w.sample_seed)
    d_cfg = torch.from_numpy(S).cuda()
    d_e = torch.empty(129, dtype=torch.float64, device="cuda")
    d_l = torch.empty_like(d_e)
    eng.local_energies_device(d_cfg, d_e, d_l)
    dev = eng.fill_stats_device(d_e)
    host = eng.estimate_energy(S)
    assert (dev.energy, dev.variance, dev.std_err, dev.k_total) == \
        (host.energy, host.variance, host.std_err, host.k_total)

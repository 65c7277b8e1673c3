"""CPU multi-process (gloo, world_size 2): sample sharding and the fill_stats
allreduce give exactly the single-process statistics, and per-sample outputs
do not depend on the sharding. Local energies come from the oracle port (CPU
test infrastructure); the code under test is the product's sharding and
collective logic (paper_2212_11296_b200/distributed.py)."""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2212_11296_b200.distributed import allreduce_stats, shard_bounds  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import PortLib
    from paper_2212_11296_b200.config import workload
    w = workload("c1")
    port_lib = PortLib()
    m = port_lib.model(w.model, 0)
    h = port_lib.hamiltonian("grid_periodic", 4, 4)
    B = 37
    start, count = shard_bounds(B, rank, world)
    S = port_lib.zero_sz_samples(16, start, count, 1)
    e, _, lpsi, _ = m.local_energies(h, S)
    est = allreduce_stats(e.astype(complex))
    out[rank] = (start, count, e, lpsi, est.energy, est.variance, est.std_err)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_cover_exactly():
    for n, world in [(10, 3), (8192, 8), (5, 8), (0, 2)]:
        seen = []
        for r in range(world):
            s, c = shard_bounds(n, r, world)
            seen.extend(range(s, s + c))
        assert seen == list(range(n))


def test_gloo_world2_stats_equal_single_process(port):
    world = 2
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    from paper_2212_11296_b200.api import fill_stats
    from paper_2212_11296_b200.config import workload
    w = workload("c1")
    m = port.model(w.model, 0)
    h = port.hamiltonian("grid_periodic", 4, 4)
    S = port.zero_sz_samples(16, 0, 37, 1)
    e_all, _, l_all, _ = m.local_energies(h, S)
    ref = fill_stats(e_all.astype(complex))
    got = [out[r] for r in range(world)]
    for start, count, e, lpsi, *_ in got:
        assert np.array_equal(e, e_all[start:start + count])  # sharding-invariant
        assert np.array_equal(lpsi, l_all[start:start + count])
    for *_, energy, var, se in got:
        assert energy == pytest.approx(ref.energy, rel=1e-13)
        assert var == pytest.approx(ref.variance, rel=1e-12)
        assert se == pytest.approx(ref.std_err, rel=1e-12)


def _bal_worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import PortLib
    import paper_2212_11296_b200 as P
    from paper_2212_11296_b200.distributed import balanced_shards
    w = P.workload("c1")
    lat = P.build_lattice("grid2d", (4, 4), periodic=True)
    S = P.zero_sz_samples(16, 0, 41, 1)
    owner = balanced_shards(S, lat.bonds, world)  # every rank computes the same plan
    mine = np.nonzero(owner == rank)[0]
    port_lib = PortLib()
    m = port_lib.model(w.model, 0)
    h = port_lib.hamiltonian("grid_periodic", 4, 4)
    e, _, _, _ = m.local_energies(h, S[mine])
    est = allreduce_stats(e.astype(complex))
    out[rank] = (mine, e, owner, est.energy, est.variance)
    dist.barrier()
    dist.destroy_process_group()


def test_balanced_shards_cover_and_balance():
    import paper_2212_11296_b200 as P
    from paper_2212_11296_b200.distributed import balanced_shards
    lat = P.build_lattice("grid2d", (16, 16), periodic=True)
    S = P.zero_sz_samples(256, 0, 1000, 1)
    K = 1 + (S[:, lat.bonds[:, 0]] != S[:, lat.bonds[:, 1]]).sum(1)
    for world in (1, 2, 3, 8):
        owner = balanced_shards(S, lat.bonds, world)
        assert owner.min() == 0 and owner.max() == world - 1
        load = np.bincount(owner, weights=K, minlength=world)
        assert load.sum() == K.sum()
        assert load.max() - load.min() <= K.max()  # LPT bound
        assert np.array_equal(owner, balanced_shards(S, lat.bonds, world))  # deterministic
    # contiguous blocks are worse balanced than the K-balanced plan
    s, c = shard_bounds(1000, 0, 8)
    blocks = [K[shard_bounds(1000, r, 8)[0]:][:shard_bounds(1000, r, 8)[1]].sum()
              for r in range(8)]
    owner = balanced_shards(S, lat.bonds, 8)
    load = np.bincount(owner, weights=K, minlength=8)
    assert load.max() - load.min() <= max(blocks) - min(blocks)


def test_gloo_world2_balanced_shards_stats(port):
    world = 2
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_bal_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    from paper_2212_11296_b200.api import fill_stats
    from paper_2212_11296_b200.config import workload
    w = workload("c1")
    m = port.model(w.model, 0)
    h = port.hamiltonian("grid_periodic", 4, 4)
    S = port.zero_sz_samples(16, 0, 41, 1)
    e_all, _, _, _ = m.local_energies(h, S)
    ref = fill_stats(e_all.astype(complex))
    seen = np.concatenate([out[r][0] for r in range(world)])
    assert np.array_equal(np.sort(seen), np.arange(41))
    for r in range(world):
        mine, e, owner, energy, var = out[r]
        assert np.array_equal(e, e_all[mine])
        assert np.array_equal(owner, out[0][2])
        assert energy == pytest.approx(ref.energy, rel=1e-13)
        assert var == pytest.approx(ref.variance, rel=1e-12)

"""Sample sharding across GPUs and the fill_stats collective.

The local-energy path shards naturally by sample (every sample's connected
set, dedup, attention and E_loc are independent: proj/src/dedup.cpp:394-420,
SPEC.md:422), so one process per GPU evaluates its own block of samples with
no data-path communication. The only collective reproduces fill_stats
(proj/src/trainer.cpp:184-198): the energy mean, the unbiased variance of
Re E_loc and its standard error over the whole batch, as two small fp64
allreduces (sum; then the centred sum of squares, the same two-pass formula
as the reference) over NCCL on GPUs or gloo on CPU.
"""
from __future__ import annotations

import math
from typing import Optional, Tuple

import numpy as np

from .api import VmcEstimate


def shard_bounds(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block of samples for `rank`: (start, count); the first
    n_total % world ranks get one extra sample."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def allreduce_stats(e_local, device=None, group=None) -> VmcEstimate:
    """fill_stats over all ranks' local energies (complex numpy array or a
    torch float64 tensor of real parts)."""
    import torch
    import torch.distributed as dist
    if isinstance(e_local, torch.Tensor):
        re = e_local.to(torch.float64)
        dev = re.device
        im_sum = torch.zeros((), dtype=torch.float64, device=dev)
    else:
        arr = np.asarray(e_local)
        dev = device if device is not None else "cpu"
        re = torch.as_tensor(np.ascontiguousarray(arr.real), dtype=torch.float64, device=dev)
        im_sum = torch.as_tensor(float(np.sum(arr.imag)), dtype=torch.float64, device=dev)
    n = torch.tensor(float(re.numel()), dtype=torch.float64, device=dev)
    v = torch.stack([n, re.sum(), im_sum])
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(v, group=group)
    n_tot = float(v[0].item())
    mean = float(v[1].item()) / n_tot
    c = ((re - mean) ** 2).sum().reshape(1)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(c, group=group)
    k = int(round(n_tot))
    var = float(c.item()) / (k - 1) if k > 1 else 0.0
    return VmcEstimate(mean, var, math.sqrt(var / k) if k else 0.0,
                       np.zeros(0, complex))


def balanced_shards(configs, bonds, world: int) -> np.ndarray:
    """owner[i] = rank of sample i, balancing the connected-set sizes
    K = 1 + #antiparallel bonds across ranks; the native
    vqnqs_balanced_shards, deterministic on every rank."""
    import ctypes as C
    from . import _native as N
    cfgs = np.ascontiguousarray(configs, np.uint8)
    b = np.ascontiguousarray(bonds, np.int32)
    owner = np.zeros(cfgs.shape[0], np.int32)
    N.check(N.lib().vqnqs_balanced_shards(N.ptr(cfgs, C.c_uint8), cfgs.shape[0], cfgs.shape[1],
                                          N.ptr(b, C.c_int32), b.shape[0], int(world),
                                          N.ptr(owner, C.c_int32)))
    return owner


class NcclComm:
    """The native NCCL communicator (vqnqs_comm_*) of one rank: rank 0's
    unique id is shared over torch.distributed (any backend), then each rank
    joins with the CUDA device of its engine. Used by
    LocalEnergyEngine.estimate_energy for the fill_stats allreduce."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        import ctypes as C
        import torch.distributed as dist
        from . import _native as N
        buf = C.create_string_buffer(128)
        if rank == 0:
            N.check(N.lib().vqnqs_comm_unique_id(buf))
        ids = [buf.raw]
        if world > 1:
            dist.broadcast_object_list(ids, src=0, group=group)
        h = C.c_void_p()
        N.check(N.lib().vqnqs_comm_create(ids[0], world, rank, device, C.byref(h)))
        self.handle = h
        self.rank, self.world, self.device = rank, world, device

    def close(self):
        from . import _native as N
        if getattr(self, "handle", None):
            N.lib().vqnqs_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def local_energies_sharded(engine, batch_global, rank: int, world: int,
                           group=None, device=None):
    """Evaluate this rank's shard of a global batch on `engine` (a
    LocalEnergyEngine on this rank's GPU) and return (E_loc shard, logpsi
    shard, global VmcEstimate)."""
    start, count = shard_bounds(len(batch_global), rank, world)
    e, lpsi = engine.local_energies(np.asarray(batch_global)[start:start + count])
    est = allreduce_stats(e, device=device, group=group)
    return e, lpsi, est

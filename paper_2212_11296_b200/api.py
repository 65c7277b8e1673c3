"""Python mirror of the reference's local-energy interface.

Names, argument meaning and error behaviour follow the reference:

* ``VqTransformer.init(cfg, seed)`` / ``.parameters()`` — proj/src/model.cpp:150-229
* ``build_lattice`` / ``HamiltonianModel`` — proj/include/vqnqs/hamiltonian.hpp:17-37
* ``Ledger`` — proj/include/vqnqs/flops.hpp:12-44
* ``local_energies(model, h, batch, ledger=None)`` — proj/include/vqnqs/trainer.hpp:76-79
* ``local_energy_batch(model, h, s)`` — proj/include/vqnqs/dedup.hpp:84-93
* ``dedup_log_prob(model, configs, base)`` — proj/include/vqnqs/dedup.hpp:77-79 (for a
  connected set generated from ``base``)
* ``fill_stats`` / ``VmcEstimate`` — proj/src/trainer.cpp:184-198

Everything numeric runs in the native library (include/vqnqs_b200.h) on a
B200; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .config import (CapabilityError, ConfigError, ModelConfig, NumericError, ShapeError,
                     UsageError)

PRECISIONS = {"fp32": 0, "bf16": 1}


# ----------------------------------------------------------------- model


@dataclass
class Parameter:
    name: str
    value: np.ndarray  # float64, reference shape


@dataclass
class VqTransformer:
    cfg: ModelConfig
    params: List[Parameter]

    @staticmethod
    def init(cfg: ModelConfig, seed: int = 0, snap_bf16: bool = False) -> "VqTransformer":
        """VqTransformer::init(cfg, Rng(seed)) — same draws, same order."""
        cfg.validate()
        desc = N.desc_of(cfg)
        n = C.c_int(0)
        N.check(N.lib().vqnqs_param_layout(C.byref(desc), C.byref(n), None))
        numels = np.zeros(n.value, np.int64)
        N.check(N.lib().vqnqs_param_layout(C.byref(desc), None, N.ptr(numels, C.c_int64)))
        bufs = [np.zeros(int(k), np.float64) for k in numels]
        arr = (N.P_F64 * len(bufs))(*[N.ptr(b, C.c_double) for b in bufs])
        N.check(N.lib().vqnqs_init_params(C.byref(desc), seed, int(snap_bf16), arr))
        shapes = param_shapes(cfg)
        return VqTransformer(cfg, [Parameter(nm, b.reshape(sh))
                                   for (nm, sh), b in zip(shapes, bufs)])

    def parameters(self) -> List[Parameter]:
        return self.params

    def snap_bf16(self) -> "VqTransformer":
        out = []
        for p in self.params:
            v = p.value.astype(np.float32)
            u = v.view(np.uint32).astype(np.uint64)
            fin = (u & 0x7F800000) != 0x7F800000
            u = np.where(fin, (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000, u)
            out.append(Parameter(p.name, u.astype(np.uint32).view(np.float32).astype(np.float64)))
        return VqTransformer(self.cfg, out)


def param_shapes(cfg: ModelConfig) -> List[Tuple[str, Tuple[int, ...]]]:
    """parameters() order and shapes (proj/src/model.cpp:113-229)."""
    d, v, t = cfg.d_hidden, cfg.vocab, cfg.seq_len
    out = [("dec.tok_embed", (v + 1, d)), ("dec.pos_embed", (t, d))]
    nblk = cfg.n_blocks + int(cfg.trailing_half_block)
    for b in range(nblk):
        half = b == cfg.n_blocks
        p = "dec.half" if half else f"dec.block{b}"
        out += [(p + ".ln1_g", (d,)), (p + ".ln1_b", (d,))]
        for w in "qkvo":
            out += [(f"{p}.w{w}", (d, d)), (f"{p}.b{w}", (d,))]
        if not half and cfg.vq_enabled:
            out.append((p + ".codebook", (cfg.vq_heads * cfg.vq_codebook,
                                          d // cfg.vq_heads)))
        if not half:
            out += [(p + ".ln2_g", (d,)), (p + ".ln2_b", (d,)), (p + ".w1", (d, 4 * d)),
                    (p + ".b1", (4 * d,)), (p + ".w2", (4 * d, d)), (p + ".b2", (d,))]
    out += [("dec.lnf_g", (d,)), ("dec.lnf_b", (d,)), ("dec.head_w", (d, v)),
            ("dec.head_b", (v,))]
    return out


# ----------------------------------------------------------- hamiltonian


@dataclass
class Lattice:
    kind: str            # "chain1d" | "grid2d"
    dims: Tuple[int, ...]
    sites: int
    bonds: np.ndarray    # [nb, 2] int32, (i < j)
    periodic: bool = False


def build_lattice(kind: str, dims: Sequence[int], periodic: bool = False) -> Lattice:
    """build_lattice (proj/src/hamiltonian.cpp:5-35); periodic adds wrap
    bonds in the same horizontals-then-verticals row-major order."""
    if kind == "chain1d":
        if len(dims) != 1 or dims[0] <= 0:
            raise ConfigError("chain1d needs one positive dimension")
        lx, ly = dims[0], 0
    elif kind == "grid2d":
        if len(dims) != 2 or dims[0] <= 0 or dims[1] <= 0:
            raise ConfigError("grid2d needs two positive dimensions")
        lx, ly = dims
    else:
        raise ConfigError(f"unknown lattice kind {kind!r}")
    nb = N.lib().vqnqs_build_lattice(lx, ly, int(periodic), None, 0)
    if nb < 0:
        N.check(-nb)
    bonds = np.zeros((nb, 2), np.int32)
    N.lib().vqnqs_build_lattice(lx, ly, int(periodic), N.ptr(bonds, C.c_int32), nb)
    return Lattice(kind, tuple(dims), lx * max(ly, 1), bonds, periodic)


@dataclass
class HamiltonianModel:
    lattice: Lattice
    kind: str = "heisenberg"
    marshall: bool = True
    J: float = 1.0
    Gamma: float = 1.0

    def n_sites(self) -> int:
        return self.lattice.sites


def zero_sz_samples(n_sites: int, start: int, count: int, seed: int = 1) -> np.ndarray:
    """SURVEY §8d sampler: sample i <- Rng(seed).split(start + i), Fisher-Yates."""
    out = np.zeros((count, n_sites), np.uint8)
    N.check(N.lib().vqnqs_zero_sz_samples(n_sites, start, count, seed, N.ptr(out, C.c_uint8)))
    return out


# ---------------------------------------------------------------- ledger

LEDGER_FIELDS = ("per_location_dense", "per_location_unique", "attention", "vq_distance",
                 "other", "per_location_dense_quantized", "per_location_unique_quantized")


@dataclass
class Ledger:
    per_location_dense: int = 0
    per_location_unique: int = 0
    attention: int = 0
    vq_distance: int = 0
    other: int = 0
    per_location_dense_quantized: int = 0
    per_location_unique_quantized: int = 0

    @staticmethod
    def from_array(a) -> "Ledger":
        return Ledger(*[int(x) for x in a])

    def as_array(self) -> np.ndarray:
        return np.array([getattr(self, f) for f in LEDGER_FIELDS], np.int64)

    def total_dense(self) -> int:
        return self.per_location_dense + self.attention + self.vq_distance + self.other

    def total_dedup(self) -> int:
        return self.per_location_unique + self.attention + self.vq_distance + self.other

    def __iadd__(self, o: "Ledger") -> "Ledger":
        for f in LEDGER_FIELDS:
            setattr(self, f, getattr(self, f) + getattr(o, f))
        return self

    @staticmethod
    def from_counts(cfg: ModelConfig, K: int, U) -> "Ledger":
        """Ledger of one local_energy_batch from its connected-set size K and
        unique-row counts U[0..L] (the engine's host-side recomputation)."""
        u = np.ascontiguousarray(U, np.int64)
        out = np.zeros(7, np.int64)
        desc = N.desc_of(cfg)
        N.check(N.lib().vqnqs_ledger_from_counts(C.byref(desc), int(K), N.ptr(u, C.c_int64),
                                                 N.ptr(out, C.c_int64)))
        return Ledger.from_array(out)

    def savings(self) -> Tuple[float, float]:
        """(total, quantized-ops) savings, proj/src/bench.cpp:110-114."""
        tot = self.total_dense() / max(1, self.total_dedup())
        q = self.per_location_dense_quantized / max(1, self.per_location_unique_quantized)
        return tot, q


# ---------------------------------------------------------------- engine


class LocalEnergyEngine:
    """One model + Hamiltonian resident on one GPU (a native handle).

    Plays the role of the (const VqTransformer&, const HamiltonianModel&)
    pair the reference passes to local_energies. Not thread-safe."""

    def __init__(self, model: VqTransformer, ham: HamiltonianModel,
                 precision: str = "bf16", device: int = 0):
        if ham.kind != "heisenberg":
            raise CapabilityError("GPU path implements the Heisenberg connected set only")
        if ham.n_sites() != model.cfg.n_sites:
            raise ShapeError("configuration size != site count")
        self.cfg = model.cfg
        self.ham = ham
        self.precision = precision
        self.device = device
        desc = N.desc_of(model.cfg)
        vals = [np.ascontiguousarray(p.value, np.float64).reshape(-1) for p in model.params]
        arr = (N.P_F64 * len(vals))(*[N.ptr(v, C.c_double) for v in vals])
        h = C.c_void_p()
        N.check(N.lib().vqnqs_gpu_create(C.byref(desc), arr, len(vals), PRECISIONS[precision],
                                         device, C.byref(h)))
        self._h = h
        bonds = np.ascontiguousarray(ham.lattice.bonds, np.int32)
        N.check(N.lib().vqnqs_gpu_set_hamiltonian(self._h, N.ptr(bonds, C.c_int32),
                                                  bonds.shape[0], ham.n_sites(),
                                                  int(ham.marshall)))
        self.n_bonds = bonds.shape[0]

    def close(self):
        if getattr(self, "_h", None):
            N.lib().vqnqs_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # host buffers in, host buffers out (the reference-facing call)
    def local_energies(self, batch, ledger: Optional[Ledger] = None):
        """Returns (E_loc complex[B], logpsi float[B]); adds into ledger."""
        cfgs = np.ascontiguousarray(batch, np.uint8)
        if cfgs.ndim != 2 or cfgs.shape[1] != self.cfg.n_sites:
            raise ShapeError("configuration size != site count")
        B = cfgs.shape[0]
        e_re = np.zeros(B)
        e_im = np.zeros(B)
        lpsi = np.zeros(B)
        led = np.zeros(7, np.int64)
        N.check(N.lib().vqnqs_gpu_local_energies(self._h, N.ptr(cfgs, C.c_uint8), B,
                                                 N.ptr(e_re, C.c_double), N.ptr(e_im, C.c_double),
                                                 N.ptr(lpsi, C.c_double), N.ptr(led, C.c_int64)))
        if ledger is not None:
            ledger += Ledger.from_array(led)
        return e_re + 1j * e_im, lpsi

    # device buffers (torch tensors) in/out, on `stream` (torch stream or None)
    def local_energies_device(self, d_configs, d_e, d_logpsi, stream=None) -> Ledger:
        led = np.zeros(7, np.int64)
        st = C.c_void_p(stream.cuda_stream) if stream is not None else None
        N.check(N.lib().vqnqs_gpu_local_energies_device(
            self._h, C.c_void_p(d_configs.data_ptr()), d_configs.shape[0],
            C.c_void_p(d_e.data_ptr()), C.c_void_p(d_logpsi.data_ptr()),
            N.ptr(led, C.c_int64), st))
        return Ledger.from_array(led)

    def connected_log_probs(self, base) -> np.ndarray:
        base = np.ascontiguousarray(base, np.uint8)
        cap = self.n_bonds + 1
        lp = np.zeros(cap)
        K = N.lib().vqnqs_gpu_connected_log_probs(self._h, N.ptr(base, C.c_uint8),
                                                  N.ptr(lp, C.c_double), cap)
        if K < 0:
            N.check(-K)
        return lp[:K]

    def taps(self, batch):
        """Per-sample K, U[L+1], per-location codes [L, K*T, vq_heads] (-1 in
        blocks without VQ) and row log-probs."""
        cfgs = np.ascontiguousarray(batch, np.uint8)
        B = cfgs.shape[0]
        L = self.cfg.n_layers
        T = self.cfg.seq_len
        H = self.cfg.vq_heads
        cap = B * (self.n_bonds + 1) * T * L * H
        K = np.zeros(B, np.int32)
        U = np.zeros((B, L + 1), np.int64)
        codes = np.zeros(cap, np.int32)
        lpcap = B * (self.n_bonds + 1)
        lp = np.zeros(lpcap)
        N.check(N.lib().vqnqs_gpu_taps(self._h, N.ptr(cfgs, C.c_uint8), B, N.ptr(K, C.c_int32),
                                       N.ptr(U, C.c_int64), N.ptr(codes, C.c_int32), cap,
                                       N.ptr(lp, C.c_double), lpcap))
        out, lps, pos, lpos = [], [], 0, 0
        for s in range(B):
            n = L * int(K[s]) * T * H
            out.append(codes[pos:pos + n].reshape(L, int(K[s]) * T, H))
            lps.append(lp[lpos:lpos + int(K[s])])
            pos += n
            lpos += int(K[s])
        return K, U, out, lps

    def system_name(self) -> str:
        """system_name, proj/src/bench.cpp:46-55."""
        return f"{self.ham.kind} " + "x".join(str(x) for x in self.ham.lattice.dims)

    def sample(self, count: int, seed: int, skip: int = 0):
        """VqTransformer::sample(count, Rng(seed)) (proj/src/model.cpp:485-525)
        on the GPU: (configs [count x n_sites] uint8, log_probs [count]).
        skip = uniforms of the Rng(seed) stream already consumed by earlier
        batches (count x seq_len each)."""
        configs = np.zeros((count, self.cfg.n_sites), np.uint8)
        lp = np.zeros(count)
        N.check(N.lib().vqnqs_gpu_sample(self._h, int(count), int(seed), int(skip),
                                         N.ptr(configs, C.c_uint8), N.ptr(lp, C.c_double)))
        return configs, lp

    def set_reuse(self, reuse: bool) -> None:
        """reuse=False selects the reference's no-reuse regime
        (dense_local_energy, proj/src/bench.cpp:19-36): same outputs, every
        location computed."""
        N.check(N.lib().vqnqs_gpu_set_reuse(self._h, int(bool(reuse))))

    def estimate_energy(self, batch, comm=None, ledger: Optional[Ledger] = None):
        """fill_stats of estimate_energy (proj/src/trainer.cpp:184-211) over
        this rank's shard `batch`, reduced over every rank of `comm` (a
        distributed.NcclComm; None = this process alone) on the device.
        Returns a VmcEstimate whose energy / variance / std_err are global and
        whose local_energies are this rank's; `ledger` is added the whole
        job's ledger."""
        cfgs = np.ascontiguousarray(batch, np.uint8)
        if cfgs.ndim != 2 or cfgs.shape[1] != self.cfg.n_sites:
            raise ShapeError("configuration size != site count")
        B = cfgs.shape[0]
        e_re = np.zeros(B)
        lpsi = np.zeros(B)
        led = np.zeros(7, np.int64)
        st = np.zeros(4)
        N.check(N.lib().vqnqs_gpu_estimate_energy(
            self._h, comm.handle if comm is not None else None, N.ptr(cfgs, C.c_uint8), B,
            N.ptr(e_re, C.c_double), N.ptr(lpsi, C.c_double), N.ptr(led, C.c_int64),
            N.ptr(st, C.c_double)))
        if ledger is not None:
            ledger += Ledger.from_array(led)
        est = VmcEstimate(float(st[0]), float(st[1]), float(st[2]), e_re + 0j)
        est.k_total = int(st[3])
        est.logpsi = lpsi
        return est

    def fill_stats_device(self, d_e, comm=None, stream=None) -> "VmcEstimate":
        """fill_stats over device-resident local energies (a torch float64
        tensor, this rank's shard), global over `comm`'s ranks."""
        st = np.zeros(4)
        N.check(N.lib().vqnqs_gpu_fill_stats_device(
            self._h, comm.handle if comm is not None else None, C.c_void_p(d_e.data_ptr()),
            d_e.shape[0], N.ptr(st, C.c_double),
            C.c_void_p(stream.cuda_stream) if stream is not None else None))
        est = VmcEstimate(float(st[0]), float(st[1]), float(st[2]), np.zeros(0, complex))
        est.k_total = int(st[3])
        return est

    def set_code_override(self, codes) -> None:
        """Test hook (include/vqnqs_b200_debug.h): force the VQ code of every
        active location to codes[i, layer, row, position] (int16, rows in
        bond order, -1 keeps the computed code) for calls on batches of
        exactly len(codes) samples, so values after a flagged near-tie can be
        compared with the reference's; None clears."""
        f = N.lib().vqnqs_debug_set_code_override
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, C.POINTER(C.c_int16), C.c_int64]
        if codes is None:
            N.check(f(self._h, None, 0))
            return
        c = np.ascontiguousarray(codes, np.int16)
        self._override_keep = c
        N.check(f(self._h, c.ctypes.data_as(C.POINTER(C.c_int16)), int(c.shape[0])))

    def set_micro_batch(self, samples: int) -> None:
        """Samples per micro-batch (0 = sized from the working-set budget)."""
        N.check(N.lib().vqnqs_gpu_set_micro_batch(self._h, int(samples)))

    def last_launch_count(self) -> int:
        return int(N.lib().vqnqs_gpu_last_launch_count(self._h))

    def last_profile(self) -> np.ndarray:
        out = np.zeros(12)
        N.lib().vqnqs_gpu_last_profile(self._h, N.ptr(out, C.c_double), 12)
        return out


def _fingerprint(model: VqTransformer, h: HamiltonianModel) -> bytes:
    """Content hash of everything the engine snapshots at upload: the
    weights, the config, the bonds and the Hamiltonian's options."""
    import hashlib
    m = hashlib.blake2b(digest_size=16)
    m.update(repr(model.cfg).encode())
    for p in model.params:
        m.update(np.ascontiguousarray(p.value, np.float64).tobytes())
    m.update(np.ascontiguousarray(h.lattice.bonds, np.int32).tobytes())
    m.update(repr((h.kind, h.marshall, h.J, h.Gamma, h.n_sites())).encode())
    return m.digest()


# One cached engine for the stateless module-level calls. It is keyed on the
# CONTENT of the model and Hamiltonian (not on id()), so a VMC loop that
# updates parameters in place gets a fresh upload instead of stale weights,
# and a single slot bounds the device memory it holds. Callers that evaluate
# one model many times should hold a LocalEnergyEngine themselves: hashing
# the weights costs a pass over them per call.
_CACHE: Dict[str, object] = {}


def _engine_for(model, h, precision, device) -> LocalEnergyEngine:
    key = (_fingerprint(model, h), precision, device)
    if _CACHE.get("key") != key:
        old = _CACHE.pop("engine", None)
        if old is not None:
            old.close()
        _CACHE["engine"] = LocalEnergyEngine(model, h, precision, device)
        _CACHE["key"] = key
    return _CACHE["engine"]


def local_energies(model: VqTransformer, h: HamiltonianModel, batch,
                   ledger: Optional[Ledger] = None, precision: str = "fp32",
                   device: int = 0) -> np.ndarray:
    """local_energies(model, h, batch, ledger) — complex E_loc per sample.

    Stateless like the reference: every call evaluates the model's CURRENT
    weights (the upload is cached on a content hash of model and h)."""
    e, _ = _engine_for(model, h, precision, device).local_energies(batch, ledger)
    return e


def local_energy_batch(model: VqTransformer, h: HamiltonianModel, s,
                       precision: str = "fp32", device: int = 0):
    """local_energy_batch(model, h, s) -> (value, ledger)."""
    led = Ledger()
    e = local_energies(model, h, np.asarray(s, np.uint8)[None, :], led, precision, device)
    return complex(e[0]), led


@dataclass
class VmcEstimate:
    energy: float = 0.0
    variance: float = 0.0
    std_err: float = 0.0
    local_energies: np.ndarray = field(default_factory=lambda: np.zeros(0, complex))


def fill_stats(e_loc) -> VmcEstimate:
    """fill_stats (proj/src/trainer.cpp:184-198): mean and unbiased variance of Re E."""
    e = np.asarray(e_loc)
    k = e.shape[0]
    mean = float(np.sum(e.real)) / k
    var = float(np.sum((e.real - mean) ** 2)) / (k - 1) if k > 1 else 0.0
    return VmcEstimate(mean, var, math.sqrt(var / k), e)


# ---------------------------------------------------------------- gradient


class LogProbGradient:
    """d/dtheta sum_i w_i log P(s_i) on the GPU: the
    backward of vmc_gradient (proj/src/trainer.cpp:236-244) through the dense
    decoder with the straight-through VQ surrogate (autodiff.cpp:536-655)."""

    def __init__(self, model: VqTransformer, device: int = 0):
        self.model = model
        self.cfg = model.cfg
        desc = N.desc_of(model.cfg)
        vals = [np.ascontiguousarray(p.value, np.float64).reshape(-1) for p in model.params]
        arr = (N.P_F64 * len(vals))(*[N.ptr(v, C.c_double) for v in vals])
        h = C.c_void_p()
        N.check(N.lib().vqnqs_grad_create(C.byref(desc), arr, len(vals), device, C.byref(h)))
        self._h = h
        self._sizes = [int(p.value.size) for p in model.params]

    def close(self):
        if getattr(self, "_h", None):
            N.lib().vqnqs_grad_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def grad(self, configs, weights, vq_tau: float = 1.0):
        """([Parameter(name, grad)] in parameters() order, log P per sample)."""
        cfgs = np.ascontiguousarray(configs, np.uint8)
        w = np.ascontiguousarray(weights, np.float64)
        if cfgs.ndim != 2 or cfgs.shape[1] != self.cfg.n_sites or w.shape != (cfgs.shape[0],):
            raise ShapeError("configs [B x n_sites] and weights [B] expected")
        g = np.zeros(sum(self._sizes))
        lp = np.zeros(cfgs.shape[0])
        N.check(N.lib().vqnqs_grad_log_prob(self._h, N.ptr(cfgs, C.c_uint8), cfgs.shape[0],
                                            N.ptr(w, C.c_double), float(vq_tau),
                                            N.ptr(g, C.c_double), N.ptr(lp, C.c_double)))
        out, off = [], 0
        for p, n in zip(self.model.params, self._sizes):
            out.append(Parameter(p.name, g[off:off + n].reshape(p.value.shape)))
            off += n
        return out, lp


def vmc_gradient(engine: LocalEnergyEngine, grad: LogProbGradient, k_samples: int, seed: int,
                 vq_tau: float = 1.0, skip: int = 0):
    """vmc_gradient (proj/src/trainer.cpp:213-246, phase network off, gumbel
    off) on the GPU: K samples drawn with the model's sampler, local energies,
    weights w_i = Re(E_i - mean E) / K, then the backward. Returns
    ([Parameter(name, grad)], VmcEstimate)."""
    if k_samples < 2:
        raise ConfigError("k_samples must be >= 2")
    configs, _ = engine.sample(k_samples, seed, skip=skip)
    e, _ = engine.local_energies(configs)
    est = fill_stats(e)
    cmean = np.sum(e) / k_samples
    wa = np.real(e - cmean) / k_samples
    grads, _ = grad.grad(configs, wa, vq_tau)
    return grads, est

"""TEST INFRASTRUCTURE — ctypes front-ends for the two CPU checkers.

* ``RefLib``  wraps ``oracle/_ref/libvqnqs_ref.so``: the reference's own
  hot-path sources (proj/src/{flops,tensor,hamiltonian,model,dedup}.cpp)
  compiled unmodified, see oracle/Makefile and oracle/ref_harness.cpp.
* ``PortLib`` wraps ``oracle/_port/libvqnqs_oracle.so``: our plain-C
  restatement of the same algorithm (oracle/vqnqs_oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` legs may import this module. The product package
(paper_2212_11296_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libvqnqs_ref.so")
PORT_SO = os.path.join(HERE, "_port", "libvqnqs_oracle.so")

STATUS_NAMES = {1: "ConfigError", 2: "ShapeError", 3: "CapabilityError",
                4: "NumericError", 5: "UsageError", 6: "RuntimeError"}


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS_NAMES.get(status, "RuntimeError")


class ModelDesc(C.Structure):
    """Mirror of vqnqs_model_desc (include/vqnqs_b200.h)."""
    _fields_ = [("n_sites", C.c_int32), ("group_size", C.c_int32),
                ("d_hidden", C.c_int32), ("n_heads", C.c_int32),
                ("n_blocks", C.c_int32), ("trailing_half_block", C.c_int32),
                ("vq_enabled", C.c_int32), ("vq_heads", C.c_int32),
                ("vq_codebook", C.c_int32), ("phase_enabled", C.c_int32),
                ("vq_init_scale", C.c_double)]


def desc_from(cfg) -> ModelDesc:
    return ModelDesc(cfg.n_sites, cfg.group_size, cfg.d_hidden, cfg.n_heads,
                     cfg.n_blocks, int(cfg.trailing_half_block),
                     int(cfg.vq_enabled), cfg.vq_heads, cfg.vq_codebook,
                     int(cfg.phase_enabled), float(cfg.vq_init_scale))


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


P_U8, P_F64, P_I64, P_I32, P_F32 = (C.POINTER(C.c_uint8), C.POINTER(C.c_double),
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_float))

LATTICE_CODES = {"chain": 0, "grid": 1, "grid_periodic": 2, "chain_periodic": 3}


@dataclass
class Taps:
    K: int
    U: np.ndarray        # [L+1] int64
    codes: np.ndarray    # [L, K*T, H] int32
    gaps: np.ndarray     # [L, K*T] float32
    lp: np.ndarray       # [K] float64
    I_final: np.ndarray  # [K*T] int32


class _Common:
    """Shared C surface of the two checker libraries (same symbol names with
    prefix ``ref_`` / ``orc_``)."""

    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        f = self._f
        f("last_error").restype = C.c_char_p
        f("set_bf16_products").argtypes = [C.c_int]
        f("model_create").restype = C.c_void_p
        f("model_create").argtypes = [C.POINTER(ModelDesc), C.c_uint64, C.c_int]
        f("model_destroy").argtypes = [C.c_void_p]
        f("model_num_params").argtypes = [C.c_void_p]
        f("model_param").restype = C.c_int64
        f("model_param").argtypes = [C.c_void_p, C.c_int, C.POINTER(P_F64),
                                     C.POINTER(C.c_char_p)]
        f("ham_create").restype = C.c_void_p
        f("ham_create").argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_double, C.c_double]
        f("ham_destroy").argtypes = [C.c_void_p]
        f("ham_bonds").argtypes = [C.c_void_p, P_I32, C.c_int]
        f("connected_set").argtypes = [C.c_void_p, P_U8, C.c_int, P_U8, P_F64]
        f("zero_sz_samples").argtypes = [C.c_int, C.c_int64, C.c_int64,
                                         C.c_uint64, P_U8]
        f("local_energies").argtypes = [C.c_void_p, C.c_void_p, P_U8, C.c_int64,
                                        C.c_int, P_F64, P_F64, P_F64, P_I64]
        f("local_energies_fast").argtypes = [C.c_void_p, C.c_void_p, P_U8,
                                             C.c_int64, C.c_int, P_F64]
        f("dedup_log_prob").argtypes = [C.c_void_p, P_U8, C.c_int64, P_U8, P_F64]
        f("dense_log_prob").argtypes = [C.c_void_p, P_U8, C.c_int64, P_F64]
        f("sample").argtypes = [C.c_void_p, C.c_int, C.c_uint64, P_U8, P_F64]
        if self.prefix == "ref_":  # wire formats: the reference's own code
            f("save_checkpoint").argtypes = [C.c_void_p, C.c_char_p]
            f("load_checkpoint").restype = C.c_void_p
            f("load_checkpoint").argtypes = [C.c_char_p]
            f("measure_and_emit").argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                              C.c_uint64, C.c_double, C.c_char_p]
            f("log_prob_grad").argtypes = [C.c_void_p, P_U8, C.c_int64, P_F64, C.c_double,
                                           P_F64, P_F64]
        f("taps").argtypes = [C.c_void_p, C.c_void_p, P_U8, P_I64, P_I32, P_F32,
                              P_F64, P_I32]

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, st):
        if st != 0:
            raise OracleError(st, self._f("last_error")().decode())

    def set_bf16(self, on: bool):
        self._f("set_bf16_products")(int(on))

    def zero_sz_samples(self, n_sites, start, count, seed=1):
        out = np.zeros((count, n_sites), np.uint8)
        self._f("zero_sz_samples")(n_sites, start, count, seed, _p(out, C.c_uint8))
        return out

    # ----- model -----
    def model(self, cfg, seed=0, snap_bf16=False):
        d = desc_from(cfg)
        h = self._f("model_create")(C.byref(d), seed, int(snap_bf16))
        if not h:
            raise OracleError(1, self._f("last_error")().decode())
        return OracleModel(self, h, cfg)

    def load_checkpoint(self, path, cfg):
        """The reference's load_checkpoint (proj/src/checkpoint.cpp:79-124)."""
        h = self._f("load_checkpoint")(str(path).encode())
        if not h:
            raise OracleError(1, self._f("last_error")().decode())
        return OracleModel(self, h, cfg)

    def hamiltonian(self, lattice="grid_periodic", lx=4, ly=4, kind="heisenberg",
                    marshall=True, J=1.0, Gamma=1.0):
        h = self._f("ham_create")(0 if kind == "tfim" else 1,
                                  LATTICE_CODES[lattice], lx, ly, int(marshall),
                                  J, Gamma)
        if not h:
            raise OracleError(1, self._f("last_error")().decode())
        return OracleHam(self, h, lx * (ly if "grid" in lattice else 1))


class OracleHam:
    def __init__(self, lib, h, n):
        self.lib, self.h, self.n_sites = lib, h, n

    def __del__(self):
        try:
            self.lib._f("ham_destroy")(self.h)
        except Exception:
            pass

    def bonds(self):
        nb = self.lib._f("ham_bonds")(self.h, None, 0)
        out = np.zeros((nb, 2), np.int32)
        self.lib._f("ham_bonds")(self.h, _p(out, C.c_int32), nb)
        return out

    def connected_set(self, s):
        s = np.ascontiguousarray(s, np.uint8)
        K = self.lib._f("connected_set")(self.h, _p(s, C.c_uint8), 0, None, None)
        if K < 0:
            raise OracleError(-K, self.lib._f("last_error")().decode())
        cf = np.zeros((K, self.n_sites), np.uint8)
        co = np.zeros(K, np.float64)
        self.lib._f("connected_set")(self.h, _p(s, C.c_uint8), K,
                                     _p(cf, C.c_uint8), _p(co, C.c_double))
        return cf, co


class OracleModel:
    def __init__(self, lib, h, cfg):
        self.lib, self.h, self.cfg = lib, h, cfg

    def __del__(self):
        try:
            self.lib._f("model_destroy")(self.h)
        except Exception:
            pass

    def log_prob_grad(self, configs, weights, vq_tau=1.0):
        """d/dtheta sum_i w_i log P(s_i) on the reference's tape (build_log_prob +
        weighted_sum + backward, proj/src/trainer.cpp:236-244): ([(name, grad)],
        log-probs)."""
        configs = np.ascontiguousarray(configs, np.uint8)
        w = np.ascontiguousarray(weights, np.float64)
        params = self.params()
        total = sum(p.size for _, p in params)
        g = np.zeros(total)
        lp = np.zeros(configs.shape[0])
        self.lib._check(self.lib._f("log_prob_grad")(
            self.h, _p(configs, C.c_uint8), configs.shape[0], _p(w, C.c_double), vq_tau,
            _p(g, C.c_double), _p(lp, C.c_double)))
        out, off = [], 0
        for name, p in params:
            out.append((name, g[off:off + p.size].copy()))
            off += p.size
        return out, lp

    def save_checkpoint(self, path):
        self.lib._check(self.lib._f("save_checkpoint")(self.h, str(path).encode()))

    def measure_and_emit(self, ham, samples_per_batch, batches, seed, directory,
                         reference_per_site=float("nan")):
        """measure_flops + emit_table (proj/src/bench.cpp:65-124, 270-290)."""
        self.lib._check(self.lib._f("measure_and_emit")(
            self.h, ham.h, samples_per_batch, batches, seed, reference_per_site,
            str(directory).encode()))

    def params(self):
        """[(name, float64 array)] in parameters() order."""
        out = []
        n = self.lib._f("model_num_params")(self.h)
        for i in range(n):
            ptr = P_F64()
            name = C.c_char_p()
            numel = self.lib._f("model_param")(self.h, i, C.byref(ptr), C.byref(name))
            arr = np.ctypeslib.as_array(ptr, shape=(numel,)).copy()
            out.append((name.value.decode(), arr))
        return out

    def set_param(self, i, values):
        ptr = P_F64()
        numel = self.lib._f("model_param")(self.h, i, C.byref(ptr), None)
        v = np.ascontiguousarray(values, np.float64).reshape(-1)
        assert v.size == numel
        np.ctypeslib.as_array(ptr, shape=(numel,))[:] = v

    def local_energies(self, ham, configs, workers=1, with_logpsi=True):
        configs = np.ascontiguousarray(configs, np.uint8)
        B = configs.shape[0]
        e_re = np.zeros(B)
        e_im = np.zeros(B)
        lpsi = np.zeros(B) if with_logpsi else None
        led = np.zeros(7, np.int64)
        st = self.lib._f("local_energies")(self.h, ham.h, _p(configs, C.c_uint8), B,
                                           workers, _p(e_re, C.c_double),
                                           _p(e_im, C.c_double),
                                           _p(lpsi, C.c_double), _p(led, C.c_int64))
        self.lib._check(st)
        return e_re, e_im, lpsi, led

    def local_energies_fast(self, ham, configs, workers=1):
        configs = np.ascontiguousarray(configs, np.uint8)
        e_re = np.zeros(configs.shape[0])
        st = self.lib._f("local_energies_fast")(self.h, ham.h,
                                                _p(configs, C.c_uint8),
                                                configs.shape[0], workers,
                                                _p(e_re, C.c_double))
        self.lib._check(st)
        return e_re

    def dedup_log_prob(self, configs, base):
        configs = np.ascontiguousarray(configs, np.uint8)
        base = np.ascontiguousarray(base, np.uint8)
        lp = np.zeros(configs.shape[0])
        self.lib._check(self.lib._f("dedup_log_prob")(
            self.h, _p(configs, C.c_uint8), configs.shape[0], _p(base, C.c_uint8),
            _p(lp, C.c_double)))
        return lp

    def dense_log_prob(self, configs):
        configs = np.ascontiguousarray(configs, np.uint8)
        lp = np.zeros(configs.shape[0])
        self.lib._check(self.lib._f("dense_log_prob")(
            self.h, _p(configs, C.c_uint8), configs.shape[0], _p(lp, C.c_double)))
        return lp

    def sample(self, count, seed):
        """VqTransformer::sample (proj/src/model.cpp:485-525) with Rng(seed)."""
        out = np.zeros((count, self.cfg.n_sites), np.uint8)
        lp = np.zeros(count)
        self.lib._check(self.lib._f("sample")(self.h, count, seed, _p(out, C.c_uint8),
                                              _p(lp, C.c_double)))
        return out, lp

    def taps(self, ham, s):
        cfg = self.cfg
        s = np.ascontiguousarray(s, np.uint8)
        K = ham.connected_set(s)[0].shape[0]
        T = -(-cfg.n_sites // cfg.group_size)
        L = cfg.n_blocks + int(cfg.trailing_half_block)
        H = cfg.vq_heads
        U = np.zeros(L + 1, np.int64)
        codes = np.zeros((L, K * T, H), np.int32)
        gaps = np.zeros((L, K * T), np.float32)
        lp = np.zeros(K)
        If = np.zeros(K * T, np.int32)
        self.lib._check(self.lib._f("taps")(
            self.h, ham.h, _p(s, C.c_uint8), _p(U, C.c_int64), _p(codes, C.c_int32),
            _p(gaps, C.c_float), _p(lp, C.c_double), _p(If, C.c_int32)))
        return Taps(K, U, codes, gaps, lp, If)


class RefLib(_Common):
    prefix = "ref_"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)


class PortLib(_Common):
    prefix = "orc_"

    def __init__(self, path: str = PORT_SO):
        super().__init__(path)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def port_available() -> bool:
    return os.path.exists(PORT_SO)

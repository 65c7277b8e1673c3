"""ctypes binding of the native library (include/vqnqs_b200.h).

The library is built in-tree (``python -m paper_2212_11296_b200.build``).
There is no fallback: if the .so is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .config import STATUS_ERRORS, VqnqsError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                        "libvqnqs_b200.so")


class ModelDesc(C.Structure):
    _fields_ = [("n_sites", C.c_int32), ("group_size", C.c_int32),
                ("d_hidden", C.c_int32), ("n_heads", C.c_int32),
                ("n_blocks", C.c_int32), ("trailing_half_block", C.c_int32),
                ("vq_enabled", C.c_int32), ("vq_heads", C.c_int32),
                ("vq_codebook", C.c_int32), ("phase_enabled", C.c_int32),
                ("vq_init_scale", C.c_double)]


def desc_of(cfg) -> ModelDesc:
    if cfg.local_dim != 2:
        from .config import ConfigError
        raise ConfigError("only d=2 local states")
    return ModelDesc(cfg.n_sites, cfg.group_size, cfg.d_hidden, cfg.n_heads,
                     cfg.n_blocks, int(cfg.trailing_half_block), int(cfg.vq_enabled),
                     cfg.vq_heads, cfg.vq_codebook, int(cfg.phase_enabled),
                     float(cfg.vq_init_scale))


P_U8, P_F64, P_I64, P_I32 = (C.POINTER(C.c_uint8), C.POINTER(C.c_double),
                             C.POINTER(C.c_int64), C.POINTER(C.c_int32))

# Every symbol include/vqnqs_b200.h declares, with its ctypes signature.
SIGNATURES = {
    "vqnqs_last_error": (C.c_char_p, []),
    "vqnqs_param_layout": (C.c_int, [C.POINTER(ModelDesc), C.POINTER(C.c_int), P_I64]),
    "vqnqs_init_params": (C.c_int, [C.POINTER(ModelDesc), C.c_uint64, C.c_int,
                                    C.POINTER(P_F64)]),
    "vqnqs_build_lattice": (C.c_int, [C.c_int, C.c_int, C.c_int, P_I32, C.c_int]),
    "vqnqs_zero_sz_samples": (C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_uint64, P_U8]),
    "vqnqs_ledger_from_counts": (C.c_int, [C.POINTER(ModelDesc), C.c_int64, P_I64, P_I64]),
    "vqnqs_gpu_create": (C.c_int, [C.POINTER(ModelDesc), C.POINTER(P_F64), C.c_int, C.c_int,
                                   C.c_int, C.POINTER(C.c_void_p)]),
    "vqnqs_gpu_set_hamiltonian": (C.c_int, [C.c_void_p, P_I32, C.c_int, C.c_int, C.c_int]),
    "vqnqs_gpu_set_reuse": (C.c_int, [C.c_void_p, C.c_int]),
    "vqnqs_gpu_set_micro_batch": (C.c_int, [C.c_void_p, C.c_int]),
    "vqnqs_comm_unique_id": (C.c_int, [C.c_char_p]),
    "vqnqs_comm_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(C.c_void_p)]),
    "vqnqs_comm_destroy": (C.c_int, [C.c_void_p]),
    "vqnqs_gpu_estimate_energy": (C.c_int, [C.c_void_p, C.c_void_p, P_U8, C.c_int64, P_F64,
                                            P_F64, P_I64, P_F64]),
    "vqnqs_gpu_fill_stats_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                              P_F64, C.c_void_p]),
    "vqnqs_balanced_shards": (C.c_int, [P_U8, C.c_int64, C.c_int, P_I32, C.c_int, C.c_int,
                                        P_I32]),
    "vqnqs_grad_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "vqnqs_grad_log_prob": (C.c_int, [C.c_void_p, P_U8, C.c_int64, P_F64, C.c_double, P_F64,
                                      P_F64]),
    "vqnqs_grad_destroy": (C.c_int, [C.c_void_p]),
    "vqnqs_gpu_sample": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint64, C.c_uint64, P_U8,
                                   P_F64]),
    "vqnqs_gpu_local_energies": (C.c_int, [C.c_void_p, P_U8, C.c_int64, P_F64, P_F64, P_F64,
                                           P_I64]),
    "vqnqs_gpu_local_energies_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64,
                                                  C.c_void_p, C.c_void_p, P_I64, C.c_void_p]),
    "vqnqs_gpu_connected_log_probs": (C.c_int, [C.c_void_p, P_U8, P_F64, C.c_int]),
    "vqnqs_gpu_taps": (C.c_int, [C.c_void_p, P_U8, C.c_int64, P_I32, P_I64, P_I32, C.c_int64,
                                  P_F64, C.c_int64]),
    "vqnqs_gpu_last_launch_count": (C.c_int64, [C.c_void_p]),
    "vqnqs_gpu_last_profile": (C.c_int, [C.c_void_p, P_F64, C.c_int]),
    "vqnqs_gpu_destroy": (C.c_int, [C.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load the native library (once). Raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"native library missing: {LIB_PATH}. Build it with "
                    "`python -m paper_2212_11296_b200.build` (there is no CPU fallback).")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
        return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().vqnqs_last_error().decode(errors="replace")
        raise STATUS_ERRORS.get(status, VqnqsError)(msg)


def ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None

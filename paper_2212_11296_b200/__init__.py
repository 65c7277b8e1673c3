"""B200-native local-energy step of VQ-NQS (arXiv 2212.11296).

The reference's local-energy interface (proj/include/vqnqs/{trainer,dedup}.hpp)
re-implemented on hand-written sm_100a kernels behind a C ABI
(include/vqnqs_b200.h). See DESIGN.md.
"""
from .config import (CapabilityError, ConfigError, ModelConfig, NumericError, ShapeError,
                     UsageError, VqnqsError, WORKLOADS, Workload, workload)

_API = {"VqTransformer", "Parameter", "Lattice", "build_lattice", "HamiltonianModel",
        "zero_sz_samples", "Ledger", "LocalEnergyEngine", "local_energies",
        "local_energy_batch", "VmcEstimate", "fill_stats", "param_shapes", "LogProbGradient",
        "vmc_gradient"}


def __getattr__(name):
    if name in _API:
        from . import api
        return getattr(api, name)
    raise AttributeError(name)

"""Model configuration and the five BASELINE workloads.

``ModelConfig`` mirrors the reference's ``vqnqs::ModelConfig``
(proj/include/vqnqs/model.hpp:13-48) field for field, including
``validate()`` (proj/src/model.cpp:10-27) and the derived ``seq_len``,
``vocab`` and ``last_vocab``. ``WORKLOADS`` pins every decision SURVEY §8(d)
asks the run config to record (periodic bond order, group_size=2, no trailing
half block, H=1, vq_init_scale=1/d, Marshall sign, zero-Sz sampler seeds).
"""
from __future__ import annotations

import math
from dataclasses import asdict, dataclass, field, replace


class VqnqsError(RuntimeError):
    """Base of the reference's error taxonomy (proj/include/vqnqs/common.hpp:14-28)."""


class ConfigError(VqnqsError):
    pass


class ShapeError(VqnqsError):
    pass


class CapabilityError(VqnqsError):
    pass


class NumericError(VqnqsError):
    pass


class UsageError(VqnqsError):
    pass


STATUS_ERRORS = {1: ConfigError, 2: ShapeError, 3: CapabilityError,
                 4: NumericError, 5: UsageError, 6: VqnqsError}


@dataclass(frozen=True)
class ModelConfig:
    n_sites: int = 4
    local_dim: int = 2
    group_size: int = 2
    d_hidden: int = 32
    n_heads: int = 4
    n_blocks: int = 2
    trailing_half_block: bool = True
    vq_enabled: bool = True
    vq_heads: int = 1
    vq_codebook: int = 64
    vq_temperature: float = 1.0
    vq_gumbel: bool = False
    vq_init_scale: float = 0.05
    phase_enabled: bool = False

    @property
    def seq_len(self) -> int:
        return (self.n_sites + self.group_size - 1) // self.group_size

    @property
    def vocab(self) -> int:
        return self.local_dim ** self.group_size

    @property
    def last_vocab(self) -> int:
        rem = self.n_sites % self.group_size
        return self.vocab if rem == 0 else self.local_dim ** rem

    @property
    def n_layers(self) -> int:
        return self.n_blocks + int(self.trailing_half_block)

    def validate(self) -> None:
        """proj/src/model.cpp:10-27, same messages."""
        if self.n_sites < 1:
            raise ConfigError("n_sites must be positive")
        if self.local_dim != 2:
            raise ConfigError("only d=2 local states")
        if self.group_size < 1 or self.group_size > 16:
            raise ConfigError("group_size out of range")
        if self.d_hidden < 1:
            raise ConfigError("d_hidden must be positive")
        if self.n_heads < 1 or self.d_hidden % self.n_heads != 0:
            raise ConfigError("d_hidden must divide into n_heads")
        if self.n_blocks < 0:
            raise ConfigError("n_blocks must be nonnegative")
        if self.n_blocks == 0 and not self.trailing_half_block:
            raise ConfigError("model needs at least one block")
        if self.vq_enabled:
            if self.vq_heads < 1 or self.d_hidden % self.vq_heads != 0:
                raise ConfigError("d_hidden must divide into vq_heads")
            if self.vq_codebook < 1:
                raise ConfigError("vq_codebook must be positive")
            if not self.vq_temperature > 0:
                raise ConfigError("vq_temperature must be > 0")


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config with the SURVEY §8(d) decisions applied."""
    name: str
    L: int                    # periodic L x L lattice
    batch: int                # zero-Sz samples per batch
    model: ModelConfig
    precision: str            # "fp32" | "bf16" (GEMM operand precision)
    sample_seed: int = 1      # sample i <- Rng(sample_seed).split(i)
    weight_seed: int = 0      # VqTransformer::init(cfg, Rng(weight_seed))
    marshall: bool = True
    notes: str = ""

    @property
    def n_sites(self) -> int:
        return self.L * self.L

    @property
    def n_bonds(self) -> int:
        return 2 * self.L * self.L

    def record(self) -> dict:
        d = asdict(self)
        d["model"] = asdict(self.model)
        d.update(lattice=f"{self.L}x{self.L} periodic", n_bonds=self.n_bonds,
                 bond_order="horizontals then verticals, row-major, (min,max)",
                 hamiltonian="heisenberg J=1, marshall off-diagonal -1/2")
        return d


def _model(n, d, layers, heads, q) -> ModelConfig:
    return ModelConfig(n_sites=n, group_size=2, d_hidden=d, n_heads=heads,
                       n_blocks=layers, trailing_half_block=False, vq_enabled=True,
                       vq_heads=1, vq_codebook=q, vq_init_scale=1.0 / d)


WORKLOADS = {
    "c1_4x4": Workload("c1_4x4", 4, 256, _model(16, 32, 2, 4, 64), "fp32",
                       notes="reference's CPU-runnable case"),
    "c2_6x6": Workload("c2_6x6", 6, 1024, _model(36, 64, 4, 4, 128), "fp32"),
    "c3_10x10": Workload("c3_10x10", 10, 4096, _model(100, 128, 6, 8, 256), "bf16"),
    "c4_16x16": Workload("c4_16x16", 16, 8192, _model(256, 256, 8, 8, 512), "bf16"),
    "c5_12x12": Workload("c5_12x12", 12, 4096, _model(144, 768, 12, 12, 1024), "bf16"),
}


def workload(name: str) -> Workload:
    for k, w in WORKLOADS.items():
        if name == k or name == k.split("_")[0]:
            return w
    raise ConfigError(f"unknown workload {name!r}; choose from {list(WORKLOADS)}")


def n_params(cfg: ModelConfig) -> int:
    d, v, t = cfg.d_hidden, cfg.vocab, cfg.seq_len
    blk = 2 * d + 4 * (d * d + d) + 2 * d + d * 4 * d + 4 * d + 4 * d * d + d
    cb = cfg.vq_codebook * cfg.vq_heads * (d // cfg.vq_heads) if cfg.vq_enabled else 0
    return (v + 1) * d + t * d + cfg.n_blocks * (blk + cb) + 2 * d + d * v + v

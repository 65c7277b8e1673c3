"""Wire formats around the hot path.

* Checkpoints (proj/src/checkpoint.cpp:53-126): magic "VQNQS1\\0", a uint64
  little-endian header length, a compact JSON header
  {"config": {...}, "tensors": [{"name", "shape", "offset"}, ...]} (keys in
  sorted order, as nlohmann::json's std::map objects print them), then every
  parameter as raw float64 in parameters() order. `load_checkpoint` reads the
  reference's files into a VqTransformer the GPU engine takes as is;
  `save_checkpoint` writes byte-identical files.
* The measurement report (measure_flops + emit_table, proj/src/bench.cpp:
  65-124, 218-290): B configurations drawn with the model's own sampler,
  local energies under the FLOP ledger, and report.csv / report.json with the
  reference's columns, formats and key order. Here both the draws and the
  local energies run on the GPU.
"""
from __future__ import annotations

import json
import math
import os
import struct
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from .api import Ledger, LocalEnergyEngine, Parameter, VqTransformer, param_shapes
from .config import CapabilityError, ConfigError, ModelConfig

MAGIC = b"VQNQS1\0"
CONFIG_KEYS = ("n_sites", "local_dim", "group_size", "d_hidden", "n_heads", "n_blocks",
               "trailing_half_block", "vq_enabled", "vq_heads", "vq_codebook",
               "vq_temperature", "vq_gumbel", "vq_init_scale", "phase_enabled")


def _config_json(cfg: ModelConfig) -> dict:
    """to_json(ModelConfig), proj/src/checkpoint.cpp:19-34."""
    return {k: getattr(cfg, k) for k in CONFIG_KEYS}


def save_checkpoint(model: VqTransformer, path: str) -> None:
    """save_checkpoint, proj/src/checkpoint.cpp:53-77."""
    manifest, offset = [], 0
    for p in model.parameters():
        manifest.append({"name": p.name, "offset": offset, "shape": list(p.value.shape)})
        offset += 8 * int(p.value.size)
    header = json.dumps({"config": _config_json(model.cfg), "tensors": manifest},
                        sort_keys=True, separators=(",", ":")).encode()
    try:
        with open(path, "wb") as f:
            f.write(MAGIC)
            f.write(struct.pack("<Q", len(header)))
            f.write(header)
            for p in model.parameters():
                f.write(np.ascontiguousarray(p.value, "<f8").tobytes())
    except OSError as e:
        raise ConfigError(f"cannot open checkpoint for writing: {path}") from e


def load_checkpoint(path: str) -> VqTransformer:
    """load_checkpoint, proj/src/checkpoint.cpp:79-124 (same checks, same
    ConfigError messages)."""
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError as e:
        raise ConfigError(f"cannot open checkpoint: {path}") from e
    if blob[:len(MAGIC)] != MAGIC:
        raise ConfigError(f"not a model checkpoint: {path}")
    if len(blob) < len(MAGIC) + 8:
        raise ConfigError("corrupt checkpoint header")
    (n,) = struct.unpack_from("<Q", blob, len(MAGIC))
    if n > (1 << 30):
        raise ConfigError("corrupt checkpoint header")
    start = len(MAGIC) + 8
    if len(blob) < start + n:
        raise ConfigError("truncated checkpoint header")
    try:
        header = json.loads(blob[start:start + n].decode())
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise ConfigError(f"bad checkpoint header: {e}") from e
    c = header["config"]
    cfg = ModelConfig(**{k: type(getattr(ModelConfig(), k))(c[k]) for k in CONFIG_KEYS})
    cfg.validate()
    if cfg.phase_enabled:
        raise CapabilityError("checkpoint has the phase network (out of the GPU path's scope)")
    shapes = param_shapes(cfg)
    tensors = header["tensors"]
    if len(tensors) != len(shapes):
        raise ConfigError("checkpoint tensor count mismatch")
    data = start + n
    params = []
    for entry, (name, shape) in zip(tensors, shapes):
        if entry["name"] != name:
            raise ConfigError(f"checkpoint tensor order mismatch at {name}")
        if tuple(entry["shape"]) != tuple(shape):
            raise ConfigError(f"checkpoint tensor shape mismatch at {name}")
        off = data + int(entry["offset"])
        cnt = int(np.prod(shape))
        if off + 8 * cnt > len(blob):
            raise ConfigError(f"truncated checkpoint data at {name}")
        params.append(Parameter(name, np.frombuffer(blob, "<f8", cnt, off).reshape(shape).copy()))
    return VqTransformer(cfg, params)


# ------------------------------------------------------------- the report

@dataclass
class MeasurementReport:
    """MeasurementReport, proj/include/vqnqs/bench.hpp:17-39."""
    system: str
    model_bits: str
    n_sites: int
    batches: int
    samples_per_batch: int
    flops_dense: int = 0
    flops_dedup: int = 0
    per_location: int = 0
    attention: int = 0
    vq_distance: int = 0
    other: int = 0
    quantized_dense: int = 0
    quantized_dedup: int = 0
    total_savings: float = 1.0
    quantized_ops_savings: float = 1.0
    energy: float = 0.0
    energy_per_site: float = 0.0
    reference_energy: float = math.nan
    relative_error: float = math.nan


def model_bits_label(cfg: ModelConfig) -> str:
    """proj/src/bench.cpp:57-63."""
    if not cfg.vq_enabled:
        return "baseline"
    bits = cfg.vq_heads * math.log2(cfg.vq_codebook)
    if bits == math.floor(bits):
        return f"{int(bits)}b"
    return "%.1fb" % bits


def measure_flops(engine: LocalEnergyEngine, samples_per_batch: int, batches: int, seed: int,
                  reference_per_site: float = math.nan, system: Optional[str] = None
                  ) -> MeasurementReport:
    """measure_flops, proj/src/bench.cpp:65-124, with rng = Rng(seed): batch b
    continues the same uniform stream (skip = b * samples_per_batch * T)."""
    if samples_per_batch < 1 or batches < 1:
        raise ConfigError("measurement needs at least one sample and one batch")
    cfg = engine.cfg
    T = cfg.seq_len
    rep = MeasurementReport(system=system or engine.system_name(), model_bits=model_bits_label(cfg),
                            n_sites=cfg.n_sites, batches=batches,
                            samples_per_batch=samples_per_batch)
    total = Ledger()
    esum, count = 0.0, 0
    for b in range(batches):
        configs, _ = engine.sample(samples_per_batch, seed, skip=b * samples_per_batch * T)
        led = Ledger()
        e, _ = engine.local_energies(configs, led)
        total += led
        esum += float(np.real(np.sum(e)))  # Re E (bench.cpp:90)
        count += len(e)
    rep.flops_dense = total.total_dense()
    rep.flops_dedup = total.total_dedup()
    rep.per_location = total.per_location_unique
    rep.attention = total.attention
    rep.vq_distance = total.vq_distance
    rep.other = total.other
    rep.quantized_dense = total.per_location_dense_quantized
    rep.quantized_dedup = total.per_location_unique_quantized
    rep.total_savings = rep.flops_dense / rep.flops_dedup
    rep.quantized_ops_savings = (rep.quantized_dense / rep.quantized_dedup
                                 if rep.quantized_dedup > 0 else 1.0)
    rep.energy = esum / count
    rep.energy_per_site = rep.energy / rep.n_sites
    rep.reference_energy = reference_per_site
    rep.relative_error = (abs(rep.energy_per_site - reference_per_site) / abs(reference_per_site)
                          if math.isfinite(reference_per_site) else math.nan)
    return rep


CSV_HEADER = ("system,model,n_sites,batches,samples_per_batch,energy,energy_per_site,"
              "reference_energy,relative_error,total_savings,quantized_ops_savings,"
              "flops_dense,flops_dedup,per_location,attention,vq_distance,other,"
              "quantized_dense,quantized_dedup")


def csv_row(r: MeasurementReport) -> str:
    """proj/src/bench.cpp:225-246."""
    row = f"{r.system},{r.model_bits},{r.n_sites},{r.batches},{r.samples_per_batch}," \
          f"{'%.6f' % r.energy},{'%.6f' % r.energy_per_site},"
    row += "%.6f" % r.reference_energy if math.isfinite(r.reference_energy) else ""
    row += ","
    row += "%.1e" % r.relative_error if math.isfinite(r.relative_error) else ""
    row += (f",{'%.6f' % r.total_savings},{'%.6f' % r.quantized_ops_savings},"
            f"{r.flops_dense},{r.flops_dedup},{r.per_location},{r.attention},"
            f"{r.vq_distance},{r.other},{r.quantized_dense},{r.quantized_dedup}")
    return row


def report_json(r: MeasurementReport) -> dict:
    """proj/src/bench.cpp:248-268."""
    j = {"system": r.system, "model": r.model_bits, "n_sites": r.n_sites, "batches": r.batches,
         "samples_per_batch": r.samples_per_batch, "energy": r.energy,
         "energy_per_site": r.energy_per_site}
    if math.isfinite(r.reference_energy):
        j["reference_energy"] = r.reference_energy
        j["relative_error"] = r.relative_error
    j.update({"total_savings": r.total_savings, "quantized_ops_savings": r.quantized_ops_savings,
              "flops_dense": r.flops_dense, "flops_dedup": r.flops_dedup,
              "breakdown": {"per_location": r.per_location, "attention": r.attention,
                            "vq_distance": r.vq_distance, "other": r.other},
              "quantized_dense": r.quantized_dense, "quantized_dedup": r.quantized_dedup,
              "flop_convention": "analytic shape counts, multiply-add = 2"})
    return j


def _nl_double(x: float) -> str:
    # nlohmann::json prints doubles as the shortest round-trip form and keeps
    # a ".0" on integral values, like Python's repr
    return repr(float(x))


def _nl_dump(v, indent: int, level: int = 0) -> str:
    """nlohmann::json::dump(indent) for the value types a report holds:
    objects print their keys sorted (std::map), arrays one item per line."""
    pad, inner = " " * (indent * level), " " * (indent * (level + 1))
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [f'{inner}{json.dumps(k)}: {_nl_dump(v[k], indent, level + 1)}'
                 for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, list):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(inner + _nl_dump(x, indent, level + 1) for x in v) + \
            "\n" + pad + "]"
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, float):
        return _nl_double(v)
    return json.dumps(v)


def emit_table(reports: List[MeasurementReport], directory: str) -> None:
    """emit_table, proj/src/bench.cpp:270-290: <dir>/report.csv, report.json."""
    if not reports:
        raise ValueError("emit_table needs at least one report")
    os.makedirs(directory, exist_ok=True)
    with open(os.path.join(directory, "report.csv"), "w") as f:
        f.write(CSV_HEADER + "\n")
        for r in reports:
            f.write(csv_row(r) + "\n")
    with open(os.path.join(directory, "report.json"), "w") as f:
        f.write(_nl_dump([report_json(r) for r in reports], 2) + "\n")


def parse_report_json(path: str) -> List[MeasurementReport]:
    """Reports back from a report.json (ours or the reference's)."""
    out = []
    for j in json.load(open(path)):
        b = j["breakdown"]
        out.append(MeasurementReport(
            system=j["system"], model_bits=j["model"], n_sites=j["n_sites"],
            batches=j["batches"], samples_per_batch=j["samples_per_batch"],
            flops_dense=j["flops_dense"], flops_dedup=j["flops_dedup"],
            per_location=b["per_location"], attention=b["attention"],
            vq_distance=b["vq_distance"], other=b["other"],
            quantized_dense=j["quantized_dense"], quantized_dedup=j["quantized_dedup"],
            total_savings=j["total_savings"], quantized_ops_savings=j["quantized_ops_savings"],
            energy=j["energy"], energy_per_site=j["energy_per_site"],
            reference_energy=j.get("reference_energy", math.nan),
            relative_error=j.get("relative_error", math.nan)))
    return out

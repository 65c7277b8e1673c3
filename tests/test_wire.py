"""CPU: the §8(f) rank-4 wire formats against the reference's own writers
(tests/golden/ckpt_c1.vqnqs and report_c1/ were written by the reference's
save_checkpoint and measure_flops + emit_table through oracle/_ref; see
tests/golden/make_golden.py)."""
import math
import os
import shutil

import numpy as np
import pytest

import paper_2212_11296_b200 as P
from paper_2212_11296_b200 import wire
from paper_2212_11296_b200.config import ConfigError, ModelConfig

HERE = os.path.dirname(os.path.abspath(__file__))
CKPT = os.path.join(HERE, "golden", "ckpt_c1.vqnqs")
REPORT = os.path.join(HERE, "golden", "report_c1")


def test_load_reference_checkpoint():
    m = wire.load_checkpoint(CKPT)
    ref = P.VqTransformer.init(P.workload("c1").model, 0)
    assert m.cfg == ref.cfg
    for a, b in zip(m.params, ref.params):
        assert a.name == b.name and np.array_equal(a.value, b.value)


def test_save_is_byte_identical(tmp_path):
    out = tmp_path / "c1.vqnqs"
    wire.save_checkpoint(P.VqTransformer.init(P.workload("c1").model, 0), str(out))
    assert out.read_bytes() == open(CKPT, "rb").read()


def test_round_trip_other_configs(tmp_path):
    cfg = ModelConfig(n_sites=12, group_size=3, d_hidden=24, n_heads=2, n_blocks=1,
                      trailing_half_block=True, vq_heads=2, vq_codebook=16,
                      vq_init_scale=0.125)
    m = P.VqTransformer.init(cfg, 9)
    p = tmp_path / "x.vqnqs"
    wire.save_checkpoint(m, str(p))
    m2 = wire.load_checkpoint(str(p))
    assert m2.cfg == cfg
    assert all(np.array_equal(a.value, b.value) for a, b in zip(m.params, m2.params))


def test_checkpoint_errors(tmp_path):
    blob = open(CKPT, "rb").read()
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOTVQ" + blob[5:])
    with pytest.raises(ConfigError, match="not a model checkpoint"):
        wire.load_checkpoint(str(bad))
    bad.write_bytes(blob[:20])
    with pytest.raises(ConfigError, match="truncated checkpoint header"):
        wire.load_checkpoint(str(bad))
    bad.write_bytes(blob[:-8])
    with pytest.raises(ConfigError, match="truncated checkpoint data"):
        wire.load_checkpoint(str(bad))
    with pytest.raises(ConfigError, match="cannot open"):
        wire.load_checkpoint(str(tmp_path / "missing"))


def test_report_writer_is_byte_identical(tmp_path):
    reps = wire.parse_report_json(os.path.join(REPORT, "report.json"))
    wire.emit_table(reps, str(tmp_path))
    for f in ("report.csv", "report.json"):
        assert (tmp_path / f).read_text() == open(os.path.join(REPORT, f)).read()
    # with a reference energy (the optional columns / keys)
    r = reps[0]
    r.reference_energy, r.relative_error = -0.5, abs(r.energy_per_site + 0.5) / 0.5
    row = wire.csv_row(r).split(",")
    assert row[7] == "-0.500000" and row[8] == "%.1e" % r.relative_error
    assert "reference_energy" in wire.report_json(r)


def test_model_bits_label():
    c = P.workload("c4").model
    assert wire.model_bits_label(c) == "9b"
    from dataclasses import replace
    assert wire.model_bits_label(replace(c, vq_codebook=100)) == "%.1fb" % math.log2(100)
    assert wire.model_bits_label(replace(c, vq_enabled=False)) == "baseline"


def test_live_reference_checkpoint_reader(ref, tmp_path):
    """The reference reads our files (and we read its files) for a bf16-snapped
    c3 model too."""
    w = P.workload("c3")
    m = P.VqTransformer.init(w.model, 4, snap_bf16=True)
    p = tmp_path / "c3.vqnqs"
    wire.save_checkpoint(m, str(p))
    rm = ref.load_checkpoint(str(p), w.model)
    assert all(np.array_equal(a.value.reshape(-1), b) for a, (_, b) in zip(m.params, rm.params()))

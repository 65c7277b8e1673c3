"""GPU: a reference checkpoint through the GPU path, and the reference's
measurement report reproduced with GPU draws and GPU local energies
(measure_flops, proj/src/bench.cpp:65-124): same samples, so the same FLOP
ledger to the integer; energies agree to fp32 rounding."""
import math
import os

import pytest

import paper_2212_11296_b200 as P
from paper_2212_11296_b200 import wire

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_measure_flops_matches_reference_report(tmp_path):
    model = wire.load_checkpoint(os.path.join(HERE, "golden", "ckpt_c1.vqnqs"))
    ham = P.HamiltonianModel(P.build_lattice("grid2d", (4, 4), periodic=True))
    eng = P.LocalEnergyEngine(model, ham, precision="fp32")
    rep = wire.measure_flops(eng, 8, 2, 5)
    (gold,) = wire.parse_report_json(os.path.join(HERE, "golden", "report_c1", "report.json"))
    for f in ("system", "model_bits", "n_sites", "batches", "samples_per_batch", "flops_dense",
              "flops_dedup", "per_location", "attention", "vq_distance", "other",
              "quantized_dense", "quantized_dedup", "total_savings", "quantized_ops_savings"):
        assert getattr(rep, f) == getattr(gold, f), f
    assert math.isclose(rep.energy, gold.energy, rel_tol=1e-6)
    wire.emit_table([rep], str(tmp_path))
    ours = (tmp_path / "report.csv").read_text().splitlines()
    theirs = open(os.path.join(HERE, "golden", "report_c1", "report.csv")).read().splitlines()
    assert ours[0] == theirs[0]

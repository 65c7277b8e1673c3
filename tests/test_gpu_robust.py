"""Non-finite weights must not take the device down. The reference's VQ argmin
(proj/src/model.cpp:283-319) starts at index 0 and only moves on a strictly
smaller distance, so a NaN attention row quantises to code 0 and the
evaluation carries on with that code's vector. The GPU paths (the tcgen05
certified argmin's re-scoring queue, the fp32 SIMT argmin, the gradient
engine's argmin) keep that: no out-of-range code, no illegal address, and the
CUDA context stays usable for the next evaluation."""
import numpy as np
import pytest

import paper_2212_11296_b200 as P

pytestmark = pytest.mark.gpu


def _poisoned(w, bf):
    model = P.VqTransformer.init(w.model, w.weight_seed, snap_bf16=bf)
    for p in model.params:
        if p.name == "dec.block0.wq":
            p.value[:, :] = np.nan
    return model


@pytest.mark.parametrize("name", ["c1_4x4", "c3_10x10"])
def test_nan_weights_do_not_fault(port, name):
    w = P.workload(name)
    bf = w.precision == "bf16"
    lat = P.build_lattice("grid2d", (w.L, w.L), periodic=True)
    S = P.zero_sz_samples(w.n_sites, 0, 8, w.sample_seed)
    bad = _poisoned(w, bf)
    eng = P.LocalEnergyEngine(bad, P.HamiltonianModel(lat), precision=w.precision)
    e, lp = eng.local_energies(S, None)
    assert e.shape == (8,) and lp.shape == (8,)
    if not bf:
        # fp32: the same code-0 quantisation as the reference's argmin
        port.set_bf16(False)
        om = port.model(w.model, w.weight_seed)
        for i, p in enumerate(bad.params):
            om.set_param(i, p.value)
        oh = port.hamiltonian("grid_periodic", w.L, w.L)
        ref_e, _, ref_lpsi, _ = om.local_energies(oh, S)
        assert np.allclose(lp, ref_lpsi, rtol=0, atol=1e-6, equal_nan=True)
        assert np.allclose(e, ref_e, rtol=0, atol=1e-5, equal_nan=True)
    # the context survives: a clean model evaluates normally afterwards
    clean = P.VqTransformer.init(w.model, w.weight_seed, snap_bf16=bf)
    eng2 = P.LocalEnergyEngine(clean, P.HamiltonianModel(lat), precision=w.precision)
    e2, lp2 = eng2.local_energies(S, None)
    assert np.all(np.isfinite(e2)) and np.all(np.isfinite(lp2))


def test_nan_weights_gradient_does_not_fault():
    w = P.workload("c1_4x4")
    S = P.zero_sz_samples(w.n_sites, 0, 8, w.sample_seed)
    g = P.LogProbGradient(_poisoned(w, False))
    grads, lp = g.grad(S, np.ones(8))
    assert lp.shape == (8,) and len(grads) == len(g.model.params)

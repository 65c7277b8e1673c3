"""The drop-in boundary exercised from the reference's own C++ types
(oracle/dropin_demo.cpp + include/vqnqs_b200.hpp): the reference builds the
model, Hamiltonian and batch, evaluates local_energy_batch, and the same
objects go through vqnqs_b200::local_energies. Built in the dev container
(where /root/reference exists); the binary travels to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "dropin_demo")


def _have_demo():
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/dropin_demo not built (make -C oracle dropin)")


def test_dropin_refuses_loudly_without_gpu():
    _have_demo()
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    r = subprocess.run([DEMO, "4", "32", "4", "2", "64", "8", "0"], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 3 and "NO_GPU" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("args", [["4", "32", "4", "2", "64", "64", "0"],
                                  ["6", "64", "4", "4", "128", "32", "0"]])
def test_dropin_matches_reference_on_gpu(args):
    _have_demo()
    r = subprocess.run([DEMO, *args], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr

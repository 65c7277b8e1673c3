import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    from oracle import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    return RefLib()


@pytest.fixture(scope="session")
def port():
    from oracle import PortLib, port_available
    if not port_available():
        pytest.skip("oracle/_port not built (make -C oracle port)")
    return PortLib()

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long CPU reference runs")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle, build

    build()
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import RefLib, ref_available

    if not ref_available():
        pytest.skip("reference library oracle/_ref not built (needs /root/reference)")
    return RefLib()


@pytest.fixture(scope="session")
def lib():
    """The product C-ABI library (libpasa_b200.so); loads without a GPU."""
    from paper_2503_01873_b200 import _lib

    return _lib.load()

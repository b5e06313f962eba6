import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running (trajectory) test")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="module")
def oracle_binning():
    """The oracle's SURVEY §8(c) binning mode for the mini-curve runs (protocol, curves, triaxial):
    cell-list pair enumeration, bit-identical to the brute force (tests/test_oracle_pins.py)."""
    import oracle
    oracle.set_binning(True)
    yield
    oracle.set_binning(False)

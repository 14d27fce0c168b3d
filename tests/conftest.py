import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def restatement():
    import oracle
    return oracle.Restatement()


@pytest.fixture(scope="session")
def reference():
    import oracle
    return oracle.Reference()


@pytest.fixture(scope="session")
def wl():
    import paper_1306_4627_b200 as wl
    if wl.device_count() < 1:
        pytest.fail("no CUDA device visible: the library has no CPU fallback")
    return wl

import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpxg.so")
    config.addinivalue_line("markers", "slow: long-running statistical check")


@pytest.fixture(scope="session")
def oracle():
    """The compiled reference (Philox seam) + restated loop. Built by `make -C oracle`."""
    from oracle import oracle as orc
    try:
        orc.lib("philox")
    except orc.OracleUnavailable as e:
        pytest.fail(str(e))
    return orc


@pytest.fixture(scope="session")
def pxg():
    """The product library. On a GPU box a missing .so or device is a failure, not a skip."""
    import paper_2503_23412_b200 as p
    from paper_2503_23412_b200 import _lib
    L = _lib.lib()
    if L.pxg_device_count() <= 0:
        pytest.fail("no CUDA device visible to libpxg")
    return p

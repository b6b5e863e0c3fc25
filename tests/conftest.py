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


_PARITY = {}


@pytest.fixture(scope="session")
def parity_report():
    """Collects the observed parity numbers (mismatch counts, max relative errors) of the GPU
    parity tests and writes them as JSON at the end of the session: $PXG_PARITY_REPORT, or
    gpurun_out/parity_report.json (copied under profiles/ as round evidence)."""
    import json

    def add(section, record):
        _PARITY.setdefault(section, []).append(record)

    yield add
    if _PARITY:
        path = os.environ.get("PXG_PARITY_REPORT") or os.path.join(REPO, "gpurun_out", "parity_report.json")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path, "w") as f:
            json.dump(_PARITY, f, indent=1)

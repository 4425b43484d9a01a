import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running test")
    # The C-ABI library is built in-tree; make sure it is current before any test imports it.
    from paper_2006_02464_b200 import build
    build.build()


def has_gpu() -> bool:
    from paper_2006_02464_b200._lib import lib
    return lib.cw_device_count() > 0


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("GPU test run without a visible CUDA device")
    return 0

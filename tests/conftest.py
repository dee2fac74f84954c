import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: large inputs")


@pytest.fixture(scope="session")
def ctx():
    from paper_2105_00578_b200 import Context
    c = Context(int(os.environ.get("SPB_DEVICE", "0")))
    yield c
    c.close()


@pytest.fixture(scope="session")
def ref():
    from oracle.ref import RefLib
    return RefLib()

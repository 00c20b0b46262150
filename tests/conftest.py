import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsk_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def sk():
    import paper_2605_28274_b200 as sk
    from paper_2605_28274_b200 import build
    build.build()
    if sk.device_count() < 1:
        pytest.fail("no CUDA device visible to libsk_b200.so")
    return sk


@pytest.fixture(scope="session")
def po():
    from oracle import pyoracle
    pyoracle.build()
    return pyoracle


@pytest.fixture(scope="session")
def sk_host():
    """The library for host-only entry points (no device needed)."""
    import paper_2605_28274_b200 as sk
    from paper_2605_28274_b200 import build
    build.build()
    return sk

import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: longer CPU cross-checks")


@pytest.fixture(scope="session")
def oracle():
    from checkers import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from checkers import load_ref
    r = load_ref()
    if r is None:
        pytest.skip("reference checker (oracle/_ref) not available on this machine")
    return r


def golden(name):
    with open(os.path.join(HERE, "golden", name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gold():
    return golden


@pytest.fixture(scope="session")
def engine():
    """The product package on a real B200 (GPU tests only)."""
    import paper_2305_09130_b200 as m
    if m.device_count() < 1:
        pytest.fail("GPU test run without an sm_100 device")
    return m

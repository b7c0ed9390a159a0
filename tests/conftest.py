import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running (minutes)")


@pytest.fixture(scope="session")
def tiny_spec():
    from workload import MODELS
    return MODELS["tiny"]


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Near-tie divergences are reported, never passed
    silently: every one recorded by tests/parity.py is listed here."""
    try:
        from parity import NEAR_TIES
    except ImportError:
        return
    if NEAR_TIES:
        terminalreporter.section("near-tie divergences (T4a)")
        for label, r, t, m in NEAR_TIES:
            terminalreporter.write_line("%s: request %d step %d, oracle top-2 margin %.3g" % (label, r, t, m))

import os
import sys

import pytest

# The suite checks the R41 stale counts against the oracle, so Config.count_stale defaults to True
# here; the product default (flagged targets, no stale count) has its own parity tests
# (tests/test_gpu_active.py) and is what bench.py and smoke() run.
os.environ.setdefault("VINP_COUNT_STALE", "1")
# ... and that default is used from 2^20 targets per level on (libvinp, VINP_ACTIVE_MIN): 0 here, so
# that the small test volumes run it too (read once, when the library first launches a pass)
os.environ.setdefault("VINP_ACTIVE_MIN", "0")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)  # test helpers (_bridge) by plain name; a site package shadows `tests`


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libvinp.so")
    config.addinivalue_line("markers", "slow: slower CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle.oracle as o
    o.build()
    return o

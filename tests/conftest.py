import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long CPU test")


def pytest_collection_modifyitems(config, items):
    # the full-size parity tests (minutes of CPU oracle time at 28 q) run last, so that
    # under -x or a wall-clock limit every shorter GPU test has already reported
    is_heavy = lambda it: "test_gpu_fullsize.py::" in it.nodeid  # noqa: E731
    heavy = [it for it in items if is_heavy(it)]
    if heavy:
        items[:] = [it for it in items if not is_heavy(it)] + heavy


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build_oracle()
    return oracle

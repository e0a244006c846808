import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def cfg_inputs():
    """Cache of generated synthetic inputs keyed by config id."""
    from synth.hypergraph import CONFIGS, make_input
    cache = {}

    def get(i):
        if i not in cache:
            cache[i] = make_input(CONFIGS[i])
        return cache[i]
    return get

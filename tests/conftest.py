import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libcrl.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name):
    """Parse tests/golden/<name>: 'key value  # comment' lines -> {key: float}."""
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, v = line.split()[:2]
            out[k] = float(v)
    return out


@pytest.fixture(scope="session")
def closed_forms():
    return load_golden("closed_forms.txt")

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running parity runs")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def golden_cases(name):
    """Group a flat ``key/field`` npz into {key: {field: array}}."""
    z = load_golden(name)
    out = {}
    for k in z.files:
        case, field = k.rsplit("/", 1)
        out.setdefault(case, {})[field] = z[k]
    return out


@pytest.fixture
def rng():
    return np.random.default_rng(1234)

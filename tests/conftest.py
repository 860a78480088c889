import math
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REPO)

# the paper's Fig. 1 pair (pkg/tests/conftest.py:10-11)
FIG_S = [3.0, 1.0, 4.0, 4.0, 1.0, 1.0]
FIG_T = [1.0, 3.0, 2.0, 1.0, 2.0, 2.0]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libelastik_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


def close(x, y, rel=1e-9):
    if math.isinf(x) or math.isinf(y):
        return math.isinf(x) and math.isinf(y)
    return abs(x - y) <= rel * max(1.0, abs(x), abs(y))


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def spec_from_dict(d, cls=None):
    if cls is None:
        from paper_2102_05221_b200 import DistanceSpec as cls
    return cls(**d)


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)


@pytest.fixture(scope="session")
def gpu():
    import paper_2102_05221_b200 as ekb

    if not ekb.compiled_available():
        pytest.fail("GPU test without a usable CUDA device / libelastik_b200.so (no CPU fallback exists)")
    return ekb

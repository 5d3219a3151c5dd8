import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.fail(f"missing golden fixture {path} (tests/golden/make_golden.py)")
    return np.load(path, allow_pickle=False)


@pytest.fixture(scope="session")
def built_library():
    """Make sure the in-tree .so exists (nvcc cross-compiles without a GPU)."""
    from paper_2405_10050_b200 import _build
    return _build.build()


# Reference test instances (pkg/tests/conftest.py:7-38).
UNIT_SQUARE_POINTS = [(0.0, 0.0), (1.0, 0.0), (-1.0, 0.0), (0.0, 1.0), (0.0, -1.0)]


def config2_rays(k):
    """Canonical config-2 ray recipe; first k rays."""
    s = np.random.default_rng(1).choice(20000, 10000, replace=False)
    p = np.random.default_rng(2).integers(0, 10000, 10 ** 6)[:k]
    u = np.random.default_rng(3).standard_normal((10 ** 6, 6))[:k]
    u = u / np.linalg.norm(u, axis=1, keepdims=True)
    return s, p, u

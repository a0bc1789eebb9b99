import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")

# the 12 x 4 state matrix printed for createStreamsCpu(4) from the default seed
# (reference tests/conftest.py:10-24)
PRINTED_STREAM_MATRIX = np.array([
    [12345, 336690377, 502033783, 739421137],
    [12345, 597094797, 1322587635, 1475938232],
    [12345, 1245771585, 1964121530, 730262207],
    [12345, 85196284, 1949818481, 1630192198],
    [12345, 523477687, 1607232546, 324551134],
    [12345, 2094976052, 1462898381, 795289868],
    [12345, 336690377, 502033783, 739421137],
    [12345, 597094797, 1322587635, 1475938232],
    [12345, 1245771585, 1964121530, 730262207],
    [12345, 85196284, 1949818481, 1630192198],
    [12345, 523477687, 1607232546, 324551134],
    [12345, 2094976052, 1462898381, 795289868],
], dtype=np.int64)

# reference tests/conftest.py:26
SIM_1 = (0.735, 0.842, 0.614, 0.216, 0.110, 0.870, 0.649, 0.170)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


_G = None
_A = None


def golden():
    global _G
    if _G is None:
        with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
            _G = json.load(fh)
    return _G


def golden_arrays():
    global _A
    if _A is None:
        _A = dict(np.load(os.path.join(GOLDEN_DIR, "golden.npz")))
    return _A


@pytest.fixture(scope="session")
def G():
    return golden()


@pytest.fixture(scope="session")
def A():
    return golden_arrays()


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False

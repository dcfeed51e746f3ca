import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(REPO, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) and the built librskel.so")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


_GOLD = None


def golden(name):
    """Arrays of one reference-generated case (tests/golden/make_golden.py)."""
    global _GOLD
    if _GOLD is None:
        _GOLD = np.load(GOLDEN)
    pref = name + "/"
    out = {k[len(pref):]: _GOLD[k] for k in _GOLD.files if k.startswith(pref)}
    if not out:
        raise KeyError(name)
    return out


@pytest.fixture(scope="session")
def gold():
    return golden

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running statistical test")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


@pytest.fixture(scope="session")
def golden():
    return load_golden


class LocfInputs:
    """LOCF input provider (timeseries.py:184-210 semantics) over a table."""

    def __init__(self, times, values):
        self.times = np.asarray(times, dtype=float)
        self.values = np.asarray(values, dtype=float).reshape(len(self.times), -1)

    def at(self, t):
        tol = 1e-9 * max(1.0, abs(t))
        idx = int(np.searchsorted(self.times, t + tol, side="right")) - 1
        return self.values[idx]

    def scalar(self, t):
        return float(self.at(t)[0])

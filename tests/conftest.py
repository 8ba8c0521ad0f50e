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
    if os.environ.get("SSM_GUARD_ALLOC"):
        install_guard_allocator()


def install_guard_allocator():
    """SSM_GUARD_ALLOC=1: every torch CUDA tensor ends at an unmapped guard page
    (tests/tools/guard_alloc.cpp), so an out-of-bounds kernel access faults.
    Must run before the first CUDA allocation of the process."""
    import subprocess

    import torch

    src = os.path.join(ROOT, "tests", "tools", "guard_alloc.cpp")
    so = os.path.join(ROOT, "build", "guard_alloc.so")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(so), exist_ok=True)
        cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
        subprocess.run(["g++", "-O2", "-shared", "-fPIC", src, "-o", so, f"-I{cuda}/include",
                        f"-L{cuda}/lib64/stubs", "-lcuda"], check=True)
    alloc = torch.cuda.memory.CUDAPluggableAllocator(so, "guard_malloc", "guard_free")
    torch.cuda.memory.change_current_allocator(alloc)


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

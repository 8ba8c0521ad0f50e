"""Reentrancy (SURVEY 8b "Threading"): the reference's SMC^2 may call runs from
ThreadPoolExecutor threads (smc.py:60-64).  Filters launched concurrently from
host threads give bitwise the results of the same filters run serially."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_1306_3277_b200 import LORENZ96, RngStream
from paper_1306_3277_b200.inference import build_filter_grid, particle_filter
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu


def _grid():
    g = load_golden("outer.npz")
    times = g["l96/times"]
    return build_filter_grid(0.0, times[-1], 10, times[1:], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)


@pytest.mark.parametrize("noise,P", [("host", 512), ("device", 1 << 15)])
def test_concurrent_filters_equal_serial(noise, P):
    grid = _grid()
    thetas = [np.array([8.5 + 0.5 * k, 0.05 + 0.02 * k]) for k in range(6)]

    def run(k):
        out = particle_filter(LORENZ96, thetas[k], grid, RngStream(90 + k), n_particles=P,
                              resampler="systematic", noise=noise)
        return out.loglik, out.trajectory

    serial = [run(k) for k in range(6)]
    with ThreadPoolExecutor(max_workers=6) as ex:
        par = list(ex.map(run, range(6)))
    for (a, ta), (b, tb) in zip(serial, par):
        assert a == b
        np.testing.assert_array_equal(ta, tb)

"""GPU tests of the outer loops (PMMH, SMC^2) against the reference's own
runs (tests/golden/outer.npz, made by make_golden.gen_outer_loops).

With noise="host" every draw is the reference's (same RngStream keys and
order), so theta sequences and accept decisions must be identical and the
log-likelihoods equal to 1e-12 relative (float64)."""

import numpy as np
import pytest

from paper_1306_3277_b200 import LORENZ96, WINDKESSEL, RngStream
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample, mh_sample_chains, smc_sampler
from tests.conftest import LocfInputs, load_golden

pytestmark = pytest.mark.gpu


def l96_runner(g, P=64, **kw):
    times = g["l96/times"]
    grid = build_filter_grid(0.0, times[-1], 10, times[1:], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)
    return FilterRunner(LORENZ96, grid, n_particles=P, resampler="systematic", **kw)


def test_pmmh_l96_matches_reference():
    g = load_golden("outer.npz")
    chains, acc = mh_sample(LORENZ96, l96_runner(g, noise="host"), 6, RngStream(21))
    assert acc == int(g["l96/mh/accepted"])
    np.testing.assert_array_equal(np.array([c.theta for c in chains]), g["l96/mh/thetas"])
    np.testing.assert_array_equal(np.array([c.init_state for c in chains]), g["l96/mh/inits"])
    np.testing.assert_allclose([c.loglik for c in chains], g["l96/mh/logliks"], rtol=1e-12)
    np.testing.assert_array_equal(chains[-1].trajectory, g["l96/mh/traj_last"])


def test_smc2_l96_matches_reference():
    g = load_golden("outer.npz")
    res = smc_sampler(LORENZ96, l96_runner(g, noise="host"), 6, RngStream(22), theta_resampler="systematic")
    np.testing.assert_array_equal(res.thetas, g["l96/smc/thetas"])
    np.testing.assert_allclose(res.logliks, g["l96/smc/logliks"], rtol=1e-12)
    np.testing.assert_allclose(res.log_v, g["l96/smc/log_v"], rtol=1e-10, atol=1e-12)
    np.testing.assert_array_equal(res.trajectories, g["l96/smc/trajectories"])
    np.testing.assert_allclose([d["ess"] for d in res.diagnostics], g["l96/smc/ess"], rtol=1e-10)
    np.testing.assert_array_equal([d["acceptance"] for d in res.diagnostics], g["l96/smc/acceptance"])


def test_pmmh_windkessel_matches_reference():
    g = load_golden("outer.npz")
    inputs = LocfInputs(g["wk/in_times"], g["wk/in_values"])
    times = np.linspace(0.0, 0.4, 41)
    grid = build_filter_grid(0.0, 0.4, 40, times[1:], g["wk/obs_v"], np.ones((40, 1), bool), n_obs=1)
    runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=128, resampler="systematic", noise="host")
    chains, acc = mh_sample(WINDKESSEL, runner, 6, RngStream(23))
    assert acc == int(g["wk/mh/accepted"])
    np.testing.assert_array_equal(np.array([c.theta for c in chains]), g["wk/mh/thetas"])
    np.testing.assert_allclose([c.loglik for c in chains], g["wk/mh/logliks"], rtol=1e-12)


def test_pmmh_chains_batched_equal_serial():
    g = load_golden("outer.npz")
    runner = l96_runner(g, P=2048)
    rngs = [RngStream(40 + c) for c in range(4)]
    batched, acc = mh_sample_chains(LORENZ96, runner, 5, rngs)
    for c in range(4):
        serial, a = mh_sample(LORENZ96, runner, 5, RngStream(40 + c))
        assert a == acc[c]
        np.testing.assert_array_equal([s.theta for s in serial], [s.theta for s in batched[c]])
        assert [s.loglik for s in serial] == [s.loglik for s in batched[c]]


def test_smc2_device_noise_runs():
    g = load_golden("outer.npz")
    res = smc_sampler(LORENZ96, l96_runner(g, P=1024), 32, RngStream(5), theta_resampler="systematic")
    assert res.thetas.shape == (32, 2)
    assert np.all((res.thetas[:, 0] >= 8.0) & (res.thetas[:, 0] <= 12.0))
    assert np.isclose(np.exp(res.log_v).sum(), 1.0)
    assert res.trajectories.shape == (32, 11, 8)
    assert len(res.diagnostics) == 5

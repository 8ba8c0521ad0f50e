"""Device Kalman filter (ssm_kalman_filter) against the
reference (tests/golden/kalman.npz): windkessel logliks, filtered means and a
smoothing trajectory with the reference's draws (the reference's KalmanRun is
correct for scalar models); the multi-state models (LinOsc, Wide: coupled ode,
inputs, partial masks) against a textbook filter run on the reference's own
extracted systems (the reference's gain is wrong there, see make_golden.dense_kf).
Tolerance: 1e-10 relative on logliks (different but equivalent recursions)."""

import json

import numpy as np
import pytest

from paper_1306_3277_b200 import WINDKESSEL, RngStream
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample, particle_filter
from paper_1306_3277_b200.inference.kalman import advance_kalman_runs, kalman_filter, kalman_runs
from paper_1306_3277_b200.lineargauss import extract_linear_gaussian
from tests.conftest import LocfInputs, load_golden
from tests.test_cpu_kalman import _flow, _lowered

pytestmark = pytest.mark.gpu


def wk_case():
    g = load_golden("kalman.npz")
    in_times = np.round(np.arange(0, 1.0001, 0.01), 10)
    inputs = LocfInputs(in_times, _flow(in_times))
    t = g["wk/times"]
    grid = build_filter_grid(0.0, 0.4, 40, t[1:], g["wk/obs_v"], g["wk/obs_m"], n_obs=1)
    return g, grid, inputs


def osc_case():
    g = load_golden("kalman.npz")
    t = g["osc/times"]
    grid = build_filter_grid(0.0, 3.0, 30, t[1:], g["osc/obs_v"], g["osc/obs_m"], n_obs=2)
    return g, grid, LocfInputs(g["osc/in_times"], g["osc/in_values"]), json.loads(str(g["osc/desc"]))


def test_windkessel_kf_matches_reference():
    g, grid, inputs = wk_case()
    for j in range(2):
        sys_ = extract_linear_gaussian(WINDKESSEL, g["wk/thetas"][j : j + 1], grid.times, inputs)
        res = kalman_filter(sys_, grid, RngStream(40 + j))
        np.testing.assert_allclose(res.loglik, float(g[f"wk/{j}/loglik"]), rtol=1e-12)
        np.testing.assert_allclose([s.mean for s in res.summaries], g[f"wk/{j}/means"], rtol=1e-12)
        np.testing.assert_allclose(res.trajectory, g[f"wk/{j}/traj"], rtol=1e-10)


def test_linosc_and_wide_kf_match_textbook_filter():
    g, grid, inputs, desc = osc_case()
    sys_ = extract_linear_gaussian(desc, g["osc/thetas"], grid.times, inputs)
    runs = kalman_runs(sys_, grid)
    advance_kalman_runs(runs, grid.last)
    for j, r in enumerate(runs):
        np.testing.assert_allclose(r.loglik, float(g[f"osc/{j}/loglik"]), rtol=1e-10)
        np.testing.assert_allclose([r.filtered(i).mean for i in range(grid.last + 1)], g[f"osc/{j}/means"],
                                   rtol=1e-9, atol=1e-12)
    gg = load_golden("generic.npz")
    grid = build_filter_grid(0.0, 2.0, 20, gg["Wide/obs_t"], gg["Wide/obs_v"], gg["Wide/obs_m"], n_obs=12)
    sys_ = extract_linear_gaussian(_lowered("Wide"), g["wide/thetas"], grid.times,
                                   LocfInputs(gg["Wide/in_times"], gg["Wide/in_values"]))
    runs = kalman_runs(sys_, grid)
    advance_kalman_runs(runs, grid.last)
    for j, r in enumerate(runs):
        np.testing.assert_allclose(r.loglik, float(g[f"wide/{j}/loglik"]), rtol=1e-10)
        np.testing.assert_allclose(r.filtered(grid.last).mean, g[f"wide/{j}/means"][-1], rtol=1e-9, atol=1e-12)


def test_resumable_and_clone():
    g, grid, inputs, desc = osc_case()
    sys_ = extract_linear_gaussian(desc, g["osc/thetas"][:1], grid.times, inputs)
    r = kalman_runs(sys_, grid)[0]
    a = r.advance_to(12)
    c = r.clone()
    b = r.advance_to(grid.last)
    b2 = c.advance_to(grid.last)
    assert b == b2
    np.testing.assert_allclose(a + b, float(g["osc/0/loglik"]), rtol=1e-10)
    assert r.advance_to(5) == 0.0  # already past


def test_smoothing_sample_moments():
    """Backward draws: the sample mean and covariance of many trajectories at t0
    match the smoothing distribution from a dense RTS smoother."""
    g, grid, inputs, desc = osc_case()
    sys_ = extract_linear_gaussian(desc, g["osc/thetas"][:1], grid.times, inputs)
    r = kalman_runs(sys_, grid)[0]
    r.advance_to(grid.last)
    draws = np.array([r.sample_trajectory(RngStream(1000 + k)) for k in range(4000)])
    mu, P, mu_p, P_p = r._records()
    A = sys_.A[0]
    ms, Ps = mu[-1], P[-1]
    for i in range(grid.last - 1, -1, -1):  # Rauch-Tung-Striebel
        J = P[i] @ A[i].T @ np.linalg.inv(P_p[i + 1])
        ms = mu[i] + J @ (ms - mu_p[i + 1])
        Ps = P[i] + J @ (Ps - P_p[i + 1]) @ J.T
    m = draws[:, 0].mean(axis=0)
    se = np.sqrt(np.diag(Ps) / len(draws))
    assert np.all(np.abs(m - ms) < 5 * se), (m, ms, se)
    np.testing.assert_allclose(np.cov(draws[:, 0].T), Ps, rtol=0.15, atol=1e-3)


def test_pmmh_kalman_windkessel_matches_reference():
    g, grid, inputs = wk_case()
    runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, filter_kind="kalman")
    chains, acc = mh_sample(WINDKESSEL, runner, 8, RngStream(24))
    assert acc == int(g["wk/mh/accepted"])
    np.testing.assert_array_equal([c.theta for c in chains], g["wk/mh/thetas"])
    np.testing.assert_allclose([c.loglik for c in chains], g["wk/mh/logliks"], rtol=1e-12)


def test_particle_filter_unbiased_vs_kalman_linosc():
    """The bootstrap filter's likelihood estimate is unbiased for exp(loglik):
    the device PF on the generic LinOsc model averages to the device KF."""
    from paper_1306_3277_b200 import generic

    g, grid, inputs, desc = osc_case()
    theta = g["osc/thetas"][0]
    kf = extract_linear_gaussian(desc, theta[None], grid.times, inputs)
    r = kalman_runs(kf, grid)[0]
    r.advance_to(grid.last)
    model = generic.from_description(desc)
    lls = np.array([particle_filter(model, theta, grid, RngStream(500 + k), inputs=inputs, n_particles=1 << 14,
                                    resampler="systematic").loglik for k in range(24)])
    m = np.log(np.mean(np.exp(lls - lls.max()))) + lls.max()
    se = lls.std(ddof=1) / np.sqrt(len(lls))
    assert abs(m - r.loglik) < 5 * se + 0.02, (m, r.loglik, se)


def test_smc2_kalman_windkessel_matches_reference():
    from paper_1306_3277_b200.inference import smc_sampler

    g, grid, inputs = wk_case()
    runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, filter_kind="kalman")
    res = smc_sampler(WINDKESSEL, runner, 6, RngStream(25), theta_resampler="systematic")
    np.testing.assert_array_equal(res.thetas, g["wk/smc/thetas"])
    np.testing.assert_allclose(res.logliks, g["wk/smc/logliks"], rtol=1e-12)
    np.testing.assert_allclose(res.log_v, g["wk/smc/log_v"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(res.trajectories, g["wk/smc/trajectories"], rtol=1e-10)


@pytest.mark.parametrize("case", ["osc", "wk"])
def test_device_backward_sampling_equals_host(case):
    """ssm_kalman_sample (device, one thread per run) against the host
    restatements of kalman.py:98-114 (batched and serial), same draws: equal to
    the rounding of the covariance-form algebra."""
    from paper_1306_3277_b200.inference.kalman import _sample_kalman_trajectories_host, sample_kalman_trajectories

    if case == "osc":
        g, grid, inputs, desc = osc_case()
        sys_ = extract_linear_gaussian(desc, g["osc/thetas"], grid.times, inputs)
        upto = 17
    else:
        g, grid, inputs = wk_case()
        thetas = np.array([1.8, 3.0, 0.06, 25.0]) * np.random.default_rng(3).uniform(0.8, 1.2, size=(40, 4))
        sys_ = extract_linear_gaussian(WINDKESSEL, thetas, grid.times, inputs)
        upto = grid.last
    runs = kalman_runs(sys_, grid)
    advance_kalman_runs(runs, upto)
    got = sample_kalman_trajectories(runs, [RngStream(70 + k) for k in range(len(runs))])
    host = _sample_kalman_trajectories_host(runs, [RngStream(70 + k) for k in range(len(runs))])
    for k, r in enumerate(runs):
        scale = max(1.0, float(np.max(np.abs(host[k]))))
        assert np.max(np.abs(got[k] - host[k])) <= 1e-10 * scale, (k, np.max(np.abs(got[k] - host[k])))
        serial = r._sample_trajectory_serial(RngStream(70 + k))
        assert np.max(np.abs(got[k] - serial)) <= 1e-10 * scale

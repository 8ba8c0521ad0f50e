"""Statistical validation of the device-noise path -- the path the benchmark
times (-m gpu).  Its draws (Philox4x32-10 + float32 Box-Muller, ssm_common.cuh)
are not numpy's, so agreement with the reference is in law, within Monte
Carlo error (north star):

  * the device standard normals themselves: moments, Kolmogorov-Smirnov,
    tail mass beyond 4 and 5 sigma, the documented truncation at 6.77 sigma
    (u1 >= 2^-33), cross-slot / lag / cross-step correlations;
  * L96 filter log-likelihood estimates (benchmark data, 2^14 particles,
    systematic and the default multinomial) against the reference's own
    estimates on the same data (tests/golden/stat.npz, make_stat_golden.py);
  * windkessel PMMH posterior means (config 3's model, 2^12-particle filters,
    200 MH steps, device theta-level draws) against 8 reference chains;
  * L96 SMC^2 posterior means (64 theta x 2^12) against 8 reference runs.
Every comparison is |mean_dev - mean_ref| <= 4 sqrt(se_dev^2 + se_ref^2) with
standard errors from independent seeds / chains / replicate runs.
"""

import math

import numpy as np
import pytest
from scipy import stats

from paper_1306_3277_b200 import LORENZ96, WINDKESSEL, RngStream, _lib
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample_chains, smc_sampler
from tests.conftest import LocfInputs, load_golden
from tests.device_draws import device_normals

pytestmark = pytest.mark.gpu


def _agree(dev, ref, k=4.0):
    dev, ref = np.asarray(dev, float), np.asarray(ref, float)
    se = math.sqrt(dev.var(ddof=1) / dev.shape[0] + ref.var(ddof=1) / ref.shape[0])
    return abs(dev.mean() - ref.mean()), k * se


# ------------------------------------------------------------------ the generator


@pytest.fixture(scope="module")
def l96_normals():
    z = device_normals(_lib.SSM_MODEL_LORENZ96, (0x1234567, 0x89ABCDEF), 1 << 20, 3, 0)  # (8, 2^20)
    return z


def test_device_normals_moments_and_ks(l96_normals):
    z = l96_normals.reshape(-1)
    N = z.size
    assert abs(z.mean()) < 4 / math.sqrt(N)
    assert abs(z.var() - 1.0) < 4 * math.sqrt(2.0 / N)
    assert abs(stats.skew(z)) < 4 * math.sqrt(6.0 / N)
    assert abs(stats.kurtosis(z)) < 4 * math.sqrt(24.0 / N)
    ks = stats.kstest(z, "norm")
    assert ks.pvalue > 1e-4, ks
    for n in range(8):  # every slot on its own
        assert stats.kstest(l96_normals[n], "norm").pvalue > 1e-4


def test_device_normals_tails_and_truncation(l96_normals):
    z = np.abs(l96_normals.reshape(-1))
    N = z.size
    for c in (3.0, 4.0, 5.0):
        p = 2 * stats.norm.sf(c)
        cnt = int(np.sum(z > c))
        assert abs(cnt - N * p) <= 4 * math.sqrt(N * p) + 2, (c, cnt, N * p)
    # u1 = (a + 1/2) 2^-32 >= 2^-33: |z| <= sqrt(-2 ln 2^-33) = 6.77 (documented in the bench config)
    assert z.max() <= math.sqrt(-2 * math.log(2.0**-33)) + 1e-3


def test_device_normals_independence(l96_normals):
    z = l96_normals
    n = z.shape[1]
    lim = 4 / math.sqrt(n)
    c = np.corrcoef(z)
    assert np.max(np.abs(c - np.eye(8))) < lim  # across slots (one Philox block feeds 4)
    for lag in (1, 32, 256):  # across particles (counter neighbours, warp / block strides)
        assert abs(np.corrcoef(z[0, :-lag], z[0, lag:])[0, 1]) < lim
    z4 = device_normals(_lib.SSM_MODEL_LORENZ96, (0x1234567, 0x89ABCDEF), 1 << 20, 4, 0)
    z3s1 = device_normals(_lib.SSM_MODEL_LORENZ96, (0x1234567, 0x89ABCDEF), 1 << 20, 3, 1)
    for other in (z4, z3s1):  # across grid steps and sub-steps
        assert abs(np.corrcoef(z[0], other[0])[0, 1]) < lim
    # windkessel's single normal per particle and sub-step
    w = device_normals(_lib.SSM_MODEL_WINDKESSEL, (7, 8), 1 << 22, 5, 0)
    assert abs(w.mean()) < 4 / math.sqrt(w.size) and abs(w.var() - 1) < 4 * math.sqrt(2.0 / w.size)
    assert stats.kstest(w, "norm").pvalue > 1e-4


# ------------------------------------------------------------------ filters and outer loops


def _l96_bench_grid():
    from oracle import ssm_oracle as O

    theta = np.array([10.0, 0.1])
    times = np.linspace(0.0, 2.0, 41)
    obs = O.simulate_l96(theta, times, O.Stream(1))
    ov = np.array([obs[k][0] for k in range(1, 41)])
    om = np.array([obs[k][1] for k in range(1, 41)])
    return theta, build_filter_grid(0.0, 2.0, 40, times[1:], ov, om, n_obs=8)


@pytest.mark.parametrize("scheme", ["systematic", "multinomial"])
def test_l96_device_noise_loglik_matches_reference_in_law(scheme):
    """64 reference filter runs vs 256 device runs, same data and size."""
    g = load_golden("stat.npz")
    P, T = int(g["sizes"][0]), int(g["sizes"][1])
    theta, grid = _l96_bench_grid()
    runner = FilterRunner(LORENZ96, grid, n_particles=P, resampler=scheme)
    B = 256
    res = runner.run_batch([theta] * B, [None] * B, [RngStream(5000 + s) for s in range(B)], upto=T)
    dev = np.array([r[0] for r in res])
    ref = g[f"l96_pf/{scheme}/loglik"]
    d, tol = _agree(dev, ref)
    assert d <= tol, (dev.mean(), ref.mean(), tol)
    # same spread too (the device multinomial is the sorted order-statistics draw)
    f = dev.var(ddof=1) / ref.var(ddof=1)
    assert stats.f.cdf(f, B - 1, ref.size - 1) > 1e-4 and stats.f.sf(f, B - 1, ref.size - 1) > 1e-4, f


def test_windkessel_pmmh_posterior_matches_reference():
    """Config 3's sampler (PMMH on the windkessel, device filters and device
    theta-level draws) against the reference's PMMH: posterior means of
    (R, C, Z, log sigma2) after 50 burn-in steps, chains independent."""
    g = load_golden("stat.npz")
    gp = load_golden("pf.npz")
    _, _, _, P, n_chains, n_mh, *_ = (int(v) for v in g["sizes"])
    inputs = LocfInputs(gp["wk/in_times"], gp["wk/in_values"])
    grid = build_filter_grid(0.0, 1.0, 100, np.linspace(0, 1, 101)[1:], gp["wk/obs_v"], np.ones((100, 1), bool),
                             n_obs=1)
    runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=P, resampler="multinomial")
    C = 32
    chains, acc = mh_sample_chains(WINDKESSEL, runner, n_mh, [RngStream(9000 + c) for c in range(C)],
                                   theta_draws="device")
    # sigma2's posterior is heavy-tailed on these data (chains wander to 1e9, Windkessel.bi:37-40
    # inverse-gamma prior): its mean is compared on the log scale
    summ = lambda th: np.concatenate([th[..., :3], np.log(th[..., 3:])], axis=-1)  # noqa: E731
    dev = summ(np.array([[s.theta for s in ch] for ch in chains]))[:, 50:].mean(axis=1)  # (C, 4) chain means
    ref = summ(g["wk_pmmh/thetas"])[:, 50:].mean(axis=1)
    for k in range(4):
        d, tol = _agree(dev[:, k], ref[:, k])
        assert d <= tol, (k, dev[:, k].mean(), ref[:, k].mean(), tol)
    ra = g["wk_pmmh/accepted"] / n_mh
    da = np.asarray(acc) / n_mh
    d, tol = _agree(da, ra)
    assert d <= tol, (da.mean(), ra.mean())


def test_l96_smc2_posterior_matches_reference():
    """Config 4's sampler (SMC^2 with device filters, systematic at both
    levels) against 8 reference SMC^2 runs: weighted posterior means of
    (F, sigma2) over independent replicate runs."""
    g = load_golden("stat.npz")
    *_, P, n_theta, _ = (int(v) for v in g["sizes"])
    grid = build_filter_grid(0.0, 1.0, 20, g["l96_sparse/obs_t"], g["l96_sparse/obs_v"], g["l96_sparse/obs_m"],
                             n_obs=8)
    runner = FilterRunner(LORENZ96, grid, n_particles=P, resampler="systematic")
    means = []
    for r in range(16):
        res = smc_sampler(LORENZ96, runner, n_theta, RngStream(700 + r), theta_resampler="systematic",
                          theta_draws="device")
        w = np.exp(res.log_v - res.log_v.max())
        means.append((w / w.sum()) @ res.thetas)
    dev = np.array(means)
    ref = g["l96_smc2/post_mean"]
    for k in range(2):
        d, tol = _agree(dev[:, k], ref[:, k])
        assert d <= tol, (k, dev[:, k].mean(), ref[:, k].mean(), tol)

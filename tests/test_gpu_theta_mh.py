"""Device theta-level MH (theta_mh.py) against the reference.

draws="host" injects the reference's own draws: theta sequences, accept
decisions and log-likelihoods must match the reference runs in
tests/golden/outer.npz up to the normcdf / normcdfinv rounding of the
truncated-Gaussian sampler (theta to 1e-13 relative; logliks of filters run at
those thetas to 1e-10).  draws="device" is checked by distribution against the
host sampler and by re-evaluating its densities with the host formulas."""

import numpy as np
import pytest
from scipy import stats

from paper_1306_3277_b200 import LORENZ96, WINDKESSEL, RngStream
from paper_1306_3277_b200.errors import DistributionParameterError
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample_chains, smc_sampler
from paper_1306_3277_b200.inference.mcmc import MhChainState
from paper_1306_3277_b200.inference.theta_mh import DeviceThetaChains
from paper_1306_3277_b200.models import parameter_logpdf_batch, propose_batch
from tests.conftest import LocfInputs, load_golden

pytestmark = pytest.mark.gpu


def l96_runner(g, P=64, **kw):
    times = g["l96/times"]
    grid = build_filter_grid(0.0, times[-1], 10, times[1:], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)
    return FilterRunner(LORENZ96, grid, n_particles=P, resampler="systematic", **kw)


def wk_runner(g, P=128, **kw):
    inputs = LocfInputs(g["wk/in_times"], g["wk/in_values"])
    times = np.linspace(0.0, 0.4, 41)
    grid = build_filter_grid(0.0, 0.4, 40, times[1:], g["wk/obs_v"], np.ones((40, 1), bool), n_obs=1)
    return FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=P, resampler="systematic", **kw)


def test_pmmh_l96_host_draws_match_reference():
    g = load_golden("outer.npz")
    chains, acc = mh_sample_chains(LORENZ96, l96_runner(g, noise="host"), 6, [RngStream(21)], theta_draws="host")
    chains = chains[0]
    assert int(acc[0]) == int(g["l96/mh/accepted"])
    np.testing.assert_allclose(np.array([c.theta for c in chains]), g["l96/mh/thetas"], rtol=1e-13)
    np.testing.assert_allclose(np.array([c.init_state for c in chains]), g["l96/mh/inits"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose([c.loglik for c in chains], g["l96/mh/logliks"], rtol=1e-10)


def test_pmmh_windkessel_host_draws_match_reference():
    g = load_golden("outer.npz")
    chains, acc = mh_sample_chains(WINDKESSEL, wk_runner(g, noise="host"), 6, [RngStream(23)], theta_draws="host")
    chains = chains[0]
    assert int(acc[0]) == int(g["wk/mh/accepted"])
    np.testing.assert_allclose(np.array([c.theta for c in chains]), g["wk/mh/thetas"], rtol=1e-13)
    np.testing.assert_allclose([c.loglik for c in chains], g["wk/mh/logliks"], rtol=1e-10)


def test_smc2_l96_host_draws_match_reference():
    g = load_golden("outer.npz")
    res = smc_sampler(LORENZ96, l96_runner(g, noise="host"), 6, RngStream(22), theta_resampler="systematic",
                      theta_draws="host")
    np.testing.assert_allclose(res.thetas, g["l96/smc/thetas"], rtol=1e-13)
    np.testing.assert_allclose(res.logliks, g["l96/smc/logliks"], rtol=1e-10)
    np.testing.assert_allclose(res.log_v, g["l96/smc/log_v"], rtol=1e-8, atol=1e-10)
    np.testing.assert_array_equal([d["acceptance"] for d in res.diagnostics], g["l96/smc/acceptance"])


def _states(spec, C, seed, with_init):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(C):
        if spec is LORENZ96:
            th = np.array([rng.uniform(8.2, 11.8), rng.uniform(0.05, 0.5)])
        else:
            th = np.array([rng.uniform(0.5, 3), rng.uniform(0.5, 5), rng.uniform(0.01, 0.1), rng.uniform(5, 50)])
        x0 = rng.uniform(-0.9, 2.9, size=8) if with_init else None
        lp = float(parameter_logpdf_batch(spec, th[None])[0])
        out.append(MhChainState(theta=th, trajectory=None, loglik=rng.normal(-50, 5), log_prior=lp, init_state=x0))
    return out


@pytest.mark.parametrize("spec,with_init", [(LORENZ96, True), (LORENZ96, False), (WINDKESSEL, False)])
def test_propose_host_draws_equal_host_blocks(spec, with_init):
    C = 257
    states = _states(spec, C, 3, with_init)
    rngs = [RngStream(900 + c).child(1) for c in range(C)]
    dev = DeviceThetaChains(spec, states)
    th, x0, lq_f, lq_r, lp = dev.propose(rngs, 1, draws="host")
    rngs = [RngStream(900 + c).child(1) for c in range(C)]
    h_th, h_x0, h_f, h_r, h_lp = propose_batch(spec, [s.theta for s in states],
                                               [s.init_state for s in states] if with_init else None, rngs)
    np.testing.assert_allclose(th, h_th, rtol=1e-13)
    if with_init:
        np.testing.assert_allclose(x0, np.array(h_x0), rtol=1e-13, atol=1e-14)
    fin = np.isfinite(h_lp)
    np.testing.assert_array_equal(np.isfinite(lp), fin)
    for a, b in ((lq_f, h_f), (lq_r, h_r), (lp, h_lp)):
        np.testing.assert_allclose(a[fin], b[fin], rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("spec", [LORENZ96, WINDKESSEL])
def test_propose_device_draws_distribution_and_densities(spec):
    C = 4096
    states = _states(spec, 1, 5, spec is LORENZ96) * C  # every chain at the same point
    dev = DeviceThetaChains(spec, states)
    th, x0, lq_f, lq_r, lp = dev.propose([RngStream(77).child(c) for c in range(C)], 3, draws="device")
    rngs = [RngStream(78).child(c) for c in range(C)]
    h_th, h_x0, *_ = propose_batch(spec, [s.theta for s in states],
                                   [s.init_state for s in states] if spec is LORENZ96 else None, rngs)
    for k in range(spec.n_param):
        assert stats.ks_2samp(th[:, k], h_th[:, k]).pvalue > 1e-4, k
    if x0 is not None:
        assert stats.ks_2samp(x0[:, 0], np.array(h_x0)[:, 0]).pvalue > 1e-4
    # the device densities of its own draws equal the host formulas
    inits = [s.init_state for s in states] if x0 is not None else None
    ref = propose_batch.__globals__
    lqf = np.zeros(C)
    lqr = np.zeros(C)
    t0 = states[0].theta
    tg = [(0, 0.1, 8.0, 12.0)] if spec is LORENZ96 else [(0, 0.03, 0.0, np.inf), (1, 0.1, 0.0, np.inf),
                                                          (2, 0.002, 0.0, np.inf)]
    for slot, sd, lo, hi in tg:
        lqf += ref["_tg_logpdf"](th[:, slot], t0[slot], sd, lo, hi)
        lqr += ref["_tg_logpdf"](t0[slot], th[:, slot], sd, lo, hi)
    ig = spec.n_param - 1
    lqf += ref["d_invgamma_logpdf"](th[:, ig], 2.0, 3.0 * t0[ig])
    lqr += ref["d_invgamma_logpdf"](t0[ig], 2.0, 3.0 * th[:, ig])
    if inits is not None:
        x_old = np.array(inits)
        lqf = lqf + ref["_tg_logpdf"](x0, x_old, 0.1, -1.0, 3.0).sum(axis=1)
        lqr = lqr + ref["_tg_logpdf"](x_old, x0, 0.1, -1.0, 3.0).sum(axis=1)
    np.testing.assert_allclose(lq_f, lqf, rtol=1e-11, atol=1e-10)
    np.testing.assert_allclose(lq_r, lqr, rtol=1e-11, atol=1e-10)
    h_lp = parameter_logpdf_batch(spec, th)
    if x0 is not None:
        h_lp = h_lp + np.where(np.all((x0 >= -1) & (x0 <= 3), axis=1), -8 * np.log(4.0), -np.inf)
    np.testing.assert_allclose(lp, h_lp, rtol=1e-12, atol=1e-12)


def test_accept_matches_metropolis_rule():
    C = 1000
    states = _states(WINDKESSEL, C, 9, False)
    dev = DeviceThetaChains(WINDKESSEL, states)
    rngs = [RngStream(300 + c) for c in range(C)]
    th, _, lq_f, lq_r, lp = dev.propose(rngs, 1, draws="host")
    ua = dev._inj[2].cpu().numpy()
    ll_new = np.random.default_rng(4).normal(-50, 5, size=C)
    ll_new[::7] = -np.inf
    ll_new[::11] = np.nan
    ok = dev.accept(ll_new, 1)
    cur_ll = np.array([s.loglik for s in states])
    cur_lp = np.array([s.log_prior for s in states])
    with np.errstate(invalid="ignore"):
        r = (ll_new + lp + lq_r) - (cur_ll + cur_lp + lq_f)
        want = np.where(np.isnan(r) | (r == -np.inf), False, ua <= np.exp(np.minimum(r, 0.0)))
    want &= lp != -np.inf
    np.testing.assert_array_equal(ok, want)
    assert 0 < ok.sum() < C
    np.testing.assert_array_equal(dev.theta.cpu().numpy()[ok], th[ok])
    np.testing.assert_array_equal(dev.loglik.cpu().numpy()[ok], ll_new[ok])
    np.testing.assert_array_equal(dev.theta.cpu().numpy()[~ok], np.array([s.theta for s in states])[~ok])


def test_device_draws_pmmh_runs_and_mixes():
    g = load_golden("outer.npz")
    runner = wk_runner(g, P=1024)
    chains, acc = mh_sample_chains(WINDKESSEL, runner, 20, [RngStream(60 + c) for c in range(8)],
                                   theta_draws="device")
    assert len(chains) == 8 and all(len(c) == 20 for c in chains)
    assert 0 < acc.sum() < 8 * 20
    th = np.array([[s.theta for s in c] for c in chains])
    assert np.all(th > 0)
    # the same chains again: device draws are a pure function of the streams
    chains2, acc2 = mh_sample_chains(WINDKESSEL, runner, 20, [RngStream(60 + c) for c in range(8)],
                                     theta_draws="device")
    np.testing.assert_array_equal(acc, acc2)
    np.testing.assert_array_equal(th, np.array([[s.theta for s in c] for c in chains2]))


def test_invalid_parameter_raises():
    states = _states(WINDKESSEL, 4, 1, False)
    states[2].theta[3] = -1.0  # inverse-gamma scale 3*sigma2 < 0
    dev = DeviceThetaChains(WINDKESSEL, states)
    with pytest.raises(DistributionParameterError):
        dev.propose([RngStream(c) for c in range(4)], 1, draws="device")

"""Device theta-level blocks of GENERATED models (codegen `struct Theta`,
ssm_gen_theta_propose; SURVEY 8f row 1 for generic models).

draws="host": the device walk runs on the reference's own standard variates
(recorded from each chain's stream while the reference walk runs), so the
proposal, both proposal densities and the prior equal the host blocks up to
CUDA's log / lgamma / normcdf / normcdfinv (theta to 1e-13; densities 1e-11),
and PMMH / SMC^2 runs reproduce the reference's goldens.  draws="device":
the proposal law against the host sampler (KS), and the device's densities
of its own draws against the host formulas."""

import json
import os

import numpy as np
import pytest
from scipy import stats

from paper_1306_3277_b200 import RngStream, generic
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample_chains, smc_sampler
from paper_1306_3277_b200.inference.mcmc import MhChainState
from paper_1306_3277_b200.inference.theta_mh import DeviceThetaChains
from tests.conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "gen_models.json")) as fh:
    FIX = json.load(fh)


def model(name):
    d = dict(FIX["lowered"][name])
    d.pop("fingerprint", None)
    return generic.from_description(d)


def _grid(g, name, m):
    T = len(g[f"{name}/times"]) - 1
    return build_filter_grid(0.0, float(g[f"{name}/times"][-1]), T, g[f"{name}/obs_t"], g[f"{name}/obs_v"],
                             g[f"{name}/obs_m"], n_obs=m.n_obs)


def _states(m, C, seed, with_init):
    th = m.sample_parameter(RngStream(seed), size=C)
    x0 = m.sample_initial(th, RngStream(seed + 1)) if with_init else None
    rng = np.random.default_rng(seed)
    return [MhChainState(theta=th[c].copy(), trajectory=None, loglik=float(rng.normal(-50, 5)),
                         log_prior=m.parameter_logpdf(th[c]), init_state=None if x0 is None else x0[c].copy())
            for c in range(C)]


CASES = [("StochVol", False), ("PredatorPrey", False), ("Lorenz96", True), ("Lorenz96", False), ("Wide", False)]


@pytest.mark.parametrize("name,with_init", CASES)
def test_generic_propose_host_draws_equal_host_blocks(name, with_init):
    m = model(name)
    C = 193
    states = _states(m, C, 5, with_init)
    dev = DeviceThetaChains(m, states)
    th, x0, lq_f, lq_r, lp = dev.propose([RngStream(700 + c).child(2) for c in range(C)], 2, draws="host")
    h_th, h_x0, h_f, h_r, h_lp = m.propose_batch([s.theta for s in states],
                                                 [s.init_state for s in states] if with_init else None,
                                                 [RngStream(700 + c).child(2) for c in range(C)])
    np.testing.assert_allclose(th, h_th, rtol=1e-13, atol=1e-15)
    if with_init:
        np.testing.assert_allclose(x0, np.array(h_x0), rtol=1e-13, atol=1e-14)
    fin = np.isfinite(h_lp)
    np.testing.assert_array_equal(np.isfinite(lp), fin)
    assert fin.any()
    for a, b in ((lq_f, h_f), (lq_r, h_r), (lp, h_lp)):
        np.testing.assert_allclose(a[fin], b[fin], rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("name", ["StochVol", "PredatorPrey"])
def test_generic_pmmh_and_smc2_device_theta_match_reference(name):
    """The generic goldens (reference runs, tests/golden/generic.npz) with the
    theta-level blocks on the device and the reference's draws injected."""
    g = load_golden("generic.npz")
    m = model(name)
    runner = FilterRunner(m, _grid(g, name, m), n_particles=64, resampler="systematic", noise="host")
    chains, acc = mh_sample_chains(m, runner, 5, [RngStream(31)], theta_draws="host")
    assert int(acc[0]) == int(g[f"{name}/mh/accepted"])
    np.testing.assert_allclose(np.array([c.theta for c in chains[0]]), g[f"{name}/mh/thetas"], rtol=1e-12)
    np.testing.assert_allclose([c.loglik for c in chains[0]], g[f"{name}/mh/logliks"], rtol=1e-9)
    res = smc_sampler(m, runner, 6, RngStream(32), theta_resampler="systematic", theta_draws="host")
    np.testing.assert_allclose(res.thetas, g[f"{name}/smc/thetas"], rtol=1e-12)
    np.testing.assert_allclose(res.logliks, g[f"{name}/smc/logliks"], rtol=1e-9)
    np.testing.assert_allclose(res.log_v, g[f"{name}/smc/log_v"], rtol=1e-8, atol=1e-10)


def test_generic_l96_pmmh_with_initial_proposals_device_theta_matches_reference():
    """proposal_initial through the generated walk (x0 jointly with theta)."""
    g = load_golden("outer.npz")
    times = g["l96/times"]
    grid = build_filter_grid(0.0, times[-1], 10, times[1:], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)
    m = model("Lorenz96")
    runner = FilterRunner(m, grid, n_particles=64, resampler="systematic", noise="host")
    chains, acc = mh_sample_chains(m, runner, 6, [RngStream(21)], theta_draws="host")
    assert int(acc[0]) == int(g["l96/mh/accepted"])
    np.testing.assert_allclose(np.array([c.theta for c in chains[0]]), g["l96/mh/thetas"], rtol=1e-13)
    np.testing.assert_allclose(np.array([c.init_state for c in chains[0]]), g["l96/mh/inits"], rtol=1e-13,
                               atol=1e-15)
    np.testing.assert_allclose([c.loglik for c in chains[0]], g["l96/mh/logliks"], rtol=1e-10)


@pytest.mark.parametrize("name,with_init", [("StochVol", False), ("PredatorPrey", False), ("Lorenz96", True)])
def test_generic_propose_device_draws_distribution_and_densities(name, with_init):
    m = model(name)
    C = 4096
    states = _states(m, 1, 9, with_init) * C  # every chain at the same point
    dev = DeviceThetaChains(m, states)
    th, x0, lq_f, lq_r, lp = dev.propose([RngStream(81).child(c) for c in range(C)], 4, draws="device")
    h_th, h_x0, *_ = m.propose_batch([s.theta for s in states], [s.init_state for s in states] if with_init else None,
                                     [RngStream(82).child(c) for c in range(C)])
    for k in range(m.n_param):
        assert stats.ks_2samp(th[:, k], h_th[:, k]).pvalue > 1e-4, k
    if with_init:
        assert stats.ks_2samp(x0[:, 0], np.array(h_x0)[:, 0]).pvalue > 1e-4
    # the device densities of its own draws are the host formulas (first 256 chains)
    t0, i0 = states[0].theta, states[0].init_state
    for c in range(256):
        f = m.proposal_parameter_logpdf(t0, th[c])
        r = m.proposal_parameter_logpdf(th[c], t0)
        p = m.parameter_logpdf(th[c])
        if with_init:
            f += m.proposal_initial_logpdf(th[c], i0, x0[c])
            r += m.proposal_initial_logpdf(t0, x0[c], i0)
            p += m.initial_logpdf(th[c], x0[c])
        np.testing.assert_allclose([lq_f[c], lq_r[c], lp[c]], [f, r, p], rtol=1e-11, atol=1e-11)


def test_generic_device_draws_pmmh_reproducible():
    g = load_golden("generic.npz")
    m = model("StochVol")
    runner = FilterRunner(m, _grid(g, "StochVol", m), n_particles=256, resampler="systematic")
    rngs = [RngStream(90 + c) for c in range(6)]
    a, acc_a = mh_sample_chains(m, runner, 8, rngs, theta_draws="device")
    b, acc_b = mh_sample_chains(m, runner, 8, [RngStream(90 + c) for c in range(6)], theta_draws="device")
    np.testing.assert_array_equal(acc_a, acc_b)
    np.testing.assert_array_equal(np.array([[s.theta for s in c] for c in a]), np.array([[s.theta for s in c] for c in b]))
    assert 0 < acc_a.sum() < 6 * 8

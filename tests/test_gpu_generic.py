"""Generic-model path on the GPU: models lowered from the
reference IR (tests/golden/gen_models.json) and compiled with NVRTC, run
through the reference's own entry points.

  - Lorenz '96 through the generic kernel with the reference's draws
    (noise="host", exact): bitwise the reference (states, ancestors,
    trajectory), log-likelihood within 1e-12 -- the same bar as the
    hand-written kernel;
  - Windkessel: np.exp vs the device exp (neither correctly rounded): 1e-12;
  - StochVol / PredatorPrey (tests/models/*.bi, not hand-written anywhere):
    reference PF runs with host draws; sin / pow / mod / log / normcdf /
    lgamma differ from numpy/scipy at the ulp level, so states and
    log-likelihoods within 1e-9 and ancestors equal;
  - device noise: the generic L96 filter agrees statistically with the
    hand-written one, and the generic Windkessel filter is unbiased against
    the reference's Kalman likelihood.
"""

import json
import os

import numpy as np
import pytest

from paper_1306_3277_b200 import LORENZ96, RngStream, generic
from paper_1306_3277_b200 import simulate as S
from paper_1306_3277_b200.errors import DistributionParameterError
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, particle_filter
from tests.conftest import GOLDEN, LocfInputs, load_golden

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "gen_models.json")) as fh:
    FIX = json.load(fh)


def model(name):
    d = dict(FIX["lowered"][name])
    d.pop("fingerprint", None)
    return generic.from_description(d)


def normwise(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


def _l96_grid(g):
    return build_filter_grid(0.0, 2.0, 20, g["l96/obs_t"], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)


def _anc(out):
    return np.array([h[1].cpu().numpy() for h in out.run.history[1:] if h[1] is not None])


@pytest.mark.parametrize("scheme", ["systematic", "multinomial", "stratified"])
def test_generic_l96_host_noise_bitwise_reference(scheme):
    g = load_golden("pf.npz")
    out = particle_filter(model("Lorenz96"), g["l96/theta"], _l96_grid(g), RngStream(7), n_particles=256,
                          resampler=scheme, noise="host")
    ref = float(g[f"l96/{scheme}/loglik"])
    assert abs(out.loglik - ref) <= 1e-12 * abs(ref)
    np.testing.assert_array_equal(out.run.x, g[f"l96/{scheme}/x_final"])
    np.testing.assert_array_equal(out.trajectory, g[f"l96/{scheme}/traj"])
    np.testing.assert_array_equal(_anc(out), g[f"l96/{scheme}/anc"][1:])


@pytest.mark.parametrize("scheme", ["multinomial", "systematic"])
def test_generic_windkessel_host_noise_matches_reference(scheme):
    g = load_golden("pf.npz")
    inputs = LocfInputs(g["wk/in_times"], g["wk/in_values"])
    grid = build_filter_grid(0.0, 1.0, 100, np.linspace(0, 1, 101)[1:], g["wk/obs_v"], np.ones((100, 1), bool),
                             n_obs=1)
    out = particle_filter(model("Windkessel"), g["wk/theta"], grid, RngStream(7), inputs=inputs,
                          n_particles=1024, resampler=scheme, noise="host")
    ref = float(g[f"wk/{scheme}/loglik"])
    assert abs(out.loglik - ref) <= 1e-12 * abs(ref)
    assert normwise(out.trajectory, g[f"wk/{scheme}/traj"]) <= 1e-12


def _grid(g, name):
    m = model(name)
    T = len(g[f"{name}/times"]) - 1
    return m, build_filter_grid(0.0, float(g[f"{name}/times"][-1]), T, g[f"{name}/obs_t"], g[f"{name}/obs_v"],
                                g[f"{name}/obs_m"], n_obs=m.n_obs)


@pytest.mark.parametrize("name", ["StochVol", "PredatorPrey"])
@pytest.mark.parametrize("scheme", ["systematic", "multinomial"])
def test_generic_test_models_host_noise_match_reference(name, scheme):
    g = load_golden("generic.npz")
    m, grid = _grid(g, name)
    out = particle_filter(m, g[f"{name}/theta"], grid, RngStream(11), n_particles=512, resampler=scheme,
                          noise="host")
    ref = float(g[f"{name}/{scheme}/loglik"])
    assert abs(out.loglik - ref) <= 1e-9 * max(1.0, abs(ref)), (out.loglik, ref)
    np.testing.assert_array_equal(_anc(out), g[f"{name}/{scheme}/anc"][1:])
    assert normwise(out.run.x, g[f"{name}/{scheme}/x_final"]) <= 1e-9
    assert normwise(out.trajectory, g[f"{name}/{scheme}/traj"]) <= 1e-9


@pytest.mark.parametrize("name", ["StochVol", "PredatorPrey"])
def test_generic_single_step_and_density(name):
    """simulate.step_transition / observe_logpdf through the generic kernel with
    the reference's draws (one grid step, several RK4 steps for PredatorPrey)."""
    g = load_golden("generic.npz")
    m = model(name)
    th = g[f"{name}/theta"]
    dt = float(g[f"{name}/times"][1] - g[f"{name}/times"][0])
    x1 = S.step_transition(m, th, g[f"{name}/x0"], None, 0.0, dt, RngStream(6))
    assert normwise(x1, g[f"{name}/x1"]) <= 1e-12
    lp = S.observe_logpdf(m, th, g[f"{name}/x1"], None, g[f"{name}/obs_v"][0], g[f"{name}/obs_m"][0])
    assert normwise(lp, g[f"{name}/g1"]) <= 1e-12


def test_generic_parameter_error_raised():
    g = load_golden("generic.npz")
    m, grid = _grid(g, "StochVol")
    with pytest.raises(DistributionParameterError):
        particle_filter(m, np.array([0.0, 0.5, -1.0]), grid, RngStream(1), n_particles=256)  # sigma < 0


def test_generic_l96_device_noise_agrees_with_hand_written():
    """Same model, independent device draws: the two filters' mean
    log-likelihoods agree within Monte Carlo error."""
    g = load_golden("pf.npz")
    grid = _l96_grid(g)
    th = [g["l96/theta"]] * 24
    lls = []
    for spec in (LORENZ96, model("Lorenz96")):
        runner = FilterRunner(spec, grid, n_particles=1 << 14, resampler="systematic")
        res = runner.run_batch(th, [None] * len(th), [RngStream(300 + k) for k in range(len(th))])
        lls.append(np.array([r[0] for r in res]))
    se = np.sqrt(lls[0].var(ddof=1) / len(th) + lls[1].var(ddof=1) / len(th))
    assert abs(lls[0].mean() - lls[1].mean()) < 4 * se + 0.05, (lls[0].mean(), lls[1].mean(), se)


def test_generic_windkessel_device_noise_unbiased_vs_kalman():
    g = load_golden("pf.npz")
    kf = float(g["wk/kf_loglik"])
    inputs = LocfInputs(g["wk/in_times"], g["wk/in_values"])
    grid = build_filter_grid(0.0, 1.0, 100, np.linspace(0, 1, 101)[1:], g["wk/obs_v"], np.ones((100, 1), bool),
                             n_obs=1)
    runner = FilterRunner(model("Windkessel"), grid, inputs=inputs, n_particles=4096, resampler="systematic")
    res = runner.run_batch([g["wk/theta"]] * 48, [None] * 48, [RngStream(2000 + k) for k in range(48)])
    ll = np.array([r[0] for r in res])
    se = ll.std(ddof=1) / np.sqrt(len(ll))
    assert abs(ll.mean() - kf) < 4 * se + 0.02, (ll.mean(), kf, se)


def test_generic_f32_and_fast_modes_track_exact():
    g = load_golden("generic.npz")
    m, grid = _grid(g, "PredatorPrey")
    base = particle_filter(m, g["PredatorPrey/theta"], grid, RngStream(3), n_particles=4096,
                           resampler="systematic", exact=True, upto=6)
    fast = particle_filter(m, g["PredatorPrey/theta"], grid, RngStream(3), n_particles=4096,
                           resampler="systematic", exact=False, upto=6)
    f32 = particle_filter(m, g["PredatorPrey/theta"], grid, RngStream(3), n_particles=4096,
                          resampler="systematic", dtype="float32", upto=6)
    assert abs(fast.loglik - base.loglik) <= 1e-6 * max(1.0, abs(base.loglik))
    assert abs(f32.loglik - base.loglik) <= 0.05 * max(1.0, abs(base.loglik))


@pytest.mark.parametrize("name", ["StochVol", "PredatorPrey"])
def test_generic_pmmh_and_smc2_match_reference(name):
    from paper_1306_3277_b200.inference import mh_sample, smc_sampler

    g = load_golden("generic.npz")
    m, grid = _grid(g, name)
    runner = FilterRunner(m, grid, n_particles=64, resampler="systematic", noise="host")
    chains, acc = mh_sample(m, runner, 5, RngStream(31))
    assert acc == int(g[f"{name}/mh/accepted"])
    np.testing.assert_allclose(np.array([c.theta for c in chains]), g[f"{name}/mh/thetas"], rtol=1e-12)
    np.testing.assert_allclose([c.loglik for c in chains], g[f"{name}/mh/logliks"], rtol=1e-9)
    res = smc_sampler(m, runner, 6, RngStream(32), theta_resampler="systematic")
    np.testing.assert_allclose(res.thetas, g[f"{name}/smc/thetas"], rtol=1e-12)
    np.testing.assert_allclose(res.logliks, g[f"{name}/smc/logliks"], rtol=1e-9)
    np.testing.assert_allclose(res.log_v, g[f"{name}/smc/log_v"], rtol=1e-8, atol=1e-10)


def test_generic_l96_pmmh_with_initial_proposals_matches_reference():
    """Lorenz '96 through the generic path end to end in PMMH, including the
    proposal_initial block (x0 proposed jointly with theta): the reference's chain."""
    from paper_1306_3277_b200.inference import mh_sample

    g = load_golden("outer.npz")
    times = g["l96/times"]
    grid = build_filter_grid(0.0, times[-1], 10, times[1:], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)
    m = model("Lorenz96")
    assert m.has_proposal_initial
    runner = FilterRunner(m, grid, n_particles=64, resampler="systematic", noise="host")
    chains, acc = mh_sample(m, runner, 6, RngStream(21))
    assert acc == int(g["l96/mh/accepted"])
    np.testing.assert_array_equal(np.array([c.theta for c in chains]), g["l96/mh/thetas"])
    np.testing.assert_array_equal(np.array([c.init_state for c in chains]), g["l96/mh/inits"])
    np.testing.assert_allclose([c.loglik for c in chains], g["l96/mh/logliks"], rtol=1e-12)


def test_generic_l96_ess_gate_and_sparse_obs_bitwise_reference():
    """ESS-gated resampling and a sparse observation mask (4 of 8 slots, every
    other step) through the generic kernel with the reference's draws."""
    g = load_golden("pf.npz")
    m = model("Lorenz96")
    out = particle_filter(m, g["l96/theta"], _l96_grid(g), RngStream(9), n_particles=256, resampler="systematic",
                          ess_rel=0.5, noise="host")
    assert abs(out.loglik - float(g["l96/ess/loglik"])) <= 1e-12 * abs(float(g["l96/ess/loglik"]))
    np.testing.assert_array_equal(out.trajectory, g["l96/ess/traj"])
    grid = build_filter_grid(0.0, 2.0, 20, g["l96/obs_t"], g["l96s/obs_v"], g["l96s/obs_m"], n_obs=8)
    out = particle_filter(m, g["l96/theta"], grid, RngStream(8), n_particles=128, resampler="systematic",
                          noise="host")
    assert abs(out.loglik - float(g["l96s/loglik"])) <= 1e-12 * abs(float(g["l96s/loglik"]))
    np.testing.assert_array_equal(out.trajectory, g["l96s/traj"])


def test_generic_sharded_one_rank_equals_particle_filter():
    from paper_1306_3277_b200.inference import particle_filter_sharded

    g = load_golden("generic.npz")
    m, grid = _grid(g, "StochVol")
    th = g["StochVol/theta"]
    ll, traj = particle_filter_sharded(m, th, grid, RngStream(31), 1 << 14, resampler="systematic")
    out = particle_filter(m, th, grid, RngStream(31), n_particles=1 << 14, resampler="systematic", exact=False)
    assert ll == out.loglik
    np.testing.assert_array_equal(traj, out.trajectory)


def test_generic_twelve_observations_two_inputs_bitwise_reference():
    """Wide.bi: 12 observed slots (one step partially masked) and two LOCF inputs,
    through the per-step device tables (ssm_pw_args.y_vec / u_vec): bitwise the
    reference's run with its draws."""
    g = load_golden("generic.npz")
    m = model("Wide")
    assert m.n_obs == 12 and m.n_input == 2
    inputs = LocfInputs(g["Wide/in_times"], g["Wide/in_values"])
    grid = build_filter_grid(0.0, 2.0, 20, g["Wide/obs_t"], g["Wide/obs_v"], g["Wide/obs_m"], n_obs=12)
    out = particle_filter(m, g["Wide/theta"], grid, RngStream(12), inputs=inputs, n_particles=512,
                          resampler="systematic", noise="host")
    ref = float(g["Wide/loglik"])
    assert abs(out.loglik - ref) <= 1e-12 * abs(ref), (out.loglik, ref)
    np.testing.assert_array_equal(out.run.x, g["Wide/x_final"])
    np.testing.assert_array_equal(out.trajectory, g["Wide/traj"])
    # device noise through the native driver (per-step table offsets in ssm_step_desc)
    # against host draws through the per-step loop, same P: equal within Monte Carlo error
    lls = {}
    for noise in ("device", "host"):
        lls[noise] = np.array([particle_filter(m, g["Wide/theta"], grid, RngStream(40 + k), inputs=inputs,
                                               n_particles=1 << 13, resampler="systematic", noise=noise,
                                               exact=False).loglik for k in range(6)])
    se = np.sqrt(lls["device"].var(ddof=1) / 6 + lls["host"].var(ddof=1) / 6)
    assert abs(lls["device"].mean() - lls["host"].mean()) < 4 * se + 0.5, (lls, se)


@pytest.mark.parametrize("name", ["Lorenz96", "StochVol", "PredatorPrey"])
def test_generic_simple_variant_equals_general(name, monkeypatch):
    """The SIMPLE generated kernel (one sub-step, one RK4 step per ode; chosen from
    SSM_HINT_SINGLE_SUBSTEP) is the general kernel with its loops removed:
    bitwise the same filter.  PredatorPrey (4 RK4 steps per grid step) must not
    take it."""
    from paper_1306_3277_b200.inference import particle as particle_mod

    m = model(name)
    if name == "Lorenz96":  # grid step = delta = h: one sub-step, one RK4 step
        g = load_golden("pf.npz")
        theta = g["l96/theta"]
        grid = build_filter_grid(0.0, 2.0, 40, g["l96/obs_t"], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)
    else:
        g = load_golden("generic.npz")
        m, grid = _grid(g, name)
        theta = g[f"{name}/theta"]
    sched = particle_mod.Schedule(grid, m, None, "cuda")
    assert any(sched.single[1:]) == (name != "PredatorPrey")
    outs = []
    for no_hints in (False, True):
        monkeypatch.setattr(particle_mod, "_NO_HINTS", no_hints)
        outs.append(particle_filter(m, theta, grid, RngStream(17), n_particles=40000, resampler="systematic",
                                    exact=False))
    assert outs[0].loglik == outs[1].loglik
    np.testing.assert_array_equal(outs[0].trajectory, outs[1].trajectory)
    np.testing.assert_array_equal(np.asarray(outs[0].run.x), np.asarray(outs[1].run.x))

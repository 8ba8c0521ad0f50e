"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import ssm_oracle as O
from tests.conftest import LocfInputs, load_golden


def test_versions_recorded():
    g = load_golden("pf.npz")
    assert "numpy" in str(g["versions"])


@pytest.mark.parametrize("case", ["onehot", "half", "ties", "zeros_mixed", "lognormal_1k",
                                  "uniform_4097", "degenerate_2k", "tiny_16384"])
@pytest.mark.parametrize("scheme", ["multinomial", "stratified", "systematic"])
def test_resample_exact(case, scheme):
    g = load_golden("resample.npz")
    w = g[f"{case}/w"]
    cum = O.cumulative(w)
    np.testing.assert_array_equal(cum, g[f"{case}/cum"])
    anc = O.resample_with(w, scheme, g[f"{case}/{scheme}/u"])
    np.testing.assert_array_equal(anc, g[f"{case}/{scheme}/anc"])


def test_resample_tie_kat():
    g = load_golden("resample.npz")
    anc = O.resample_with(g["kat_ties/w"], "multinomial", g["kat_ties/u"], size=5)
    np.testing.assert_array_equal(anc, g["kat_ties/anc"])
    np.testing.assert_array_equal(anc, [1, 0, 1, 2, 2])


def test_onehot_all_zero_ancestors():
    g = load_golden("resample.npz")
    for s in ("multinomial", "stratified", "systematic"):
        assert (g[f"onehot/{s}/anc"] == 0).all()
    assert list(g["half/systematic/anc"]) == [0, 1]


@pytest.mark.parametrize("case", ["normal", "wide", "ties", "with_ninf", "one_dominant"])
def test_logsumexp(case):
    g = load_golden("lse.npz")
    assert O.logsumexp(g[f"{case}/a"]) == float(g[f"{case}/lse"])


@pytest.mark.parametrize("c", range(5))
def test_l96_step_bitwise(c):
    g = load_golden("l96_step.npz")
    W = g[f"c{c}/W"]
    x, t_fail = O.l96_transition(g[f"c{c}/theta"], g[f"c{c}/x_in"], float(g[f"c{c}/t"]),
                                 float(g[f"c{c}/dt"]), lambda k, d: W[k].T)
    assert t_fail is None
    np.testing.assert_array_equal(x, g[f"c{c}/x_out"])
    np.testing.assert_array_equal(O.l96_obs_logpdf(x, g[f"c{c}/y"], g[f"c{c}/mask"]), g[f"c{c}/g"])
    np.testing.assert_array_equal(O.l96_obs_logpdf(x, g[f"c{c}/y"], np.ones(8, bool)),
                                  g[f"c{c}/g_all"])


def test_l96_fixed_point():
    g = load_golden("l96_step.npz")
    np.testing.assert_array_equal(g["fixed/x_out"], 10.0)
    x, _ = O.l96_transition([10.0, 0.0], np.full((4, 8), 10.0), 0.0, 0.05,
                            lambda k, d: np.zeros((4, 8)))
    np.testing.assert_array_equal(x, 10.0)


@pytest.mark.parametrize("c", range(3))
def test_wk_step_bitwise(c):
    g = load_golden("wk_step.npz")
    inputs = LocfInputs(g["in_times"], g["in_values"])
    xi = g[f"c{c}/xi"]
    theta = g[f"c{c}/theta"]
    t, dt = float(g[f"c{c}/t"]), float(g[f"c{c}/dt"])
    x, _ = O.wk_transition(theta, g[f"c{c}/x_in"], t, dt, lambda k, sd: xi[k], inputs.scalar)
    np.testing.assert_array_equal(x, g[f"c{c}/x_out"])
    gl = O.wk_obs_logpdf(theta, x, inputs.scalar(t + dt), g[f"c{c}/y"], np.array([True]))
    np.testing.assert_array_equal(gl, g[f"c{c}/g"])


def _l96_grid(g, prefix="l96"):
    times = np.linspace(0.0, 2.0, 21) if prefix == "l96s" else g["l96/times"]
    obs = {k + 1: (g[f"{prefix}/obs_v"][k], g[f"{prefix}/obs_m"][k])
           for k in range(len(g[f"{prefix}/obs_v"]))}
    return O.Grid(times, obs)


@pytest.mark.parametrize("scheme", ["systematic", "multinomial", "stratified"])
def test_pf_l96_end_to_end_bitwise(scheme):
    g = load_golden("pf.npz")
    grid = _l96_grid(g)
    ll, traj, f = O.particle_filter("lorenz96", g["l96/theta"], grid, O.Stream(7),
                                    n_particles=256, resampler=scheme)
    assert ll == float(g[f"l96/{scheme}/loglik"])
    np.testing.assert_array_equal(traj, g[f"l96/{scheme}/traj"])
    np.testing.assert_array_equal(f.x, g[f"l96/{scheme}/x_final"])
    np.testing.assert_array_equal(f.logw, g[f"l96/{scheme}/logw_final"])
    anc = np.array([h[1] for h in f.history[1:]])
    np.testing.assert_array_equal(anc, g[f"l96/{scheme}/anc"])


def test_pf_l96_ess_and_sparse():
    g = load_golden("pf.npz")
    ll, traj, _ = O.particle_filter("lorenz96", g["l96/theta"], _l96_grid(g), O.Stream(9),
                                    n_particles=256, resampler="systematic", ess_rel=0.5)
    assert ll == float(g["l96/ess/loglik"])
    np.testing.assert_array_equal(traj, g["l96/ess/traj"])
    ll, traj, _ = O.particle_filter("lorenz96", g["l96/theta"], _l96_grid(g, "l96s"), O.Stream(8),
                                    n_particles=128, resampler="systematic")
    assert ll == float(g["l96s/loglik"])
    np.testing.assert_array_equal(traj, g["l96s/traj"])


@pytest.mark.parametrize("scheme", ["multinomial", "systematic"])
def test_pf_windkessel_end_to_end(scheme):
    g = load_golden("pf.npz")
    inputs = LocfInputs(g["wk/in_times"], g["wk/in_values"])
    times = np.linspace(0.0, 1.0, 101)
    obs = {k + 1: (g["wk/obs_v"][k], np.array([True])) for k in range(100)}
    ll, traj, _ = O.particle_filter("windkessel", g["wk/theta"], O.Grid(times, obs), O.Stream(7),
                                    n_particles=1024, resampler=scheme, inputs=inputs.scalar)
    assert ll == float(g[f"wk/{scheme}/loglik"])
    np.testing.assert_array_equal(traj, g[f"wk/{scheme}/traj"])

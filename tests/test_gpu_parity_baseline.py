"""Parity at the BASELINE.json configuration sizes and on the kernels that the
golden-vector tests do not reach directly (-m gpu).

  * config 2 (L96, 2^20 particles, systematic, float64): the reference's own
    draws (noise="host", exact arithmetic) -> log-likelihood within 1e-12 of the
    oracle, ancestors and trajectory bitwise;
  * the HEADLINE kernel (the benchmark's pw_kernel<L96, f64, fast, device
    noise, SIMPLE> plus the tile-record resampling path) against the oracle
    run on exactly the draws the device consumed (tests/device_draws.py):
    ancestors equal at every step, states / log-likelihood / trajectory within
    1e-10 (FMA arithmetic, 1e-12 per step), at 2^16 and at config 2's 2^20,
    for all three schemes; the windkessel SIMPLE kernel likewise at 2^16;
  * the 2^24 headline size: the tile path's exact fixed-point CDF against the
    reference's float64 cumsum -- a documented bound on ancestor disagreement
    (DESIGN.md section 5);
  * the persistent small-P kernel (config 1 and the 2^10 / 2^12 sweep points)
    over a full run against the multi-kernel path, and config 1 / config 3's
    2^16 windkessel filters against the exact Kalman likelihood.
Reference anchors: inference/particle.py:96-149, inference/resampling.py:22-36,
core/simulate.py:132-193.
"""

import numpy as np
import pytest
import torch

from oracle import ssm_oracle as O
from paper_1306_3277_b200 import LORENZ96, WINDKESSEL, RngStream
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, particle_filter
from paper_1306_3277_b200.rng import device_key
from tests.conftest import LocfInputs, load_golden
from tests.device_draws import DeviceDrawStream, device_init_l96

pytestmark = pytest.mark.gpu

SCHEMES = ["multinomial", "stratified", "systematic"]


def normwise(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


def _bench_l96_grid(T, seed=1):
    """The benchmark data recipe: theta* = (10, 0.1), grid
    linspace(0, 2, 41), all 8 slots observed every step; first T steps."""
    theta = np.array([10.0, 0.1])
    times = np.linspace(0.0, 2.0, 41)
    obs = O.simulate_l96(theta, times, O.Stream(seed))
    ov = np.array([obs[k][0] for k in range(1, 41)])
    om = np.array([obs[k][1] for k in range(1, 41)])
    grid = build_filter_grid(0.0, 2.0, 40, times[1:], ov, om, n_obs=8)
    ogrid = O.Grid(grid.times, {k: (ov[k - 1], om[k - 1]) for k in range(1, 41)})
    return theta, grid, ogrid


def _device_anc(run, T):
    out = []
    for i in range(1, T + 1):
        a = run.history[i][1]
        out.append(np.arange(run.n_particles) if a is None else a.cpu().numpy())
    return out


# ------------------------------------------------------------------ config 2, reference draws


def test_config2_l96_2p20_host_noise_matches_oracle():
    """Config 2 (2^20 particles, systematic, float64) on the reference's own
    draws: the exact float64 kernels + the tile-record resampler give the
    oracle's (= the reference's, tests/test_oracle_golden.py) filter."""
    P, T = 1 << 20, 4
    theta, grid, ogrid = _bench_l96_grid(T)
    out = particle_filter(LORENZ96, theta, grid, RngStream(21), n_particles=P, resampler="systematic",
                          noise="host", upto=T)
    ll, traj, f = O.particle_filter("lorenz96", theta, ogrid, O.Stream(21), n_particles=P,
                                    resampler="systematic", upto=T)
    assert abs(out.loglik - ll) <= 1e-12 * abs(ll), (out.loglik, ll)
    for i, a in enumerate(_device_anc(out.run, T), start=1):
        np.testing.assert_array_equal(a, f.history[i][1], err_msg=f"ancestors at step {i}")
    np.testing.assert_array_equal(out.run.x, f.x)
    np.testing.assert_array_equal(out.trajectory, traj)


# ------------------------------------------------------------------ headline kernel, device draws


def _oracle_on_device_draws(model, theta, ogrid, rng, P, scheme, T, x0, inputs=None):
    keys_init = device_key(rng.child(0))
    keys_adv = device_key(rng.child(1))
    f = O.OracleFilter(model, theta, ogrid, P, scheme, inputs=inputs)
    f.init(O.Stream(0))
    f.x = x0
    f.history = [(x0, None)]
    f.advance_to(T, DeviceDrawStream(model, keys_init, keys_adv, P, scheme))
    traj = f.sample_trajectory(O.Stream(rng.seed, rng.key).child(2))
    return f, traj


@pytest.mark.parametrize("P,T", [(1 << 16, 10), (1 << 20, 3)])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_headline_kernel_matches_oracle_on_device_draws(P, T, scheme):
    """The benchmark path itself -- device Philox noise, float64 FMA, the SIMPLE
    fused kernel, resampling from its tile records (sorted multinomial for the
    default scheme) -- against the oracle fed the same draws."""
    theta, grid, ogrid = _bench_l96_grid(T)
    rng = RngStream(33)
    out = particle_filter(LORENZ96, theta, grid, rng, n_particles=P, resampler=scheme, upto=T)
    x0 = device_init_l96(device_key(rng.child(0)), P)
    np.testing.assert_array_equal(out.run.history[0][0].t().cpu().numpy(), x0)  # init draws bit for bit
    f, traj = _oracle_on_device_draws("lorenz96", theta, ogrid, rng, P, scheme, T, x0)
    for i, a in enumerate(_device_anc(out.run, T), start=1):
        np.testing.assert_array_equal(a, f.history[i][1], err_msg=f"ancestors at step {i}")
    assert abs(out.loglik - f.loglik) <= 1e-10 * abs(f.loglik), (out.loglik, f.loglik)
    assert normwise(out.run.x, f.x) <= 1e-10
    assert normwise(out.run.logw, f.logw) <= 1e-10
    assert normwise(out.trajectory, traj) <= 1e-10


def _wk_setup():
    g = load_golden("pf.npz")
    inputs = LocfInputs(g["wk/in_times"], g["wk/in_values"])
    grid = build_filter_grid(0.0, 1.0, 100, np.linspace(0, 1, 101)[1:], g["wk/obs_v"], np.ones((100, 1), bool),
                             n_obs=1)
    ogrid = O.Grid(grid.times, {k: (g["wk/obs_v"][k - 1], np.ones(1, bool)) for k in range(1, 101)})
    return g, inputs, grid, ogrid


@pytest.mark.parametrize("scheme", ["systematic", "multinomial"])
def test_windkessel_simple_kernel_matches_oracle_on_device_draws(scheme):
    """Config 3's filter kernel (windkessel, one sub-step per grid step, 2^16
    particles) against the oracle on the same draws over 30 grid steps."""
    g, inputs, grid, ogrid = _wk_setup()
    P, T = 1 << 16, 30
    rng = RngStream(44)
    out = particle_filter(WINDKESSEL, g["wk/theta"], grid, rng, inputs=inputs, n_particles=P, resampler=scheme,
                          upto=T)
    x0 = out.run.history[0][0].t().double().cpu().numpy()  # float64 Box-Muller init (libm-level log)
    assert abs(x0.mean() - 90.0) < 0.5 and abs(x0.std() - 15.0) < 0.5
    f, traj = _oracle_on_device_draws("windkessel", g["wk/theta"], ogrid, rng, P, scheme, T, x0,
                                      inputs=inputs.scalar)
    for i, a in enumerate(_device_anc(out.run, T), start=1):
        np.testing.assert_array_equal(a, f.history[i][1], err_msg=f"ancestors at step {i}")
    assert abs(out.loglik - f.loglik) <= 1e-11 * abs(f.loglik), (out.loglik, f.loglik)
    assert normwise(out.run.x, f.x) <= 1e-12
    assert normwise(out.trajectory, traj) <= 1e-12


def test_windkessel_simple_equals_general_kernel_2p16(monkeypatch):
    """The windkessel SIMPLE kernel (hint) and the general sub-step loop draw the
    same normals and apply the same update: same filter at 2^16."""
    from paper_1306_3277_b200.inference import particle as particle_mod

    g, inputs, grid, _ = _wk_setup()
    kw = dict(inputs=inputs, n_particles=1 << 16, resampler="systematic", upto=50)
    a = particle_filter(WINDKESSEL, g["wk/theta"], grid, RngStream(5), **kw)
    monkeypatch.setattr(particle_mod, "_NO_HINTS", True)
    b = particle_filter(WINDKESSEL, g["wk/theta"], grid, RngStream(5), **kw)
    assert abs(a.loglik - b.loglik) <= 1e-12 * abs(b.loglik)
    for aa, bb in zip(_device_anc(a.run, 50), _device_anc(b.run, 50)):
        np.testing.assert_array_equal(aa, bb)
    assert normwise(a.run.x, b.run.x) <= 1e-13
    assert normwise(a.trajectory, b.trajectory) <= 1e-13


# ------------------------------------------------------------------ 2^24: fixed-point CDF vs cumsum


def test_tile_cdf_vs_reference_cumsum_flip_bound_2p24():
    """At the 2^24 headline size the filter path's exact fixed-point CDF and the
    reference's sequential float64 cumsum(w / w.sum()) (resampling.py:26-27)
    differ by rounding (max |dcum| ~ 6e-14).  Given the same systematic uniform,
    ancestors may then disagree only where a query falls within that rounding
    of a CDF boundary.  Documented bound: at most 64 of 2^24
    outputs per resample for log-normal(sigma=1) weights (measured 2-4), and
    every disagreeing output's query lies within 1e-12 of the reference CDF
    value that separates the two ancestors."""
    from tests.test_gpu_parity import _tile_inputs

    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    P = 1 << 24
    a_np = np.random.default_rng(1).normal(0.0, 1.0, P)
    cdf, rec, fs, w = _tile_inputs(a_np)
    cum = O.cumulative(w)
    for seed in range(3):
        u_np = np.random.default_rng(10 + seed).random(1)
        u = torch.from_numpy(u_np).cuda()
        ws = torch.empty(L.ssm_resample_workspace_bytes(1, P), dtype=torch.uint8, device="cuda")
        anc = torch.empty(P, dtype=torch.int32, device="cuda")
        _lib.check(L.ssm_resample_from_tiles(1, P, _lib.SCHEME_IDS["systematic"], _lib.ptr(cdf), _lib.ptr(rec), _lib.ptr(fs),
                                             _lib.ptr(u), None, 1, _lib.ptr(anc), _lib.ptr(ws), _lib.stream_ptr()))
        got = anc.cpu().numpy()
        q = O.queries("systematic", u_np, P)
        ref = O.search(cum, q)
        bad = np.nonzero(got != ref)[0]
        assert bad.size <= 64, bad.size
        for k in bad:
            lo, hi = min(got[k], ref[k]), max(got[k], ref[k])
            # the boundary between the two candidate ancestors (zero-weight particles between them share it)
            assert np.min(np.abs(cum[lo:hi] - q[k])) <= 1e-12, (k, got[k], ref[k])


# ------------------------------------------------------------------ persistent small-P kernel


@pytest.mark.parametrize("scheme", ["systematic", "stratified"])
@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("P", [1024, 3000])
def test_small_kernel_full_run_matches_multikernel(scheme, exact, P, monkeypatch):
    """The persistent small-P kernel (one launch, 61-bit block scan + binary
    search in shared memory) over all 20 grid steps against the multi-kernel
    path (tile records + offspring counts) with the same device draws and the
    same (general) transition: identical ancestors at every step, bitwise
    states, log-likelihood to 1e-12, the same trajectory."""
    from paper_1306_3277_b200.inference import particle as particle_mod

    g = load_golden("pf.npz")
    grid = build_filter_grid(0.0, 2.0, 20, g["l96/obs_t"], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)
    kw = dict(n_particles=P, resampler=scheme, exact=exact)
    small = particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(3), **kw)
    monkeypatch.setattr(particle_mod, "_NO_SMALL", True)
    monkeypatch.setattr(particle_mod, "_NO_HINTS", True)  # the general transition, as the small kernel
    multi = particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(3), **kw)
    for i, (aa, bb) in enumerate(zip(_device_anc(small.run, 20), _device_anc(multi.run, 20)), start=1):
        np.testing.assert_array_equal(aa, bb, err_msg=f"ancestors at step {i}")
    np.testing.assert_array_equal(small.run.x, multi.run.x)
    assert abs(small.loglik - multi.loglik) <= 1e-12 * abs(multi.loglik)
    np.testing.assert_array_equal(small.trajectory, multi.trajectory)


@pytest.mark.parametrize("P,B", [(1024, 96), (1 << 16, 24)])
def test_windkessel_filters_unbiased_vs_kalman(P, B):
    """Config 1 (1024 particles: the persistent small-P kernel) and config 3's
    2^16-particle filter (the windkessel SIMPLE multi-kernel path) with device
    noise: the mean log-likelihood estimate agrees with the reference's exact
    Kalman log-likelihood (kalman.py:115-122) within 4 standard errors (the PF
    likelihood is unbiased on the natural scale; the log bias -var/2 is below
    the SE here)."""
    g, inputs, grid, _ = _wk_setup()
    kf = float(g["wk/kf_loglik"])
    runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=P, resampler="systematic")
    res = runner.run_batch([g["wk/theta"]] * B, [None] * B, [RngStream(7000 + k) for k in range(B)])
    ll = np.array([r[0] for r in res])
    se = ll.std(ddof=1) / np.sqrt(B)
    bias = 0.5 * ll.var(ddof=1)  # E log L_hat ~ log L - var/2
    assert abs(ll.mean() + bias - kf) < 4 * se + 1e-3, (ll.mean(), kf, se, bias)


def _spy_coop(monkeypatch):
    """Record the status of every ssm_advance_coop call."""
    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    real = L.ssm_advance_coop
    ran = []

    def spy(*a):
        st = real(*a)
        ran.append(st)
        return st

    monkeypatch.setattr(L, "ssm_advance_coop", spy)
    return ran


@pytest.mark.parametrize("kw", [dict(resampler="systematic"), dict(resampler="stratified"),
                                dict(resampler="systematic", ess_rel=0.6), dict(resampler="systematic", dtype="float32"),
                                dict(resampler="stratified", sparse=True), dict(resampler="systematic", keep_history=False)])
def test_persistent_driver_equals_per_step_kernels(kw, monkeypatch):
    """ssm_advance_coop (the whole grid loop in one cooperative launch, moderate
    particle counts) runs the per-step kernels' device bodies on virtual blocks:
    bitwise the same filters (states, ancestors, log-likelihoods, trajectories)
    as ssm_advance, batched."""
    from paper_1306_3277_b200.inference import particle as particle_mod

    kw = dict(kw)
    sparse = kw.pop("sparse", False)
    theta, times = np.array([10.0, 0.1]), np.linspace(0.0, 1.0, 21)
    obs = O.simulate_l96(theta, times, O.Stream(4), obs_slots=range(4) if sparse else range(8),
                         obs_every=2 if sparse else 1)
    grid = build_filter_grid(0.0, 1.0, 20, times[1:], np.array([obs[k][0] for k in range(1, 21)]),
                             np.array([obs[k][1] for k in range(1, 21)]), n_obs=8)
    thetas = [theta, np.array([9.0, 0.2]), np.array([11.0, 0.05]), np.array([10.5, 0.1])]
    outs = []
    monkeypatch.setattr(particle_mod, "COOP_MAX_PARTICLES", 1 << 20)  # opt in (off by default)
    ran = _spy_coop(monkeypatch)
    for no_coop in (False, True):
        monkeypatch.setattr(particle_mod, "_NO_COOP", no_coop)
        runner = FilterRunner(LORENZ96, grid, n_particles=20000, **kw)
        outs.append(runner.run_batch(thetas, [None] * 4, [RngStream(40 + k) for k in range(4)]))
    assert ran and all(st == 0 for st in ran)  # the persistent driver ran (and succeeded)
    for (la, ta, ra), (lb, tb, rb) in zip(*outs):
        assert la == lb
        np.testing.assert_array_equal(ta, tb)
        np.testing.assert_array_equal(ra.x, rb.x)
        if ra.keep_history:
            for aa, bb in zip(_device_anc(ra, 20), _device_anc(rb, 20)):
                np.testing.assert_array_equal(aa, bb)


def test_persistent_driver_windkessel_pmmh_batch(monkeypatch):
    """Config 3's filter batch (8 windkessel filters x 2^16) through the
    persistent driver equals the per-step kernels bitwise."""
    from paper_1306_3277_b200.inference import particle as particle_mod

    g, inputs, grid, _ = _wk_setup()
    thetas = [g["wk/theta"] * f for f in (1.0, 0.9, 1.1, 1.05, 0.95, 1.2, 0.8, 1.15)]
    outs = []
    monkeypatch.setattr(particle_mod, "COOP_MAX_PARTICLES", 1 << 20)  # opt in (off by default)
    ran = _spy_coop(monkeypatch)
    for no_coop in (False, True):
        monkeypatch.setattr(particle_mod, "_NO_COOP", no_coop)
        runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=1 << 16, resampler="systematic")
        outs.append(runner.run_batch(thetas, [None] * 8, [RngStream(80 + k) for k in range(8)]))
    assert ran and all(st == 0 for st in ran)
    for (la, ta, _), (lb, tb, _) in zip(*outs):
        assert la == lb
        np.testing.assert_array_equal(ta, tb)


# ------------------------------------------------------------------ logw resampling at 2^20, device draws


@pytest.mark.parametrize("scheme", ["stratified", "systematic"])
@pytest.mark.parametrize("sigma", [0.0, 1.0, 10.0])
def test_resample_from_logw_device_draws_match_numpy_2p20(scheme, sigma):
    """ssm_resample_from_logw (tile records built from the log-weights, then the
    filter path's resampler; the stratified one-draw fast path) at 2^20 with
    device uniforms, against numpy: the same Philox uniforms, the reference's
    queries and float64 cumsum + searchsorted (resampling.py:22-36).  At most a
    handful of ancestors may differ, and only where a query lies within 1e-12 of
    the CDF boundary between the two candidates (fixed-point vs float cumsum)."""
    from scipy.special import logsumexp

    from paper_1306_3277_b200 import _lib
    from tests.test_gpu_parity import _philox4x32_10

    L = _lib.lib()
    P, step = 1 << 20, 3
    a_np = np.random.default_rng(7).normal(0.0, sigma, P) if sigma > 0 else np.zeros(P)
    a = torch.from_numpy(a_np).cuda()
    shift = torch.tensor([logsumexp(a_np)], dtype=torch.float64, device="cuda")
    keys_np = np.array([[1234, 5678]], dtype=np.uint32)
    keys = torch.from_numpy(keys_np.view(np.int32)).cuda()
    ws = torch.empty(L.ssm_resample_workspace_bytes(1, P), dtype=torch.uint8, device="cuda")
    anc = torch.empty(P, dtype=torch.int32, device="cuda")
    _lib.check(L.ssm_resample_from_logw(1, P, _lib.SSM_F64, _lib.SCHEME_IDS[scheme], _lib.ptr(a), _lib.ptr(shift),
                                        None, None, _lib.ptr(keys), step, _lib.ptr(anc), _lib.ptr(ws),
                                        _lib.stream_ptr()))
    got = anc.cpu().numpy()
    # device uniforms: Philox4x32-10 {k, step, 0, kPurposeResample=2} -> 53-bit (x, y); systematic: k = 0,
    # purpose kPurposeSystematic=4
    if scheme == "stratified":
        k = np.arange(P, dtype=np.uint64)
        r = _philox4x32_10([k, np.full(P, step), np.zeros(P), np.full(P, 2)], *keys_np[0])
    else:
        r = _philox4x32_10([np.zeros(1), np.full(1, step), np.zeros(1), np.full(1, 4)], *keys_np[0])
    u = ((r[0] << np.uint64(32)) | r[1]) >> np.uint64(11)
    u = u.astype(np.float64) * 2.0**-53
    q = O.queries(scheme, u, P)
    w = np.exp(a_np - logsumexp(a_np))
    cum = O.cumulative(w)
    ref = O.search(cum, q)
    bad = np.nonzero(got != ref)[0]
    assert bad.size <= 8, bad.size
    for kk in bad:
        lo, hi = min(got[kk], ref[kk]), max(got[kk], ref[kk])
        assert np.min(np.abs(cum[lo:hi] - q[kk])) <= 1e-12, (kk, got[kk], ref[kk])


def test_tma_staged_gather_variant_bitwise_equal():
    """The opt-in TMA-staged gather of the headline kernel (SSM_PW_TMA=1: per warp
    tile, cp.async.bulk copies of the contiguous ancestor range into shared
    memory) gives bitwise the same filter as the register-prefetch kernel (run in
    subprocesses: the switch is read once per process), f64 and f32."""
    import os
    import subprocess
    import sys

    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import bench\n"
        "from paper_1306_3277_b200 import LORENZ96, RngStream\n"
        "from paper_1306_3277_b200.inference import build_filter_grid, particle_filter\n"
        "t, ot, ov, om = bench.synthetic_data(40)\n"
        "g = build_filter_grid(0.0, t[-1], 40, ot, ov, om, n_obs=8)\n"
        "for dt in ('float64', 'float32'):\n"
        "    o = particle_filter(LORENZ96, bench.THETA, g, RngStream(9), n_particles=(1 << 16) + 64, "
        "resampler='systematic', dtype=dt, upto=12)\n"
        "    print(repr(o.loglik), float(np.abs(o.trajectory).sum()).hex())\n"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {"SSM_PW_TMA": "1"}):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                           env={**os.environ, **env})
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.split())
    assert outs[0] == outs[1]

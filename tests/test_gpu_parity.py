"""GPU parity tests: the CUDA path through the C ABI against the reference's
golden vectors and the CPU oracle.  Tolerances (north star / SURVEY 8c):
  - ancestors: exact, given identical (cum, u);
  - float64 exact mode: bitwise for L96 states / log-weights (reference op
    order, no FMA), 1e-12 relative for LSE-accumulated likelihoods;
  - float32: norm-wise relative ||out - ref||_inf / ||ref||_inf <= 1e-5.
"""

import numpy as np
import pytest
import torch

from oracle import ssm_oracle as O
from paper_1306_3277_b200 import LORENZ96, WINDKESSEL, RngStream
from paper_1306_3277_b200 import simulate as S
from paper_1306_3277_b200.errors import DegenerateEnsembleError, NonFiniteStateError
from paper_1306_3277_b200.inference import (FilterRunner, ParticleRun, advance_runs, build_filter_grid,
                                            init_runs, particle_filter, resample, sample_trajectories,
                                            search_cdf)
from tests.conftest import LocfInputs, load_golden

pytestmark = pytest.mark.gpu

CASES = ["onehot", "half", "ties", "zeros_mixed", "lognormal_1k", "uniform_4097", "degenerate_2k", "tiny_16384"]
SCHEMES = ["multinomial", "stratified", "systematic"]


def normwise(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


class FixedU:
    def __init__(self, u):
        self.u = np.asarray(u, dtype=float)

    def uniform(self, low=0.0, high=1.0, size=None):
        return float(self.u[0]) if size is None else self.u[:size].copy()


# ------------------------------------------------------------------ resampling


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("scheme", SCHEMES)
def test_search_exact_on_injected_cdf(case, scheme):
    g = load_golden("resample.npz")
    anc = search_cdf(g[f"{case}/cum"], g[f"{case}/{scheme}/u"], scheme)
    np.testing.assert_array_equal(anc, g[f"{case}/{scheme}/anc"])


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("scheme", SCHEMES)
def test_resample_api_matches_reference(case, scheme):
    g = load_golden("resample.npz")
    anc = resample(g[f"{case}/w"], scheme, FixedU(g[f"{case}/{scheme}/u"]))
    np.testing.assert_array_equal(anc, g[f"{case}/{scheme}/anc"])


def test_resample_tie_kat_and_errors():
    g = load_golden("resample.npz")
    anc = resample(g["kat_ties/w"], "multinomial", FixedU(g["kat_ties/u"]), size=5)
    np.testing.assert_array_equal(anc, [1, 0, 1, 2, 2])
    with pytest.raises(ValueError):
        resample(np.array([0.5, -0.1]), "systematic", FixedU([0.3]))
    with pytest.raises(ValueError):
        resample(np.array([0.5, np.nan]), "systematic", FixedU([0.3]))
    with pytest.raises(DegenerateEnsembleError):
        resample(np.zeros(5), "systematic", FixedU([0.3]))
    with pytest.raises(ValueError):
        resample(np.zeros(0), "systematic", FixedU([0.3]))


@pytest.mark.parametrize("scheme", SCHEMES)
def test_search_large_random_vs_numpy(scheme):
    rs = np.random.default_rng(5)
    P = (1 << 20) + 17
    w = np.exp(rs.normal(0, 2, P))
    cum = O.cumulative(w)
    u = rs.random(1 if scheme == "systematic" else P)
    ref = O.resample_with(w, scheme, u)
    np.testing.assert_array_equal(search_cdf(cum, u, scheme), ref)


def test_scan_cdf_is_deterministic_and_close():
    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    rs = np.random.default_rng(9)
    P = 3_000_001
    w = np.exp(rs.normal(0, 3, P))
    dev = torch.device("cuda")
    wt = torch.from_numpy(w).to(dev)
    outs = []
    for _ in range(3):
        ws = torch.empty(L.ssm_scan_workspace_bytes(1, P), dtype=torch.uint8, device=dev)
        C = torch.empty(P, dtype=torch.int64, device=dev)
        cum = torch.empty(P, dtype=torch.float64, device=dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(L.ssm_weights_scan(1, P, 1, _lib.ptr(wt), 0, None, None, _lib.ptr(C), _lib.ptr(flags),
                                      _lib.ptr(ws), _lib.stream_ptr()))
        _lib.check(L.ssm_fixed_to_cum(1, P, _lib.ptr(C), _lib.ptr(cum), _lib.stream_ptr()))
        outs.append(cum.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])
    ref = O.cumulative(w)
    assert outs[0][-1] == 1.0
    assert np.max(np.abs(outs[0] - ref)) < 1e-12
    assert np.all(np.diff(outs[0]) >= 0)


def test_gather_kernel():
    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    rs = np.random.default_rng(2)
    B, nx, P = 3, 8, 5000
    x = torch.from_numpy(rs.normal(size=(B, nx, P))).cuda()
    anc = torch.from_numpy(rs.integers(0, P, size=(B, P)).astype(np.int32)).cuda()
    out = torch.empty_like(x)
    _lib.check(L.ssm_gather(1, B, nx, P, _lib.ptr(x), _lib.ptr(anc), _lib.ptr(out), _lib.stream_ptr()))
    ref = torch.gather(x, 2, anc.long().unsqueeze(1).expand(B, nx, P))
    assert torch.equal(out, ref)


@pytest.mark.parametrize("case", ["normal", "wide", "ties", "with_ninf", "one_dominant"])
def test_logsumexp_kernel(case):
    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    g = load_golden("lse.npz")
    a = torch.from_numpy(g[f"{case}/a"]).cuda()
    P = a.numel()
    ws = torch.empty(L.ssm_lse_workspace_bytes(1, P), dtype=torch.uint8, device="cuda")
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    _lib.check(L.ssm_logsumexp(1, 1, P, _lib.ptr(a), _lib.ptr(out), None, _lib.ptr(ws), _lib.stream_ptr()))
    ref = float(g[f"{case}/lse"])
    assert abs(out[0].item() - ref) <= 1e-13 * max(1.0, abs(ref))


# ------------------------------------------------------------------ model kernels


@pytest.mark.parametrize("c", range(5))
def test_l96_step_bitwise_f64(c):
    g = load_golden("l96_step.npz")
    x = S.step_transition(LORENZ96, g[f"c{c}/theta"], g[f"c{c}/x_in"], None, float(g[f"c{c}/t"]),
                          float(g[f"c{c}/dt"]), noise=g[f"c{c}/W"])
    np.testing.assert_array_equal(x, g[f"c{c}/x_out"])
    gl = S.observe_logpdf(LORENZ96, g[f"c{c}/theta"], x, None, g[f"c{c}/y"], g[f"c{c}/mask"])
    np.testing.assert_array_equal(gl, g[f"c{c}/g"])


@pytest.mark.parametrize("c", range(5))
def test_l96_step_reference_rng(c):
    """Same RngStream as the reference -> the reference's x_out, bitwise."""
    g = load_golden("l96_step.npz")
    x = S.step_transition(LORENZ96, g[f"c{c}/theta"], g[f"c{c}/x_in"], None, float(g[f"c{c}/t"]),
                          float(g[f"c{c}/dt"]), RngStream(100 + c))
    np.testing.assert_array_equal(x, g[f"c{c}/x_out"])


@pytest.mark.parametrize("c", range(5))
def test_l96_step_fast_f64_and_f32(c):
    g = load_golden("l96_step.npz")
    args = (LORENZ96, g[f"c{c}/theta"], g[f"c{c}/x_in"], None, float(g[f"c{c}/t"]), float(g[f"c{c}/dt"]))
    x = S.step_transition(*args, noise=g[f"c{c}/W"], exact=False)
    assert normwise(x, g[f"c{c}/x_out"]) <= 1e-12
    x32 = S.step_transition(*args, noise=g[f"c{c}/W"], dtype="float32", exact=False)
    assert normwise(x32, g[f"c{c}/x_out"]) <= 1e-5
    g32 = S.observe_logpdf(LORENZ96, g[f"c{c}/theta"], x32, None, g[f"c{c}/y"], g[f"c{c}/mask"], dtype="float32")
    assert normwise(g32, g[f"c{c}/g"]) <= 1e-5


def test_l96_fixed_point():
    x = S.step_transition(LORENZ96, [10.0, 0.0], np.full((4, 8), 10.0), None, 0.0, 0.05, RngStream(1))
    np.testing.assert_array_equal(x, 10.0)


@pytest.mark.parametrize("c", range(3))
def test_wk_step_bitwise_f64(c):
    g = load_golden("wk_step.npz")
    inputs = LocfInputs(g["in_times"], g["in_values"])
    t, dt = float(g[f"c{c}/t"]), float(g[f"c{c}/dt"])
    x = S.step_transition(WINDKESSEL, g[f"c{c}/theta"], g[f"c{c}/x_in"], inputs, t, dt,
                          noise=g[f"c{c}/xi"][:, None, :])
    np.testing.assert_array_equal(x, g[f"c{c}/x_out"])
    x2 = S.step_transition(WINDKESSEL, g[f"c{c}/theta"], g[f"c{c}/x_in"], inputs, t, dt, RngStream(200 + c))
    np.testing.assert_array_equal(x2, g[f"c{c}/x_out"])
    gl = S.observe_logpdf(WINDKESSEL, g[f"c{c}/theta"], x, inputs.at(t + dt), g[f"c{c}/y"], [True])
    np.testing.assert_array_equal(gl, g[f"c{c}/g"])


def test_nonfinite_state_error_time():
    x = 1e200 * np.random.default_rng(0).normal(size=(64, 8))
    _, t_fail = O.l96_transition([10.0, 0.1], x, 0.3, 0.1, lambda k, d: np.zeros((64, 8)))
    with pytest.raises(NonFiniteStateError) as e:
        S.step_transition(LORENZ96, [10.0, 0.1], x, None, 0.3, 0.1, RngStream(3))
    assert e.value.time == t_fail
    assert abs(e.value.time - 0.35) < 1e-12


# ------------------------------------------------------------------ full filter


def _l96_grid(g, prefix="l96"):
    return build_filter_grid(0.0, 2.0, 20, g["l96/obs_t"], g[f"{prefix}/obs_v"], g[f"{prefix}/obs_m"], n_obs=8)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_pf_l96_host_noise_matches_reference(scheme):
    g = load_golden("pf.npz")
    out = particle_filter(LORENZ96, g["l96/theta"], _l96_grid(g), RngStream(7), n_particles=256,
                          resampler=scheme, noise="host")
    ref = float(g[f"l96/{scheme}/loglik"])
    assert abs(out.loglik - ref) <= 1e-12 * abs(ref)
    np.testing.assert_array_equal(out.run.x, g[f"l96/{scheme}/x_final"])
    assert normwise(out.run.logw, g[f"l96/{scheme}/logw_final"]) <= 1e-12
    np.testing.assert_array_equal(out.trajectory, g[f"l96/{scheme}/traj"])
    anc = np.array([h[1].cpu().numpy() for h in out.run.history[1:] if h[1] is not None])
    np.testing.assert_array_equal(anc, g[f"l96/{scheme}/anc"][1:])


def test_pf_l96_ess_gate_and_sparse_obs():
    g = load_golden("pf.npz")
    out = particle_filter(LORENZ96, g["l96/theta"], _l96_grid(g), RngStream(9), n_particles=256,
                          resampler="systematic", ess_rel=0.5, noise="host")
    ref = float(g["l96/ess/loglik"])
    assert abs(out.loglik - ref) <= 1e-12 * abs(ref)
    np.testing.assert_array_equal(out.trajectory, g["l96/ess/traj"])
    grid = build_filter_grid(0.0, 2.0, 20, g["l96/obs_t"], g["l96s/obs_v"], g["l96s/obs_m"], n_obs=8)
    out = particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(8), n_particles=128,
                          resampler="systematic", noise="host")
    ref = float(g["l96s/loglik"])
    assert abs(out.loglik - ref) <= 1e-12 * abs(ref)
    np.testing.assert_array_equal(out.trajectory, g["l96s/traj"])


@pytest.mark.parametrize("scheme", ["multinomial", "systematic"])
def test_pf_windkessel_host_noise_matches_reference(scheme):
    g = load_golden("pf.npz")
    inputs = LocfInputs(g["wk/in_times"], g["wk/in_values"])
    grid = build_filter_grid(0.0, 1.0, 100, np.linspace(0, 1, 101)[1:], g["wk/obs_v"], np.ones((100, 1), bool),
                             n_obs=1)
    out = particle_filter(WINDKESSEL, g["wk/theta"], grid, RngStream(7), inputs=inputs, n_particles=1024,
                          resampler=scheme, noise="host")
    ref = float(g[f"wk/{scheme}/loglik"])
    assert abs(out.loglik - ref) <= 1e-12 * abs(ref)
    assert normwise(out.trajectory, g[f"wk/{scheme}/traj"]) <= 1e-12


def test_pf_f32_host_noise_close():
    g = load_golden("pf.npz")
    out = particle_filter(LORENZ96, g["l96/theta"], _l96_grid(g), RngStream(7), n_particles=256,
                          resampler="systematic", noise="host", dtype="float32", exact=False)
    ref = float(g["l96/systematic/loglik"])
    # chaotic model + ancestor flips: statistical agreement, not per-step
    assert abs(out.loglik - ref) <= 0.05 * abs(ref)


def test_pf_windkessel_device_noise_unbiased_vs_kalman():
    g = load_golden("pf.npz")
    kf = float(g["wk/kf_loglik"])
    inputs = LocfInputs(g["wk/in_times"], g["wk/in_values"])
    grid = build_filter_grid(0.0, 1.0, 100, np.linspace(0, 1, 101)[1:], g["wk/obs_v"], np.ones((100, 1), bool),
                             n_obs=1)
    runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=4096, resampler="systematic")
    res = runner.run_batch([g["wk/theta"]] * 64, [None] * 64, [RngStream(1000 + k) for k in range(64)])
    ll = np.array([r[0] for r in res])
    se = ll.std(ddof=1) / np.sqrt(len(ll))
    assert abs(ll.mean() - kf) < 4 * se + 0.02, (ll.mean(), kf, se)


def test_batched_equals_single_device_noise():
    g = load_golden("pf.npz")
    grid = _l96_grid(g)
    thetas = [np.array([10.0, 0.1]), np.array([9.0, 0.2]), np.array([11.0, 0.05])]
    runner = FilterRunner(LORENZ96, grid, n_particles=3000, resampler="systematic")
    batch = runner.run_batch(thetas, [None] * 3, [RngStream(50 + k) for k in range(3)])
    for k, th in enumerate(thetas):
        ll, traj, _ = runner.run(th, None, RngStream(50 + k))
        assert ll == batch[k][0]
        np.testing.assert_array_equal(traj, batch[k][1])


def test_run_protocol_resume_and_clone():
    g = load_golden("pf.npz")
    grid = _l96_grid(g)
    rng = RngStream(11)
    a = ParticleRun(LORENZ96, g["l96/theta"], grid, n_particles=2048, resampler="stratified").init(rng.child(0))
    a.advance_to(7, rng.child(1))
    b = a.clone()
    inc_a = a.advance_to(20, rng.child(1))
    inc_b = b.advance_to(20, rng.child(1))
    assert inc_a == inc_b and a.loglik == b.loglik and a.pos == b.pos == 20
    c = ParticleRun(LORENZ96, g["l96/theta"], grid, n_particles=2048, resampler="stratified").init(rng.child(0))
    c.advance_to(20, rng.child(1))
    assert c.loglik == a.loglik
    t = a.sample_trajectory(rng.child(2))
    assert t.shape == (21, 8)
    assert 1.0 <= a.ess() <= 2048.0


def test_degenerate_ensemble_error():
    g = load_golden("pf.npz")
    obs_v = g["l96/obs_v"].copy()
    obs_v[4] = 1e300
    grid = build_filter_grid(0.0, 2.0, 20, g["l96/obs_t"], obs_v, g["l96/obs_m"], n_obs=8)
    with pytest.raises(DegenerateEnsembleError) as e:
        particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(7), n_particles=512)
    assert abs(e.value.time - grid.times[5]) < 1e-12


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("P_in,P_out", [(1000, 7), (7, 1000), (4096, 4096), (3, 1), (50000, 123457)])
def test_search_ragged_sizes(scheme, P_in, P_out):
    """resample(..., size=P_out) with P_out != len(weights) (resampling.py:25)."""
    rs = np.random.default_rng(P_in * 7 + P_out)
    w = np.exp(rs.normal(0, 2, P_in))
    w[rs.random(P_in) < 0.3] = 0.0
    if w.sum() == 0:
        w[0] = 1.0
    cum = O.cumulative(w)
    u = rs.random(1 if scheme == "systematic" else P_out)
    ref = O.search(cum, O.queries(scheme, u, P_out))
    np.testing.assert_array_equal(search_cdf(cum, u, scheme, P_out=P_out), ref)
    np.testing.assert_array_equal(resample(w, scheme, FixedU(u), size=P_out), O.resample_with(w, scheme, u, size=P_out))


@pytest.mark.parametrize("scheme", SCHEMES)
def test_filter_resampler_degenerate_weights(scheme):
    """All weight on one particle / uniform weights through the filter path."""
    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    P = 1 << 16
    for a_np in (np.full(P, -50.0), np.where(np.arange(P) == 1234, 0.0, -1e4)):
        a = torch.from_numpy(a_np).cuda()
        from scipy.special import logsumexp

        shift = torch.tensor([logsumexp(a_np)], dtype=torch.float64, device="cuda")
        ws = torch.empty(L.ssm_resample_workspace_bytes(1, P), dtype=torch.uint8, device="cuda")
        anc = torch.empty(P, dtype=torch.int32, device="cuda")
        u = torch.tensor(np.random.default_rng(1).random(1 if scheme == "systematic" else P), device="cuda")
        _lib.check(L.ssm_resample_from_logw(1, P, 1, _lib.SCHEME_IDS[scheme], _lib.ptr(a), _lib.ptr(shift), None,
                                            _lib.ptr(u), None, 1, _lib.ptr(anc), _lib.ptr(ws), _lib.stream_ptr()))
        ref = O.resample_with(np.exp(a_np - logsumexp(a_np)), scheme, u.cpu().numpy())
        np.testing.assert_array_equal(anc.cpu().numpy(), ref)


def _tile_inputs(a_np):
    """cdf_local / tile_rec / fs exactly as the fused kernel documents them
    (include/ssm_b200.h ssm_tile_rec): per 32-particle tile, m_w >= max a_j,
    q_j = rint(exp(a_j - m_w) 2^52), cdf_local = tile-inclusive prefix of q."""
    from scipy.special import logsumexp

    from paper_1306_3277_b200 import _lib

    P = a_np.size
    nt = (P + 31) // 32
    pad = np.full(nt * 32, -np.inf)
    pad[:P] = a_np
    t = pad.reshape(nt, 32)
    m = t.max(axis=1)
    q = np.rint(np.exp(t - m[:, None]) * 2.0**52).astype(np.uint64)
    cdf = np.cumsum(q, axis=1, dtype=np.uint64).reshape(-1)[:P]
    rec = np.zeros(nt, dtype=[("m", "<f8"), ("Q", "<u8")])
    rec["m"], rec["Q"] = m, q.sum(axis=1, dtype=np.uint64)
    fs = np.zeros(1, dtype=_lib.FILTER_STATE_DTYPE)
    fs["incr"], fs["resample_now"] = logsumexp(a_np), 1
    fs["err_nonfinite"] = fs["err_degenerate"] = _lib.INT32_MAX
    dev = torch.device("cuda")
    as_dev = lambda arr: torch.from_numpy(arr.view(np.uint8).copy()).to(dev)  # noqa: E731
    return as_dev(cdf), as_dev(rec), as_dev(fs), np.exp(a_np - logsumexp(a_np))


def _heavy_patterns(P):
    r = np.random.default_rng(11)
    one = np.full(P, -1e4)
    one[P // 3] = 0.0
    few = np.full(P, -30.0)
    few[[5, 6, min(4000, P - 3), P // 2, P - 1]] = 0.0  # runs of ~P/5 outputs (> one block window)
    cluster = np.zeros(P)  # long runs inside staged block windows (<= 4096 outputs)
    cluster[10], cluster[min(3000, P - 1)] = np.log(1000.0), np.log(40.0)
    lognorm = r.normal(0.0, 3.0, P)  # mixed: long and short runs, ragged windows
    return {"one": one, "few": few, "cluster": cluster, "lognormal": lognorm}


@pytest.mark.parametrize("scheme", ["systematic", "stratified"])
@pytest.mark.parametrize("P", [1 << 16, 50001])
@pytest.mark.parametrize("pattern", ["one", "few", "cluster", "lognormal"])
def test_tiles_resample_heavy_runs_match_oracle(scheme, P, pattern):
    """Filter-path resampler (ssm_resample_from_tiles): staged block windows,
    the heavy-block fallback and chunked long runs give the reference's
    ancestors."""
    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    a_np = _heavy_patterns(P)[pattern]
    cdf, rec, fs, w = _tile_inputs(a_np)
    u_np = np.random.default_rng(3).random(1 if scheme == "systematic" else P)
    u = torch.from_numpy(u_np).cuda()
    ws = torch.empty(L.ssm_resample_workspace_bytes(1, P), dtype=torch.uint8, device="cuda")
    anc = torch.full((P,), -7, dtype=torch.int32, device="cuda")
    _lib.check(L.ssm_resample_from_tiles(1, P, _lib.SCHEME_IDS[scheme], _lib.ptr(cdf), _lib.ptr(rec),
                                         _lib.ptr(fs), _lib.ptr(u), None, 1, _lib.ptr(anc), _lib.ptr(ws),
                                         _lib.stream_ptr()))
    np.testing.assert_array_equal(anc.cpu().numpy(), O.resample_with(w, scheme, u_np))


def _pw_direct(x, theta, keys, d, hints, y, exact=False, anc=None, dtype="float64", tiles=None, obs_mask=0xFF,
               fs_out=None):
    """One ssm_propagate_weight launch with device noise (C ABI), returns x_out, a_out."""
    from paper_1306_3277_b200 import _lib
    from paper_1306_3277_b200.inference.particle import _fs_init, _dtype_info
    from paper_1306_3277_b200.models import LOG_SQRT_2PI

    L = _lib.lib()
    _, tdt, dt_id = _dtype_info(dtype)
    P = x.shape[0]
    dev = torch.device("cuda")
    xin = torch.from_numpy(np.ascontiguousarray(x.T)).to(dev, tdt)
    xout = torch.empty_like(xin)
    sub = np.zeros(1, dtype=_lib.SUBSTEP_DTYPE)
    sub[0]["d"], sub[0]["sd"], sub[0]["n_ode"] = d, np.sqrt(d), 1
    sub[0]["s"][0] = min(0.05, d)
    subs = torch.from_numpy(sub.view(np.uint8).copy()).to(dev)
    th = torch.from_numpy(LORENZ96.derived(theta)).to(dev)
    kt = torch.from_numpy(np.asarray(keys, dtype=np.uint32).view(np.int32).reshape(1, 2)).to(dev)
    fs = _fs_init(1, dev)
    ws = torch.empty(L.ssm_pw_workspace_bytes(1, P), dtype=torch.uint8, device=dev)
    a = torch.empty(P, dtype=tdt, device=dev)
    A = _lib.PwArgs()
    A.model, A.dtype, A.B, A.P, A.step, A.n_sub = 0, dt_id, 1, P, 3, 1
    A.exact, A.check_finite, A.has_obs, A.obs_mask = int(exact), 1, 1, obs_mask
    for n in range(8):
        A.y[n] = float(y[n])
    A.log_w0, A.obs_log_sd, A.log_sqrt_2pi, A.ess_rel = -np.log(P), np.log(0.5), LOG_SQRT_2PI, -1.0
    A.x_in, A.x_out, A.a_out, A.theta, A.subs = xin.data_ptr(), xout.data_ptr(), a.data_ptr(), th.data_ptr(), subs.data_ptr()
    A.keys, A.fs, A.workspace, A.hints = kt.data_ptr(), fs.data_ptr(), ws.data_ptr(), hints
    if tiles is not None:
        cloc = torch.empty(P, dtype=torch.int64, device=dev)
        trec = torch.empty(((P + 31) // 32) * 16, dtype=torch.uint8, device=dev)
        A.cdf_local, A.tile_rec = cloc.data_ptr(), trec.data_ptr()
    _lib.check(L.ssm_propagate_weight(A, _lib.stream_ptr()))
    if tiles is not None:
        rec = trec.cpu().numpy().view([("m", "<f8"), ("Q", "<u8")])
        tiles.update(cdf=cloc.cpu().numpy().view(np.uint64), m=rec["m"], Q=rec["Q"])
    if fs_out is not None:
        fs_out.update(err_nonfinite=int(fs.cpu().numpy().reshape(-1).view(_lib.FILTER_STATE_DTYPE)["err_nonfinite"][0]))
    return xout.t().double().cpu().numpy(), a.double().cpu().numpy()


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("d", [0.05, 0.04999999999999999, 0.05000000000000002])
@pytest.mark.parametrize("mask", [0xFF, 0x0F, 0x81])
def test_specialised_kernel_equals_general(dtype, d, mask):
    """The SIMPLE (single sub-step) fused kernel must compute the same step as
    the general kernel (same device draws), for full and partial observation masks."""
    rs = np.random.default_rng(3)
    P = 5000
    x = rs.uniform(-1, 3, (P, 8))
    y = rs.normal(0, 3, 8)
    keys = [123456789, 987654321]
    x1, a1 = _pw_direct(x, [10.0, 0.1], keys, d, 1, y, dtype=dtype, obs_mask=mask)
    x0, a0 = _pw_direct(x, [10.0, 0.1], keys, d, 0, y, dtype=dtype, obs_mask=mask)
    tol = 1e-12 if dtype == "float64" else 1e-5
    assert normwise(x1, x0) <= tol
    assert normwise(a1, a0) <= tol


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("mask", [0xFF, 0x0F])
@pytest.mark.parametrize("bad", ["none", "inf", "nan"])
def test_fused_nonfinite_flag_both_kernels(dtype, mask, bad):
    """Non-finite states are flagged at the step (err = step * 64 + sub-step) by the
    SIMPLE kernel (whose full-observation path checks through the observation sum)
    and by the general kernel alike; finite states are never flagged."""
    rs = np.random.default_rng(4)
    P = 3000
    x = rs.uniform(-1, 3, (P, 8))
    if bad == "inf":
        x[1234, 5] = 1e200  # overflows inside RK4
    elif bad == "nan":
        x[77, 0] = np.nan
    y = rs.normal(0, 3, 8)
    for hints in (1, 0):
        fs = {}
        _pw_direct(x, [10.0, 0.1], [5, 6], 0.05, hints, y, dtype=dtype, obs_mask=mask, fs_out=fs)
        want = 3 * 64 if bad != "none" else np.iinfo(np.int32).max
        assert fs["err_nonfinite"] == want, (hints, fs)


def test_fast_device_noise_filter_tracks_exact():
    """Fast (FMA) and exact float64 filters share the device draws, so over a
    short window their likelihoods agree to round-off amplification."""
    g = load_golden("pf.npz")
    grid = _l96_grid(g)
    lls = []
    for exact in (True, False):
        out = particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(17), n_particles=1 << 14,
                              resampler="systematic", exact=exact, upto=8)
        lls.append(out.loglik)
    assert abs(lls[0] - lls[1]) <= 1e-6 * abs(lls[0]), lls


@pytest.mark.parametrize("P", [2, 33, 1000, 4097, 70001])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_pf_ragged_sizes_match_oracle(P, scheme):
    """Partial warp tiles, non-power-of-two P and the minimum P=2, with the
    reference's draws: loglik within 1e-12 of the oracle, trajectory bitwise."""
    g = load_golden("pf.npz")
    grid = _l96_grid(g)
    T = 6 if P > 10000 else 12
    out = particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(5 + P), n_particles=P, resampler=scheme,
                          noise="host", upto=T)
    ograd = O.Grid(grid.times, {k + 1: (g["l96/obs_v"][k], g["l96/obs_m"][k]) for k in range(20)})
    ll, traj, _ = O.particle_filter("lorenz96", g["l96/theta"], ograd, O.Stream(5 + P), n_particles=P,
                                    resampler=scheme, upto=T)
    assert abs(out.loglik - ll) <= 1e-12 * abs(ll), (out.loglik, ll)
    np.testing.assert_array_equal(out.trajectory, traj)


def test_pf_upto_zero_and_unobserved_steps():
    g = load_golden("pf.npz")
    grid = _l96_grid(g)
    out = particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(1), n_particles=64, upto=0)
    assert out.loglik == 0.0 and out.trajectory.shape == (1, 8)
    # all observations masked: pure propagation, loglik stays 0, no resampling
    masked = build_filter_grid(0.0, 2.0, 20, g["l96/obs_t"], g["l96/obs_v"], np.zeros_like(g["l96/obs_m"]), n_obs=8)
    out = particle_filter(LORENZ96, g["l96/theta"], masked, RngStream(1), n_particles=5000, resampler="systematic")
    assert out.loglik == 0.0
    assert all(h[1] is None or np.array_equal(h[1].cpu().numpy(), np.arange(5000)) for h in out.run.history[1:])


@pytest.mark.parametrize("P", [64, 5000])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_trajectory_pick_on_uniform_weights_matches_oracle(P, scheme):
    """The final multinomial pick when the last weights are uniform -- at upto=0
    and after trailing unobserved grid steps (the resample that follows the last
    observation leaves uniform weights) -- draws from the run's stream like the
    reference (particle.py:137-149): trajectories bitwise the oracle's, and
    different streams pick different particles."""
    g = load_golden("pf.npz")
    grid = _l96_grid(g)
    og = O.Grid(grid.times, {k + 1: (g["l96/obs_v"][k], g["l96/obs_m"][k]) for k in range(20)})
    for seed in (3, 4):
        out = particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(seed), n_particles=P, resampler=scheme,
                              noise="host", upto=0)
        ll, traj, _ = O.particle_filter("lorenz96", g["l96/theta"], og, O.Stream(seed), n_particles=P,
                                        resampler=scheme, upto=0)
        assert out.loglik == ll == 0.0
        np.testing.assert_array_equal(out.trajectory, traj)
    # observations only on the first 14 of 20 steps: the last 6 propagate with uniform weights
    mask = g["l96/obs_m"].copy()
    mask[14:] = False
    tgrid = build_filter_grid(0.0, 2.0, 20, g["l96/obs_t"], g["l96/obs_v"], mask, n_obs=8)
    otg = O.Grid(tgrid.times, {k + 1: (g["l96/obs_v"][k], mask[k]) for k in range(20)})
    picks = set()
    for seed in (5, 6, 7):
        out = particle_filter(LORENZ96, g["l96/theta"], tgrid, RngStream(seed), n_particles=P, resampler=scheme,
                              noise="host")
        ll, traj, _ = O.particle_filter("lorenz96", g["l96/theta"], otg, O.Stream(seed), n_particles=P,
                                        resampler=scheme)
        assert abs(out.loglik - ll) <= 1e-12 * abs(ll)
        np.testing.assert_array_equal(out.trajectory, traj)
        picks.add(tuple(np.round(traj[-1], 12)))
    assert len(picks) > 1


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("P", [3000, 100000])
def test_device_noise_ess_gate_runs(scheme, P):
    """ESS gate with device noise on both the persistent (small P) and the
    multi-kernel path: runs, finite, and resamples less often than without."""
    g = load_golden("pf.npz")
    grid = _l96_grid(g)
    out = particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(3), n_particles=P, resampler=scheme,
                          ess_rel=0.5)
    assert np.isfinite(out.loglik)
    assert out.trajectory.shape == (21, 8)


@pytest.mark.parametrize("P", [4096, 1000])
def test_tile_records_match_documented_format(P):
    """cdf_local / tile_rec from the fused kernel (include/ssm_b200.h):
    m_w >= max a_j of the tile and float-representable, cdf_local the tile-inclusive
    prefix of q_j = round(exp(a_j - m_w) 2^52) (kernel exp within a few ulp), Q_w
    the tile total."""
    r = np.random.default_rng(5)
    x = r.normal(0.0, 3.0, (P, 8))
    y = r.normal(0.0, 1.0, 8)
    tiles = {}
    _, a = _pw_direct(x, np.array([8.0, 0.1]), (7, 9), 0.05, 1, y, tiles=tiles)
    nt = (P + 31) // 32
    for w in range(nt):
        aw = a[32 * w: 32 * w + 32]
        m = tiles["m"][w]
        assert m >= aw.max() and np.float32(m) == m
        q = np.rint(np.exp(aw - m) * 2.0**52)
        cdf = tiles["cdf"][32 * w: 32 * w + aw.size]
        d = np.diff(np.concatenate([np.zeros(1, np.uint64), cdf])).astype(np.float64)  # each q_j <= 2^52: exact
        assert np.all(np.abs(d - q) <= 4.0 + q * 1e-15), (w, np.max(np.abs(d - q)))
        assert tiles["Q"][w] == tiles["cdf"][32 * w + aw.size - 1]


def _philox4x32_10(ctr, k0, k1):
    """numpy restatement of the device Philox4x32-10 (ssm_common.cuh) for test oracles."""
    M0, M1, W0, W1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57), 0x9E3779B9, 0xBB67AE85
    c = [np.asarray(x, dtype=np.uint64) & np.uint64(0xFFFFFFFF) for x in ctr]
    k0, k1 = int(k0), int(k1)
    for _ in range(10):
        p0, p1 = M0 * c[0], M1 * c[2]
        lo0, hi0 = p0 & np.uint64(0xFFFFFFFF), p0 >> np.uint64(32)
        lo1, hi1 = p1 & np.uint64(0xFFFFFFFF), p1 >> np.uint64(32)
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
        k0, k1 = (k0 + W0) & 0xFFFFFFFF, (k1 + W1) & 0xFFFFFFFF
    return c


@pytest.mark.parametrize("P", [1000, 2048, 5000, 1 << 16, 1 << 18])
@pytest.mark.parametrize("pattern", ["lognormal", "one", "few", "sigma10"])
def test_sorted_multinomial_matches_spacings_oracle(P, pattern):
    """SSM_MULTINOMIAL_SORTED (device-noise filter path): U_(k) = S_k / S_{P+1}
    from the device's exponential spacings, ancestors = searchsorted(cum, U, 'right')
    -- restated in numpy from the same Philox words (B = 2 filters, ragged P,
    degenerate weights); ancestors ascending."""
    from scipy.special import logsumexp

    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    pats = _heavy_patterns(P)
    pats["sigma10"] = np.random.default_rng(1234).normal(0.0, 10.0, size=P)  # ESS ~ 1
    a_np = np.stack([pats[pattern], pats["lognormal"]])
    a = torch.from_numpy(a_np).cuda()
    shift = torch.from_numpy(logsumexp(a_np, axis=1)).cuda()
    keys_np = np.array([[11, 22], [33, 44]], dtype=np.uint32)
    keys = torch.from_numpy(keys_np.view(np.int32)).cuda()
    ws = torch.empty(L.ssm_resample_workspace_bytes(2, P), dtype=torch.uint8, device="cuda")
    anc = torch.full((2, P), -1, dtype=torch.int32, device="cuda")
    step = 5
    _lib.check(L.ssm_resample_from_logw(2, P, 1, _lib.SSM_MULTINOMIAL_SORTED, _lib.ptr(a), _lib.ptr(shift), None,
                                        None, _lib.ptr(keys), step, _lib.ptr(anc), _lib.ptr(ws), _lib.stream_ptr()))
    got = anc.cpu().numpy()
    k = np.arange(P + 1, dtype=np.uint64)
    for b in range(2):
        # spacing k: Philox block k // 2, words (x, y) for even k and (z, w) for odd k
        r = _philox4x32_10([k >> np.uint64(1), np.full(P + 1, step), np.zeros(P + 1), np.full(P + 1, 5)],
                           *keys_np[b])
        odd = (k & np.uint64(1)).astype(bool)
        u = np.where(odd, (r[2] << np.uint64(32)) | r[3], (r[0] << np.uint64(32)) | r[1]) >> np.uint64(11)
        E = -np.log(1.0 - u.astype(np.float64) * 2.0**-53)
        S = np.cumsum(E)
        U = S[:P] / S[P]
        w = np.exp(a_np[b] - logsumexp(a_np[b]))
        cum = np.cumsum(w / w.sum())
        cum[-1] = 1.0
        ref = np.searchsorted(cum, U, side="right").clip(0, P - 1)
        assert np.all(np.diff(got[b]) >= 0)
        np.testing.assert_array_equal(got[b], ref)


@pytest.mark.parametrize("P", [1000, 1 << 16])
@pytest.mark.parametrize("pattern", ["lognormal", "few"])
def test_sorted_multinomial_from_tiles_matches_logw(P, pattern):
    """The filter path's sorted multinomial from the fused kernel's tile records
    equals the one from the log-weight scan (same spacings, same CDF up to the
    fixed-point rounding)."""
    from scipy.special import logsumexp

    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    a_np = _heavy_patterns(P)[pattern]
    cdf, rec, fs, _ = _tile_inputs(a_np)
    keys = torch.tensor([[77, 88]], dtype=torch.int32, device="cuda")
    ws = torch.empty(L.ssm_resample_workspace_bytes(1, P), dtype=torch.uint8, device="cuda")
    anc_t = torch.full((P,), -1, dtype=torch.int32, device="cuda")
    _lib.check(L.ssm_resample_from_tiles(1, P, _lib.SSM_MULTINOMIAL_SORTED, _lib.ptr(cdf), _lib.ptr(rec),
                                         _lib.ptr(fs), None, _lib.ptr(keys), 3, _lib.ptr(anc_t), _lib.ptr(ws),
                                         _lib.stream_ptr()))
    a = torch.from_numpy(a_np).cuda()
    shift = torch.tensor([logsumexp(a_np)], dtype=torch.float64, device="cuda")
    anc_l = torch.full((P,), -1, dtype=torch.int32, device="cuda")
    _lib.check(L.ssm_resample_from_logw(1, P, 1, _lib.SSM_MULTINOMIAL_SORTED, _lib.ptr(a), _lib.ptr(shift), None,
                                        None, _lib.ptr(keys), 3, _lib.ptr(anc_l), _lib.ptr(ws), _lib.stream_ptr()))
    np.testing.assert_array_equal(anc_t.cpu().numpy(), anc_l.cpu().numpy())


@pytest.mark.parametrize("kw", [
    dict(resampler="systematic"),
    dict(resampler="multinomial"),
    dict(resampler="stratified", exact=True),
    dict(resampler="systematic", dtype="float32"),
    dict(resampler="systematic", ess_rel=0.5),
    dict(resampler="multinomial", initial_state=np.linspace(-0.5, 2.5, 8)),
    dict(resampler="systematic", sparse=True),
])
def test_history_free_replay_equals_stored_history(kw):
    """keep_history=False stores only ancestors; sample_trajectory replays the
    chosen line with the fused kernel's transition: bitwise the same trajectory
    (and the same log-likelihood) as the run that keeps every position."""
    kw = dict(kw)
    sparse = kw.pop("sparse", False)
    theta = np.array([10.0, 0.1])
    times = np.linspace(0.0, 1.0, 21)
    obs = O.simulate_l96(theta, times, O.Stream(3), obs_slots=range(4) if sparse else range(8),
                         obs_every=2 if sparse else 1)
    ov = np.array([obs[k][0] for k in range(1, 21)])
    om = np.array([obs[k][1] for k in range(1, 21)])
    grid = build_filter_grid(0.0, 1.0, 20, times[1:], ov, om, n_obs=8)
    outs = [particle_filter(LORENZ96, theta, grid, RngStream(11), n_particles=9000, keep_history=kh, **kw)
            for kh in (True, False)]
    assert outs[0].loglik == outs[1].loglik
    np.testing.assert_array_equal(outs[0].trajectory, outs[1].trajectory)
    with pytest.raises(ValueError):
        _ = outs[1].run.history
    if kw.get("resampler") in ("systematic", "stratified"):  # ancestors ascending, in range (ESS-held steps: identity)
        for _, anc in outs[0].run.history[1:]:
            if anc is not None:
                a = anc.cpu().numpy()
                assert a.min() >= 0 and a.max() < 9000 and np.all(np.diff(a) >= 0)


def test_history_free_windkessel_and_resume():
    theta = np.array([1.8, 3.0, 0.06, 25.0])
    times = np.linspace(0.0, 0.5, 51)
    tin = np.round(np.arange(0, 0.51, 0.01), 10)
    inputs = LocfInputs(tin, O.windkessel_flow(tin))
    ys = 90.0 + np.zeros((50, 1))
    grid = build_filter_grid(0.0, 0.5, 50, times[1:], ys, np.ones((50, 1), bool), n_obs=1)
    trajs = []
    for kh in (True, False):
        run = ParticleRun(WINDKESSEL, theta, grid, inputs=inputs, n_particles=6000, resampler="systematic",
                          keep_history=kh)
        run.init(RngStream(5).child(0))
        run.advance_to(20, RngStream(5).child(1))
        run.advance_to(50, RngStream(5).child(2))  # second call: different device keys per segment
        trajs.append(run.sample_trajectory(RngStream(5).child(3)))
    np.testing.assert_array_equal(trajs[0], trajs[1])


@pytest.mark.parametrize("exact", [True, False])
def test_small_and_multikernel_paths_share_the_transition(exact, monkeypatch):
    """The persistent small-P kernel and the fused multi-kernel path run the same
    per-particle transition code (ssm_models.cuh): the first grid step (no
    resampling yet) gives bitwise-equal states from the same device draws."""
    from paper_1306_3277_b200.inference import particle as particle_mod

    g = load_golden("pf.npz")
    grid = _l96_grid(g)
    small = particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(3), n_particles=3000, upto=1, exact=exact)
    monkeypatch.setattr(particle_mod, "_NO_SMALL", True)
    multi = particle_filter(LORENZ96, g["l96/theta"], grid, RngStream(3), n_particles=3000, upto=1, exact=exact)
    np.testing.assert_array_equal(small.run.x, multi.run.x)
    if exact:
        np.testing.assert_array_equal(small.run.logw, multi.run.logw)
    else:
        assert normwise(small.run.logw, multi.run.logw) <= 1e-12


def _random_weights(seed, P, sigma, zero_frac, ties):
    r = np.random.default_rng(seed)
    w = np.exp(sigma * r.normal(size=P))
    if ties:
        w = np.round(w, 1) + 0.0
    w[r.random(P) < zero_frac] = 0.0
    if not np.any(w > 0):
        w[r.integers(P)] = 1.0
    return w


def test_resample_randomised_vs_oracle():
    """Property test (hypothesis): for random sizes (ragged, non-power-of-two,
    resampled size != P), weight shapes (log-normal spread up to degenerate,
    exact zeros, tied values) and all three schemes, the device resample()
    returns exactly the oracle's searchsorted ancestors for the same uniforms."""
    from hypothesis import HealthCheck, given, settings
    from hypothesis import strategies as st

    @settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
    @given(seed=st.integers(0, 2**31 - 1), P=st.integers(2, 9000), sigma=st.sampled_from([0.0, 0.5, 3.0, 12.0]),
           zero_frac=st.sampled_from([0.0, 0.3, 0.95]), ties=st.booleans(), scheme=st.sampled_from(SCHEMES),
           size_factor=st.sampled_from([None, 0.5, 1.7]))
    def check(seed, P, sigma, zero_frac, ties, scheme, size_factor):
        w = _random_weights(seed, P, sigma, zero_frac, ties)
        size = None if size_factor is None else max(1, int(P * size_factor))
        n = P if size is None else size
        r = np.random.default_rng(seed + 1)
        u = r.random(1 if scheme == "systematic" else n)
        got = resample(w, scheme, FixedU(u), size=size)
        want = O.resample_with(w, scheme, u, size=size)
        np.testing.assert_array_equal(got, want)

    check()

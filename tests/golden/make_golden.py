"""Generate golden vectors by running the REFERENCE itself.

Run in this container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package `ssmkit` from /root/reference/pkg/src and
writes small .npz fixtures next to this file.  The fixtures pin the CPU
oracle (`oracle/ssm_oracle.py`) and the CUDA path (`tests/test_gpu_*.py`).
Numpy/scipy versions are recorded in every file.
"""

import math
import os
import sys

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import ssmkit  # noqa: E402  (the reference)
from ssmkit import RngStream, load_model  # noqa: E402
from ssmkit.core import simulate  # noqa: E402
from ssmkit.inference import build_filter_grid, particle_filter, resample  # noqa: E402
from scipy.special import logsumexp  # noqa: E402

MODELS = "/root/reference/pkg/models"
VERSIONS = dict(numpy=np.__version__, scipy=scipy.__version__, ssmkit=ssmkit.__version__)


def load(name):
    path = {"lorenz96": "lorenz96/Lorenz96.bi", "windkessel": "windkessel/Windkessel.bi"}[name]
    with open(os.path.join(MODELS, path)) as fh:
        return load_model(fh.read())


def save(name, **arrays):
    arrays["versions"] = np.array(repr(VERSIONS))
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrays.items()})


class FixedU:
    """Duck-typed rng for `resample`: returns scripted uniforms."""

    def __init__(self, u):
        self.u = np.asarray(u, dtype=float)

    def uniform(self, low=0.0, high=1.0, size=None):
        if size is None:
            return float(self.u[0])
        return self.u[:size].copy()


class LocfInputs:
    """Last-observation-carried-forward input provider (timeseries.py:184-210
    semantics, rtol 1e-9) over a fixed (times, values) table."""

    def __init__(self, times, values):
        self.times = np.asarray(times, dtype=float)
        self.values = np.asarray(values, dtype=float)

    def at(self, t):
        tol = 1e-9 * max(1.0, abs(t))
        idx = int(np.searchsorted(self.times, t + tol, side="right")) - 1
        return self.values[idx]


def flow(t, f_max=500.0, t_s=0.3, t_d=0.5):
    tp = np.mod(t, t_s + t_d)
    return np.where(tp < t_s, f_max * np.sin(np.pi * tp / t_s) ** 2, 0.0)


def gen_resample():
    rs = np.random.default_rng(20260101)
    out = {}
    cases = []
    # (name, weights)
    cases.append(("onehot", np.array([1.0, 0.0, 0.0, 0.0])))
    cases.append(("half", np.array([0.5, 0.5])))
    cases.append(("ties", np.array([0.25, 0.25, 0.5])))
    cases.append(("zeros_mixed", np.where(rs.random(37) < 0.4, 0.0, rs.random(37))))
    cases.append(("lognormal_1k", np.exp(rs.normal(0.0, 3.0, 1000))))
    cases.append(("uniform_4097", np.ones(4097)))
    cases.append(("degenerate_2k", np.exp(rs.normal(0.0, 40.0, 2048))))
    cases.append(("tiny_16384", np.exp(rs.normal(-700.0, 2.0, 16384))))
    for name, w in cases:
        P = w.size
        cum = np.cumsum(w / w.sum())
        cum[-1] = 1.0
        out[f"{name}/w"] = w
        out[f"{name}/cum"] = cum
        for scheme in ("multinomial", "stratified", "systematic"):
            u = rs.random(P) if scheme != "systematic" else rs.random(1)
            anc = resample(w, scheme, FixedU(u))
            out[f"{name}/{scheme}/u"] = u
            out[f"{name}/{scheme}/anc"] = anc
    # tie KAT from SURVEY 4: u exactly on cum boundaries
    w = np.array([0.25, 0.25, 0.5])
    u = np.array([0.25, 0.0, 0.4999999, 0.5, 0.9999])
    out["kat_ties/w"] = w
    out["kat_ties/u"] = u
    out["kat_ties/anc"] = resample(w, "multinomial", FixedU(u), size=5)
    save("resample.npz", **out)


def gen_lse():
    rs = np.random.default_rng(7)
    arrs = {
        "normal": rs.normal(0, 1, 1000),
        "wide": rs.normal(0, 50, 4096),
        "ties": np.array([3.0, 3.0, 1.0, -2.0, 3.0]),
        "with_ninf": np.array([-np.inf, 0.5, -np.inf, 0.25]),
        "one_dominant": np.concatenate([[0.0], np.full(1023, -60.0)]),
    }
    out = {}
    for k, a in arrs.items():
        out[f"{k}/a"] = a
        out[f"{k}/lse"] = np.array(logsumexp(a))
    save("lse.npz", **out)


def gen_l96_step():
    ir = load("lorenz96")
    rs = np.random.default_rng(11)
    out = {}
    P = 257
    for c, (dt, theta) in enumerate(
        [
            (0.05, (10.0, 0.1)),
            (0.05000000000000002, (10.0, 0.1)),
            (0.1, (8.5, 0.3)),
            (0.07, (11.9, 0.05)),
            (0.03, (10.0, 0.0)),
        ]
    ):
        x = rs.uniform(-1.0, 3.0, (P, 8)) * (1.0 + 4.0 * (c % 2))
        theta = np.array(theta)
        t = 0.35
        seed = 100 + c
        x_out = simulate.step_transition(ir, theta, x, None, t, dt, RngStream(seed))
        # replay the exact draws: per sub-step, 8 slot-major normal(0, sqrt(d), P)
        rng = RngStream(seed)
        W = []
        for t_k, d in simulate.substep_schedule(t, dt, ir.delta):
            for n in range(8):
                W.append(rng.normal(0.0, math.sqrt(d), size=P))
        W = np.array(W).reshape(-1, 8, P)
        y = rs.normal(0.0, 3.0, 8)
        mask = rs.random(8) < 0.7
        mask[0] = True
        g = simulate.observe_logpdf(ir, theta, x_out, None, y, mask)
        g_all = simulate.observe_logpdf(ir, theta, x_out, None, y, np.ones(8, bool))
        out.update(
            {
                f"c{c}/x_in": x,
                f"c{c}/theta": theta,
                f"c{c}/t": np.array(t),
                f"c{c}/dt": np.array(dt),
                f"c{c}/W": W,
                f"c{c}/x_out": x_out,
                f"c{c}/y": y,
                f"c{c}/mask": mask,
                f"c{c}/g": g,
                f"c{c}/g_all": g_all,
            }
        )
    out["ncases"] = np.array(5)
    # fixed point KAT: sigma2 = 0, x = F
    xf = np.full((4, 8), 10.0)
    out["fixed/x_out"] = simulate.step_transition(ir, np.array([10.0, 0.0]), xf, None, 0.0, 0.05, RngStream(1))
    save("l96_step.npz", **out)


def gen_wk_step():
    ir = load("windkessel")
    rs = np.random.default_rng(12)
    times = np.round(np.arange(0, 2.0001, 0.01), 10)
    inputs = LocfInputs(times, flow(times)[:, None])
    out = {"in_times": times, "in_values": flow(times)}
    P = 300
    for c, (t, dt, theta) in enumerate(
        [
            (0.1, 0.01, (1.8, 3.0, 0.06, 25.0)),
            (0.2, 0.03, (0.9, 1.5, 0.03, 10.0)),
            (0.55, 0.025, (2.4, 4.0, 0.08, 40.0)),
        ]
    ):
        x = rs.normal(90.0, 15.0, (P, 1))
        theta = np.array(theta)
        seed = 200 + c
        x_out = simulate.step_transition(ir, theta, x, inputs, t, dt, RngStream(seed))
        rng = RngStream(seed)
        xi = []
        sd = 0.01 * np.sqrt(theta[None, :][:, 3])
        for t_k, d in simulate.substep_schedule(t, dt, ir.delta):
            xi.append(rng.normal(0.0, sd, size=P))
        y = np.array([rs.normal(95.0, 10.0)])
        u_obs = inputs.at(t + dt)
        g = simulate.observe_logpdf(ir, theta, x_out, u_obs, y, np.array([True]))
        out.update(
            {
                f"c{c}/x_in": x,
                f"c{c}/theta": theta,
                f"c{c}/t": np.array(t),
                f"c{c}/dt": np.array(dt),
                f"c{c}/xi": np.array(xi),
                f"c{c}/x_out": x_out,
                f"c{c}/y": y,
                f"c{c}/g": g,
            }
        )
    out["ncases"] = np.array(3)
    save("wk_step.npz", **out)


def l96_data(obs_every=1, slots=range(8), seed=1, T=40):
    """theta*=(10,0.1), grid linspace(0,2,41), data RngStream(1)."""
    ir = load("lorenz96")
    theta = np.array([10.0, 0.1])
    times = np.linspace(0.0, 2.0, T + 1)
    rng = RngStream(seed)
    x = simulate.sample_initial(ir, theta, rng.child(1), size=1)
    obs_t, obs_v, obs_m = [], [], []
    for k in range(1, len(times)):
        x = simulate.step_transition(ir, theta, x, None, times[k - 1], times[k] - times[k - 1], rng.child(2, k))
        y = simulate.simulate_obs(ir, theta, x, None, rng.child(3, k))[0]
        m = np.zeros(8, bool)
        if k % obs_every == 0:
            m[list(slots)] = True
        obs_t.append(times[k])
        obs_v.append(y)
        obs_m.append(m)
    return ir, theta, times, np.array(obs_t), np.array(obs_v), np.array(obs_m)


def gen_pf():
    out = {}
    ir, theta, times, ot, ov, om = l96_data(T=20)
    T = len(times) - 1
    grid = build_filter_grid(0.0, times[-1], T, ot, ov, om, n_obs=8)
    out["l96/times"] = grid.times
    out["l96/obs_t"] = ot
    out["l96/obs_v"] = ov
    out["l96/obs_m"] = om
    out["l96/theta"] = theta
    for scheme in ("systematic", "multinomial", "stratified"):
        res = particle_filter(ir, theta, grid, RngStream(7), n_particles=256, resampler=scheme)
        out[f"l96/{scheme}/loglik"] = np.array(res.loglik)
        out[f"l96/{scheme}/traj"] = res.trajectory
        out[f"l96/{scheme}/x_final"] = res.run.x
        out[f"l96/{scheme}/logw_final"] = res.run.logw
        out[f"l96/{scheme}/anc"] = np.array([h[1] for h in res.run.history[1:]])
    # ESS-gated run and sparse-observation run
    res = particle_filter(ir, theta, grid, RngStream(9), n_particles=256, resampler="systematic", ess_rel=0.5)
    out["l96/ess/loglik"] = np.array(res.loglik)
    out["l96/ess/traj"] = res.trajectory
    ir, theta, times, ot, ov, om = l96_data(obs_every=2, slots=range(4), T=20)
    grid = build_filter_grid(0.0, times[-1], len(times) - 1, ot, ov, om, n_obs=8)
    out["l96s/obs_v"] = ov
    out["l96s/obs_m"] = om
    res = particle_filter(ir, theta, grid, RngStream(8), n_particles=128, resampler="systematic")
    out["l96s/loglik"] = np.array(res.loglik)
    out["l96s/traj"] = res.trajectory

    # windkessel config 1: P=1024, T=100, theta*=(1.8,3,0.06,25)
    ir = load("windkessel")
    theta = np.array([1.8, 3.0, 0.06, 25.0])
    in_times = np.round(np.arange(0, 1.0001, 0.01), 10)
    inputs = LocfInputs(in_times, flow(in_times)[:, None])
    times = np.linspace(0.0, 1.0, 101)
    rng = RngStream(1)
    x = simulate.sample_initial(ir, theta, rng.child(1), size=1)
    ot, ov, om = [], [], []
    for k in range(1, len(times)):
        x = simulate.step_transition(ir, theta, x, inputs, times[k - 1], times[k] - times[k - 1], rng.child(2, k))
        y = simulate.simulate_obs(ir, theta, x, inputs.at(times[k]), rng.child(3, k))[0]
        ot.append(times[k])
        ov.append(y)
        om.append(np.ones(1, bool))
    ot, ov, om = np.array(ot), np.array(ov), np.array(om)
    grid = build_filter_grid(0.0, 1.0, 100, ot, ov, om, n_obs=1)
    out["wk/in_times"] = in_times
    out["wk/in_values"] = flow(in_times)
    out["wk/obs_v"] = ov
    out["wk/theta"] = theta
    for scheme in ("multinomial", "systematic"):
        res = particle_filter(ir, theta, grid, RngStream(7), inputs=inputs, n_particles=1024, resampler=scheme)
        out[f"wk/{scheme}/loglik"] = np.array(res.loglik)
        out[f"wk/{scheme}/traj"] = res.trajectory
    # exact likelihood from the reference's Kalman filter (statistical oracle)
    from ssmkit.inference import kalman_filter
    from ssmkit.lineargauss import extract_linear_gaussian
    system = extract_linear_gaussian(ir, theta, grid.times, inputs)
    out["wk/kf_loglik"] = np.array(kalman_filter(system, grid, RngStream(0)).loglik)
    save("pf.npz", **out)


def gen_theta_level():
    """Host theta-level blocks (prior, proposals, densities) for both models,
    with the `inf` compile shim for windkessel (SURVEY 8c known defect)."""
    import ssmkit.core.ir as I

    I.compile_expr = lambda e, t, b: eval(
        f"lambda T, X, W, U: {I.expr_source(e, t, b)}", {"np": np, "inf": np.inf, "__builtins__": {}}
    )
    out = {}
    for name in ("lorenz96", "windkessel"):
        ir = load(name)
        th = simulate.sample_parameter(ir, RngStream(3), size=5)
        out[f"{name}/prior_draws"] = th
        out[f"{name}/prior_logpdf"] = np.array([simulate.parameter_logpdf(ir, t) for t in th])
        props, fwd, rev = [], [], []
        for k, t in enumerate(th):
            tn, lq = simulate.propose_parameters(ir, t, RngStream(4, (k,)))
            props.append(tn)
            fwd.append(lq)
            rev.append(simulate.proposal_parameter_logpdf(ir, tn, t))
        out[f"{name}/proposals"] = np.array(props)
        out[f"{name}/logq_fwd"] = np.array(fwd)
        out[f"{name}/logq_rev"] = np.array(rev)
        if ir.block("proposal_initial") is not None:
            x0 = simulate.sample_initial(ir, th, RngStream(5), size=5)
            out[f"{name}/init_draws"] = x0
            out[f"{name}/init_logpdf"] = np.array([simulate.initial_logpdf(ir, th[k], x0[k]) for k in range(5)])
            xp, lq = [], []
            for k in range(5):
                a, b = simulate.propose_initial(ir, th[k], x0[k], RngStream(6, (k,)))
                xp.append(a)
                lq.append(b)
            out[f"{name}/init_props"] = np.array(xp)
            out[f"{name}/init_logq"] = np.array(lq)
            out[f"{name}/init_logq_rev"] = np.array(
                [simulate.proposal_initial_logpdf(ir, th[k], xp[k], x0[k]) for k in range(5)])
    save("theta.npz", **out)


def gen_outer_loops():
    """Reference PMMH (mh_sample) and SMC^2 (smc_sampler) at toy sizes on L96
    sparse data (4 of 8 slots, every other step, T=10), and windkessel PMMH
    (needs the `inf` shim)."""
    from ssmkit.inference import FilterRunner, mh_sample, smc_sampler

    out = {}
    ir, theta, times, ot, ov, om = l96_data(obs_every=2, slots=range(4), T=10)
    grid = build_filter_grid(0.0, times[-1], 10, ot, ov, om, n_obs=8)
    out["l96/times"] = times
    out["l96/obs_v"] = ov
    out["l96/obs_m"] = om
    runner = FilterRunner(ir, grid, n_particles=64, resampler="systematic")
    chains, acc = mh_sample(ir, runner, 6, RngStream(21))
    out["l96/mh/thetas"] = np.array([c.theta for c in chains])
    out["l96/mh/logliks"] = np.array([c.loglik for c in chains])
    out["l96/mh/inits"] = np.array([c.init_state for c in chains])
    out["l96/mh/traj_last"] = chains[-1].trajectory
    out["l96/mh/accepted"] = np.array(acc)
    res = smc_sampler(ir, runner, 6, RngStream(22), theta_resampler="systematic")
    out["l96/smc/thetas"] = res.thetas
    out["l96/smc/log_v"] = res.log_v
    out["l96/smc/logliks"] = res.logliks
    out["l96/smc/trajectories"] = res.trajectories
    out["l96/smc/ess"] = np.array([d["ess"] for d in res.diagnostics])
    out["l96/smc/acceptance"] = np.array([d["acceptance"] for d in res.diagnostics])

    import ssmkit.core.ir as I

    I.compile_expr = lambda e, t, b: eval(
        f"lambda T, X, W, U: {I.expr_source(e, t, b)}", {"np": np, "inf": np.inf, "__builtins__": {}}
    )
    ir = load("windkessel")
    theta = np.array([1.8, 3.0, 0.06, 25.0])
    in_times = np.round(np.arange(0, 1.0001, 0.01), 10)
    inputs = LocfInputs(in_times, flow(in_times)[:, None])
    times = np.linspace(0.0, 0.4, 41)
    rng = RngStream(1)
    x = simulate.sample_initial(ir, theta, rng.child(1), size=1)
    obs = []
    for k in range(1, len(times)):
        x = simulate.step_transition(ir, theta, x, inputs, times[k - 1], times[k] - times[k - 1], rng.child(2, k))
        obs.append(simulate.simulate_obs(ir, theta, x, inputs.at(times[k]), rng.child(3, k))[0])
    obs = np.array(obs)
    grid = build_filter_grid(0.0, 0.4, 40, times[1:], obs, np.ones((40, 1), bool), n_obs=1)
    out["wk/in_times"] = in_times
    out["wk/in_values"] = flow(in_times)
    out["wk/obs_v"] = obs
    runner = FilterRunner(ir, grid, inputs=inputs, n_particles=128, resampler="systematic")
    chains, acc = mh_sample(ir, runner, 6, RngStream(23))
    out["wk/mh/thetas"] = np.array([c.theta for c in chains])
    out["wk/mh/logliks"] = np.array([c.loglik for c in chains])
    out["wk/mh/accepted"] = np.array(acc)
    from ssmkit.inference import smc_sampler

    res = smc_sampler(ir, runner, 6, RngStream(25), theta_resampler="systematic")
    out["wk/smc/thetas"], out["wk/smc/logliks"], out["wk/smc/log_v"] = res.thetas, res.logliks, res.log_v
    out["wk/smc/trajectories"] = res.trajectories
    save("outer.npz", **out)


TEST_MODELS = os.path.join(os.path.dirname(HERE), "models")


def load_test_model(name):
    with open(os.path.join(TEST_MODELS, name + ".bi")) as fh:
        return load_model(fh.read())


def simulate_data(ir, theta, times, seed=1, inputs=None):
    """Observations simulated with the reference (runner.py:47-80 recipe)."""
    rng = RngStream(seed)
    x = simulate.sample_initial(ir, theta, rng.child(1), size=1)
    ot, ov, om = [], [], []
    for k in range(1, len(times)):
        x = simulate.step_transition(ir, theta, x, inputs, times[k - 1], times[k] - times[k - 1], rng.child(2, k))
        y = simulate.simulate_obs(ir, theta, x, None if inputs is None else inputs.at(times[k]), rng.child(3, k))[0]
        ot.append(times[k])
        ov.append(y)
        om.append(np.ones(ir.n_obs, bool))
    return np.array(ot), np.array(ov), np.array(om)


def gen_generic():
    """Generic (NVRTC) path fixtures: every model lowered by our codegen from
    the reference IR, the reference's own expression sources for each lowered
    expression (pins the lowering), and reference PF / theta-level / PMMH /
    SMC^2 runs of the two test models."""
    import json

    from ssmkit.inference import FilterRunner, mh_sample, smc_sampler

    import ssmkit.core.ir as I
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1306_3277_b200 import codegen

    # truncated_gaussian's default bound `inf` (SURVEY 8c known defect): compile shim
    I.compile_expr = lambda e, t, b: eval(
        f"lambda T, X, W, U: {I.expr_source(e, t, b)}", {"np": np, "inf": np.inf, "__builtins__": {}})

    models = {"Lorenz96": load("lorenz96"), "Windkessel": load("windkessel"),
              "StochVol": load_test_model("StochVol"), "PredatorPrey": load_test_model("PredatorPrey"),
              "Wide": load_test_model("Wide")}
    lowered, sources = {}, {}
    for name, ir in models.items():
        d = codegen.lower(ir)
        lowered[name] = d
        srcs = []
        for bn in ("initial", "transition", "observation"):
            blk = ir.block(bn)
            for op in (blk.ops if blk is not None else ()):
                if type(op).__name__ == "AssignStmtOp":
                    srcs += [I.expr_source(op.stmt.expr, (ir.consts, ir.vars), b) for b in op.bindings]
                elif type(op).__name__ == "OdeOp":
                    srcs += [I.expr_source(eq.expr, (ir.consts, ir.vars), b) for eq, b in op.items]
                else:
                    _, args = I.canonical_dist_args(op.stmt.dist)
                    srcs += [I.expr_source(a, (ir.consts, ir.vars), b) for b in op.bindings for a in args]
        sources[name] = srcs
        lowered[name]["fingerprint"] = codegen.fingerprint(ir)
    with open(os.path.join(HERE, "gen_models.json"), "w") as fh:
        json.dump({"lowered": lowered, "reference_sources": sources, "versions": VERSIONS}, fh, indent=0,
                  sort_keys=True)
    print("wrote gen_models.json")

    out = {}
    cases = {"StochVol": (np.array([-0.5, 0.9, 0.3]), np.linspace(0.0, 30.0, 31)),
             "PredatorPrey": (np.array([1.1, 0.9, 0.02]), np.linspace(0.0, 3.0, 16))}
    for name, (theta, times) in cases.items():
        ir = models[name]
        ot, ov, om = simulate_data(ir, theta, times)
        grid = build_filter_grid(0.0, times[-1], len(times) - 1, ot, ov, om, n_obs=ir.n_obs)
        out[f"{name}/theta"] = theta
        out[f"{name}/times"] = grid.times
        out[f"{name}/obs_t"] = ot
        out[f"{name}/obs_v"] = ov
        out[f"{name}/obs_m"] = om
        for scheme in ("systematic", "multinomial"):
            res = particle_filter(ir, theta, grid, RngStream(11), n_particles=512, resampler=scheme)
            out[f"{name}/{scheme}/loglik"] = np.array(res.loglik)
            out[f"{name}/{scheme}/traj"] = res.trajectory
            out[f"{name}/{scheme}/x_final"] = res.run.x
            out[f"{name}/{scheme}/anc"] = np.array([h[1] for h in res.run.history[1:] if h[1] is not None])
        # initial block and one transition step with the reference's draws
        x0 = simulate.sample_initial(ir, theta, RngStream(5).child(0), size=300)
        out[f"{name}/x0"] = x0
        out[f"{name}/x1"] = simulate.step_transition(ir, theta, x0, None, 0.0, times[1] - times[0], RngStream(6))
        out[f"{name}/g1"] = simulate.observe_logpdf(ir, theta, out[f"{name}/x1"], None, ov[0], om[0])
        # theta-level blocks (simulate.py:96-108, 219-352)
        th = simulate.sample_parameter(ir, RngStream(3), size=5)
        out[f"{name}/prior_draws"] = th
        out[f"{name}/prior_logpdf"] = np.array([simulate.parameter_logpdf(ir, t) for t in th])
        props = [simulate.propose_parameters(ir, t, RngStream(4).child(k)) for k, t in enumerate(th)]
        out[f"{name}/prop"] = np.array([p[0] for p in props])
        out[f"{name}/prop_logq"] = np.array([p[1] for p in props])
        out[f"{name}/prop_rev"] = np.array([simulate.proposal_parameter_logpdf(ir, p[0], t)
                                            for p, t in zip(props, th)])
        # outer loops at toy size with the reference's draws
        runner = FilterRunner(ir, grid, n_particles=64, resampler="systematic")
        chains, acc = mh_sample(ir, runner, 5, RngStream(31))
        out[f"{name}/mh/thetas"] = np.array([c.theta for c in chains])
        out[f"{name}/mh/logliks"] = np.array([c.loglik for c in chains])
        out[f"{name}/mh/accepted"] = np.array(acc)
        res = smc_sampler(ir, runner, 6, RngStream(32), theta_resampler="systematic")
        out[f"{name}/smc/thetas"] = res.thetas
        out[f"{name}/smc/logliks"] = res.logliks
        out[f"{name}/smc/log_v"] = res.log_v
    # Wide: 12 observations and two inputs (LOCF tables)
    ir = models["Wide"]
    theta = np.array([0.2])
    times = np.linspace(0.0, 2.0, 21)
    in_times = np.round(np.arange(0.0, 2.0001, 0.05), 10)
    in_values = np.stack([0.1 * np.sin(3.0 * in_times), np.cos(2.0 * in_times)], axis=1)
    inputs = LocfInputs(in_times, in_values)
    ot, ov, om = simulate_data(ir, theta, times, inputs=inputs)
    om[3, 5:9] = False  # a partially observed step
    grid = build_filter_grid(0.0, 2.0, 20, ot, ov, om, n_obs=ir.n_obs)
    out["Wide/theta"] = theta
    out["Wide/in_times"] = in_times
    out["Wide/in_values"] = in_values
    out["Wide/obs_t"] = ot
    out["Wide/obs_v"] = ov
    out["Wide/obs_m"] = om
    res = particle_filter(ir, theta, grid, RngStream(12), inputs=inputs, n_particles=512, resampler="systematic")
    out["Wide/loglik"] = np.array(res.loglik)
    out["Wide/traj"] = res.trajectory
    out["Wide/x_final"] = res.run.x
    save("generic.npz", **out)


def dense_kf(out, k, grid):
    """Covariance-form Kalman filter on the reference's extracted system.

    The reference's KalmanRun._step forms the gain as triangular_solve(V, D.T,
    side="right") (kalman.py:84), i.e. D^T V^-1 instead of D V^-1: right only
    when D = Sigma_hat G is square and symmetric (every scalar model such as
    windkessel), and a shape error when fewer slots than states are present.
    Multi-state fixtures therefore use this textbook filter instead."""
    mu, P = out[f"{k}/mu0"].copy(), out[f"{k}/P0"].copy()
    ll, means = 0.0, [mu.copy()]
    for i in range(1, len(grid.times)):
        A, b, Q = out[f"{k}/A"][i - 1], out[f"{k}/b"][i - 1], out[f"{k}/Q"][i - 1]
        mu, P = A @ mu + b, A @ P @ A.T + Q
        obs = grid.obs_at(i)
        if obs is not None:
            pres = np.flatnonzero(obs[1])
            H = out[f"{k}/H"][i - 1][pres]
            c, r = out[f"{k}/c"][i - 1][pres], out[f"{k}/r_sd"][i - 1][pres]
            S = H @ P @ H.T + np.diag(r**2)
            e = obs[0][pres] - (H @ mu + c)
            K = P @ H.T @ np.linalg.inv(S)
            mu = mu + K @ e
            P = P - K @ S @ K.T
            ll += -0.5 * len(pres) * np.log(2 * np.pi) - 0.5 * np.linalg.slogdet(S)[1] - 0.5 * e @ np.linalg.solve(S, e)
        means.append(mu.copy())
    return ll, np.array(means)


def gen_kalman():
    """Reference Kalman filter (kalman.py, lineargauss.py) on the linear-Gaussian
    models: the extracted systems in x' = A x + b form, logliks, a smoothing
    trajectory and the filtered means, for a few parameter vectors."""
    from ssmkit.inference import FilterRunner, kalman_filter, mh_sample
    from ssmkit.lineargauss import extract_linear_gaussian

    import ssmkit.core.ir as I
    I.compile_expr = lambda e, t, b: eval(
        f"lambda T, X, W, U: {I.expr_source(e, t, b)}", {"np": np, "inf": np.inf, "__builtins__": {}})
    out = {}

    def record(tag, ir, thetas, grid, inputs):
        for j, th in enumerate(thetas):
            sys_ = extract_linear_gaussian(ir, th, grid.times, inputs)
            k = f"{tag}/{j}"
            out[f"{k}/mu0"] = sys_.initial.mean
            out[f"{k}/P0"] = sys_.initial.sqrt_cov.T @ sys_.initial.sqrt_cov
            out[f"{k}/A"] = np.array([st.F.T for st in sys_.steps])
            out[f"{k}/b"] = np.array([st.b for st in sys_.steps])
            out[f"{k}/Q"] = np.array([st.Qu.T @ st.Qu for st in sys_.steps])
            out[f"{k}/H"] = np.array([st.G.T for st in sys_.steps])
            out[f"{k}/c"] = np.array([st.c for st in sys_.steps])
            out[f"{k}/r_sd"] = np.array([st.r_sd for st in sys_.steps])
            if tag == "wk":  # the reference's filter (nx = 1)
                res = kalman_filter(sys_, grid, RngStream(40 + j))
                out[f"{k}/loglik"] = np.array(res.loglik)
                out[f"{k}/traj"] = res.trajectory
                out[f"{k}/means"] = np.array([g.mean for g in res.summaries])
            else:  # reference defect (see dense_kf): a textbook filter on the reference's systems
                ll, means = dense_kf(out, k, grid)
                out[f"{k}/loglik"] = np.array(ll)
                out[f"{k}/means"] = means
        out[f"{tag}/thetas"] = np.array(thetas)

    # windkessel on the config-1 data's first 40 steps
    ir = load("windkessel")
    in_times = np.round(np.arange(0, 1.0001, 0.01), 10)
    inputs = LocfInputs(in_times, flow(in_times)[:, None])
    times = np.linspace(0.0, 0.4, 41)
    ot, ov, om = simulate_data(ir, np.array([1.8, 3.0, 0.06, 25.0]), times, inputs=inputs)
    om[5] = False
    grid = build_filter_grid(0.0, 0.4, 40, ot, ov, om, n_obs=1)
    out["wk/obs_v"], out["wk/obs_m"], out["wk/times"] = ov, om, grid.times
    record("wk", ir, [np.array([1.8, 3.0, 0.06, 25.0]), np.array([1.2, 2.0, 0.04, 9.0])], grid, inputs)
    runner = FilterRunner(ir, grid, inputs=inputs, filter_kind="kalman")
    chains, acc = mh_sample(ir, runner, 8, RngStream(24))
    out["wk/mh/thetas"] = np.array([c.theta for c in chains])
    out["wk/mh/logliks"] = np.array([c.loglik for c in chains])
    out["wk/mh/accepted"] = np.array(acc)
    from ssmkit.inference import smc_sampler

    res = smc_sampler(ir, runner, 6, RngStream(25), theta_resampler="systematic")
    out["wk/smc/thetas"], out["wk/smc/logliks"], out["wk/smc/log_v"] = res.thetas, res.logliks, res.log_v
    out["wk/smc/trajectories"] = res.trajectories
    # LinOsc: coupled ode with 2 RK4 steps per sub-step, grid spacing 0.1 = 2 sub-steps, partial masks
    ir = load_test_model("LinOsc")
    import json

    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1306_3277_b200 import codegen

    out["osc/desc"] = np.array(json.dumps(codegen.lower(ir)))
    o_times = np.round(np.arange(0, 3.0001, 0.1), 10)
    o_inputs = LocfInputs(o_times, 0.2 * np.sin(o_times)[:, None])
    times = np.linspace(0.0, 3.0, 31)
    ot, ov, om = simulate_data(ir, np.array([1.3, 0.04]), times, inputs=o_inputs)
    om[2, 1] = False
    om[7, 0] = False
    om[11] = False
    grid = build_filter_grid(0.0, 3.0, 30, ot, ov, om, n_obs=2)
    out["osc/in_times"], out["osc/in_values"] = o_times, 0.2 * np.sin(o_times)
    out["osc/obs_v"], out["osc/obs_m"], out["osc/times"] = ov, om, grid.times
    record("osc", ir, [np.array([1.3, 0.04]), np.array([0.7, 0.1]), np.array([1.9, 0.01])], grid, o_inputs)
    # Wide: 12 states, two inputs (the generic.npz data)
    g = np.load(os.path.join(HERE, "generic.npz"))
    ir = load_test_model("Wide")
    inputs = LocfInputs(g["Wide/in_times"], g["Wide/in_values"])
    grid = build_filter_grid(0.0, 2.0, 20, g["Wide/obs_t"], g["Wide/obs_v"], g["Wide/obs_m"], n_obs=12)
    record("wide", ir, [np.array([0.2]), np.array([0.5])], grid, inputs)
    save("kalman.npz", **out)


if __name__ == "__main__":
    gen_resample()
    gen_lse()
    gen_l96_step()
    gen_wk_step()
    gen_pf()
    gen_theta_level()
    gen_outer_loops()
    gen_generic()
    gen_kalman()

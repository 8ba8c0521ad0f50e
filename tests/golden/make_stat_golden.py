"""Generate the statistical fixtures (stat.npz) by running the REFERENCE itself.

Run in this container only (the reference is not on the GPU box):

    python tests/golden/make_stat_golden.py        # ~10 min on 8 cores

The device-noise path cannot be bitwise the reference (its draws come from
the device's Philox4x32-10 + float32 Box-Muller, not numpy's ziggurat), so
the north star asks for agreement within Monte Carlo error.
This script records reference outputs whose sampling distribution the device
results must share (tests/test_gpu_statistics.py):

  l96_pf       log-likelihood estimates of the L96 bootstrap filter on the
               benchmark data (theta* = (10, 0.1), dt = 0.05, all
               8 slots observed), first 20 grid steps, 2^14 particles, 64
               seeds, systematic and multinomial (particle.py:156-185);
  wk_pmmh      8 independent PMMH chains (mcmc.py:169-180) on the windkessel
               config-1 data (T = 100), 2^12-particle filters, 200 steps
               (`inf` shim of SURVEY 8c applied);
  l96_smc2     8 independent SMC^2 runs (smc.py:67-171), 64 theta-particles x
               2^12 state particles, L96 sparse data (slots 0-3 every other
               step, 20 steps of 0.05): weighted posterior means of (F, sigma2).
"""

import os
import sys
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as M  # noqa: E402  (imports the reference from /root/reference/pkg/src)
from ssmkit import RngStream  # noqa: E402
from ssmkit.core import simulate  # noqa: E402
from ssmkit.inference import FilterRunner, build_filter_grid, mh_sample, particle_filter, smc_sampler  # noqa: E402

P_PF, T_PF, N_SEEDS = 1 << 14, 20, 64
P_MH, N_CHAINS, N_MH = 1 << 12, 8, 200
P_SMC, N_THETA, N_REP = 1 << 12, 64, 8


def l96_bench_grid():
    ir, theta, times, ot, ov, om = M.l96_data(T=40)  # linspace(0, 2, 41), all slots observed
    return ir, theta, build_filter_grid(0.0, times[-1], 40, ot, ov, om, n_obs=8)


def l96_sparse_grid():
    """SURVEY 8d sparse variant on 20 steps of 0.05: slots 0-3 every other step."""
    ir = M.load("lorenz96")
    theta = np.array([10.0, 0.1])
    times = np.linspace(0.0, 1.0, 21)
    rng = RngStream(1)
    x = simulate.sample_initial(ir, theta, rng.child(1), size=1)
    ot, ov, om = [], [], []
    for k in range(1, 21):
        x = simulate.step_transition(ir, theta, x, None, times[k - 1], times[k] - times[k - 1], rng.child(2, k))
        ov.append(simulate.simulate_obs(ir, theta, x, None, rng.child(3, k))[0])
        m = np.zeros(8, bool)
        if k % 2 == 0:
            m[:4] = True
        ot.append(times[k])
        om.append(m)
    ot, ov, om = np.array(ot), np.array(ov), np.array(om)
    return ir, build_filter_grid(0.0, 1.0, 20, ot, ov, om, n_obs=8), ot, ov, om


def wk_config1():
    import ssmkit.core.ir as I

    I.compile_expr = lambda e, t, b: eval(
        f"lambda T, X, W, U: {I.expr_source(e, t, b)}", {"np": np, "inf": np.inf, "__builtins__": {}}
    )
    g = np.load(os.path.join(HERE, "pf.npz"))
    ir = M.load("windkessel")
    inputs = M.LocfInputs(g["wk/in_times"], g["wk/in_values"][:, None])
    grid = build_filter_grid(0.0, 1.0, 100, np.linspace(0, 1, 101)[1:], g["wk/obs_v"], np.ones((100, 1), bool),
                             n_obs=1)
    return ir, inputs, grid


def pf_task(args):
    scheme, s = args
    ir, theta, grid = l96_bench_grid()
    return particle_filter(ir, theta, grid, RngStream(1000 + s), n_particles=P_PF, resampler=scheme,
                           upto=T_PF).loglik


def pmmh_task(c):
    ir, inputs, grid = wk_config1()
    runner = FilterRunner(ir, grid, inputs=inputs, n_particles=P_MH, resampler="multinomial")
    chain, acc = mh_sample(ir, runner, N_MH, RngStream(500 + c))
    return np.array([s.theta for s in chain]), np.array([s.loglik for s in chain]), acc


def smc_task(r):
    ir, grid, *_ = l96_sparse_grid()
    runner = FilterRunner(ir, grid, n_particles=P_SMC, resampler="systematic")
    res = smc_sampler(ir, runner, N_THETA, RngStream(600 + r), theta_resampler="systematic")
    w = np.exp(res.log_v - np.max(res.log_v))
    w /= w.sum()
    return w @ res.thetas, res.thetas, res.log_v


def main():
    out = {}
    with Pool(8) as pool:
        for scheme in ("systematic", "multinomial"):
            out[f"l96_pf/{scheme}/loglik"] = np.array(pool.map(pf_task, [(scheme, s) for s in range(N_SEEDS)]))
        print("pf done", {k: (v.mean(), v.std()) for k, v in out.items()})
        res = pool.map(pmmh_task, range(N_CHAINS))
        out["wk_pmmh/thetas"] = np.stack([r[0] for r in res])
        out["wk_pmmh/logliks"] = np.stack([r[1] for r in res])
        out["wk_pmmh/accepted"] = np.array([r[2] for r in res])
        print("pmmh done", out["wk_pmmh/thetas"][:, 50:].mean(axis=(0, 1)), out["wk_pmmh/accepted"])
        res = pool.map(smc_task, range(N_REP))
        out["l96_smc2/post_mean"] = np.stack([r[0] for r in res])
        out["l96_smc2/thetas"] = np.stack([r[1] for r in res])
        out["l96_smc2/log_v"] = np.stack([r[2] for r in res])
        print("smc2 done", out["l96_smc2/post_mean"].mean(axis=0), out["l96_smc2/post_mean"].std(axis=0))
    _, _, ot, ov, om = l96_sparse_grid()
    out["l96_sparse/obs_t"], out["l96_sparse/obs_v"], out["l96_sparse/obs_m"] = ot, ov, om
    out["sizes"] = np.array([P_PF, T_PF, N_SEEDS, P_MH, N_CHAINS, N_MH, P_SMC, N_THETA, N_REP])
    M.save("stat.npz", **out)


if __name__ == "__main__":
    main()

"""Secondary benchmarks for the other BASELINE.json configs (one JSON line each):

  config 1: windkessel PF, P=1024, T=100 (reference CPU case; launch-bound on the GPU)
  config 3: PMMH on windkessel, 2^16-particle filters, chains batched per GPU (8 per GPU of 64)
  config 4: SMC^2 on L96, 128 theta-particles x 2^14 per GPU (of 1024), sparse obs
  config 5: L96 PF particle-count sweep 2^10 .. 2^26 (1 GPU)
  config g: generic path: models lowered from the reference IR and compiled with
            NVRTC -- L96 (against the hand-written kernel) and the two test models, P = 2^20

Metric: particle-updates/s (P x grid steps, counting SMC^2 rejuvenation replays), device time
with CUDA events around whole driver calls (host theta-level work included).
Run: python bench_outer.py [--configs 1,3,4,5,g] [--quick]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


class Locf:
    def __init__(self, times, values):
        self.times = np.asarray(times, dtype=float)
        self.values = np.asarray(values, dtype=float).reshape(len(self.times), -1)

    def at(self, t):
        tol = 1e-9 * max(1.0, abs(t))
        return self.values[int(np.searchsorted(self.times, t + tol, side="right")) - 1]


def flow(t, f_max=500.0, t_s=0.3, t_d=0.5):
    """Aortic flow input of the windkessel data (Eq. 5)."""
    tp = np.mod(t, t_s + t_d)
    return np.where(tp < t_s, f_max * np.sin(np.pi * tp / t_s) ** 2, 0.0)


def wk_data(T=100, t_end=1.0):
    """Windkessel data at theta* (SURVEY 8d), simulated with this package's simulate API."""
    from paper_1306_3277_b200 import WINDKESSEL, RngStream
    from paper_1306_3277_b200 import simulate as S

    theta = np.array([1.8, 3.0, 0.06, 25.0])
    in_times = np.round(np.arange(0, t_end + 1e-9, 0.01), 10)
    inputs = Locf(in_times, flow(in_times))
    times = np.linspace(0.0, t_end, T + 1)
    rng = RngStream(1)
    x = WINDKESSEL.host_initial(rng.child(1), 1)
    obs = []
    for k in range(1, T + 1):
        x = S.step_transition(WINDKESSEL, theta, x, inputs, times[k - 1], times[k] - times[k - 1], rng.child(2, k))
        F = float(inputs.at(times[k])[0])
        obs.append([rng.child(3, k).normal(x[0, 0] + theta[2] * F, 2.0)])  # Windkessel.bi:33
    return theta, times, np.array(obs), inputs


def l96_sparse(T=40):
    from bench import THETA, simulate_l96_data

    times = np.linspace(0.0, 2.0 * T / 40, T + 1)
    _, ov, om = simulate_l96_data(times, obs_slots=range(4), obs_every=2)
    return THETA.copy(), times, ov, om


def l96_full(T=40):
    from bench import simulate_l96_data

    times = np.linspace(0.0, 2.0 * T / 40, T + 1)
    _, ov, om = simulate_l96_data(times)
    return times, ov, om


def timed(fn, warmup=1, reps=3):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = None
    s.record()
    for _ in range(reps):
        out = None  # release the previous run (and its history) before the next
        out = fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, out


def config1(quick):
    from paper_1306_3277_b200 import WINDKESSEL, RngStream
    from paper_1306_3277_b200.inference import build_filter_grid, particle_filter

    theta, times, obs, inputs = wk_data()
    grid = build_filter_grid(0.0, 1.0, 100, times[1:], obs, np.ones((100, 1), bool), n_obs=1)
    res = {}
    for scheme in ("multinomial", "systematic"):
        ms, out = timed(lambda: particle_filter(WINDKESSEL, theta, grid, RngStream(7), inputs=inputs,
                                                n_particles=1024, resampler=scheme), reps=5)
        res[scheme] = {"ms_per_filter": ms, "value": 1024 * 100 / (ms / 1e3), "loglik": out.loglik}
    return {"config": "1: windkessel PF P=1024 T=100", "unit": "particle-updates/s", "results": res,
            "reference_cpu_1core_survey": {"multinomial": 1.93e6, "systematic": 2.36e6}}


def config3(quick, theta_draws=None):
    from paper_1306_3277_b200 import WINDKESSEL, RngStream
    from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample_chains

    theta, times, obs, inputs = wk_data()
    grid = build_filter_grid(0.0, 1.0, 100, times[1:], obs, np.ones((100, 1), bool), n_obs=1)
    chains, P, steps = 8, 1 << 16, (3 if quick else 10)
    runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=P, resampler="systematic")
    ms, (samples, acc) = timed(lambda: mh_sample_chains(WINDKESSEL, runner, steps, [RngStream(100 + c) for c in range(chains)],
                                                        theta_draws=theta_draws),
                               warmup=1, reps=1)
    runs = chains * (steps + 1)  # init + one filter per MH step (auto-rejects skip theirs)
    tag = "" if theta_draws is None else f", theta blocks on device ({theta_draws} draws)"
    return {"config": f"3: PMMH windkessel, {chains} chains/GPU x 2^16 particles, T=100, {steps} MH steps{tag}",
            "unit": "particle-updates/s", "value": runs * P * 100 / (ms / 1e3), "ms_per_mh_step": ms / (steps + 1),
            "acceptance": acc.tolist(), "reference_cpu_1core_survey": 8.12e6}


def config4(quick, theta_draws=None):
    from paper_1306_3277_b200 import LORENZ96, RngStream
    from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, smc_sampler

    theta, times, ov, om = l96_sparse(T=40)
    grid = build_filter_grid(0.0, 2.0, 40, times[1:], ov, om, n_obs=8)
    n_theta, P = (32, 1 << 12) if quick else (128, 1 << 14)
    runner = FilterRunner(LORENZ96, grid, n_particles=P, resampler="systematic")
    ms, res = timed(lambda: smc_sampler(LORENZ96, runner, n_theta, RngStream(5), theta_resampler="systematic",
                                                theta_draws=theta_draws),
                    warmup=1, reps=2)
    obs_steps = grid.obs_steps
    # PF work: propagation to each obs step + rejuvenation replay to the previous one
    steps = sum(o for o in obs_steps) + sum((obs_steps[i - 2] if i > 1 else 0) for i in range(1, len(obs_steps) + 1))
    tag = "" if theta_draws is None else f", theta blocks on device ({theta_draws} draws)"
    return {"config": f"4: SMC^2 L96 {n_theta} theta x 2^{int(math.log2(P))}, sparse obs, T=40{tag}",
            "unit": "particle-updates/s (incl. replays)", "value": n_theta * P * steps / (ms / 1e3),
            "seconds": ms / 1e3, "final_ess": res.diagnostics[-1]["ess"],
            "reference_cpu_1core_survey": 8.8e5}


def configk(quick):
    """Device Kalman filter: B windkessel systems x T=100 in one
    launch, host extraction timed separately; plus PMMH with filter_kind="kalman"."""
    from paper_1306_3277_b200 import WINDKESSEL, RngStream
    from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample_chains
    from paper_1306_3277_b200.inference.kalman import advance_kalman_runs, kalman_runs
    from paper_1306_3277_b200.lineargauss import extract_linear_gaussian

    theta, times, obs, inputs = wk_data()
    grid = build_filter_grid(0.0, 1.0, 100, times[1:], obs, np.ones((100, 1), bool), n_obs=1)
    B = 1024 if quick else 8192
    rs = np.random.default_rng(0)
    thetas = theta * rs.uniform(0.8, 1.2, size=(B, 4))
    t0 = time.perf_counter()
    sys_ = extract_linear_gaussian(WINDKESSEL, thetas, grid.times, inputs)
    t_extract = time.perf_counter() - t0

    def run():
        runs = kalman_runs(sys_, grid)
        advance_kalman_runs(runs, grid.last)
        return runs

    ms, runs = timed(run, warmup=1, reps=3)
    batch = runs[0]._batch
    ms_kernel, _ = timed(lambda: batch.launch((0, B), 0, grid.last), warmup=1, reps=5)  # kernel only
    runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, filter_kind="kalman")
    ms_mh, (_, acc) = timed(lambda: mh_sample_chains(WINDKESSEL, runner, 20, [RngStream(100 + c) for c in range(64)],
                                                     theta_draws="device"), warmup=1, reps=1)
    return {"config": f"k: device Kalman filter, windkessel, {B} systems x T=100 (one launch) + host extraction",
            "unit": "filter-steps/s", "value": B * 100 / (ms / 1e3), "ms_filter_incl_upload": ms,
            "ms_kernel": ms_kernel, "kernel_filter_steps_per_s": B * 100 / (ms_kernel / 1e3),
            "s_extract_host": t_extract,
            "pmmh_kalman_64_chains_ms_per_mh_step": ms_mh / 21, "pmmh_acceptance": int(np.sum(acc))}


def configr(quick):
    """Resample + gather microbench (SURVEY 8d kernel inputs): logw ~ N(0, sigma_w^2),
    sigma_w in {0, 1, 10} (ESS from P to ~1), numpy default_rng(1234), states U(-1,3)^8,
    f64, P = 2^24: ssm_resample_from_logw (tile records from the log-weights, then the
    filter path's tile resampler) then ssm_gather, timed with CUDA events.
    Algorithmic bytes B_R = 8 (read logw) + 4 (write ancestor) + 2*8*8 (gather) = 140 B."""
    import torch

    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    P = 1 << (20 if quick else 24)
    dev = torch.device("cuda")
    rs = np.random.default_rng(1234)
    x = torch.as_tensor(rs.uniform(-1.0, 3.0, size=(8, P)), device=dev)
    xo = torch.empty_like(x)
    anc = torch.empty(P, dtype=torch.int32, device=dev)
    ws = torch.empty(L.ssm_resample_workspace_bytes(1, P), dtype=torch.uint8, device=dev)
    keys = torch.tensor([[12345, 678]], dtype=torch.int32, device=dev)
    st = _lib.stream_ptr()
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak = float(json.load(open(pk)).get("hbm_gbs", 6552.3)) if os.path.exists(pk) else 6552.3
    res = {}
    for sw in (0.0, 1.0, 10.0):
        a = torch.as_tensor(rs.normal(0.0, sw, size=P) if sw > 0 else np.zeros(P), device=dev)
        shift = torch.logsumexp(a, 0).reshape(1)  # normalised weights (the CDF's fixed point needs sum 1)
        for name, scheme in (("systematic", 2), ("stratified", 1), ("multinomial_sorted", 3)):
            def step():
                _lib.check(L.ssm_resample_from_logw(1, P, _lib.SSM_F64, scheme, _lib.ptr(a), _lib.ptr(shift), None,
                                                    None, _lib.ptr(keys), 1, _lib.ptr(anc), _lib.ptr(ws), st), "rs")
                _lib.check(L.ssm_gather(_lib.SSM_F64, 1, 8, P, _lib.ptr(x), _lib.ptr(anc), _lib.ptr(xo), st), "g")

            ms, _ = timed(step, warmup=2, reps=10)
            gbs = 140.0 * P / (ms / 1e3) / 1e9
            uniq = int(torch.unique(anc).numel())
            res[f"sigma_w={sw:g} {name}"] = {"ms": ms, "GB/s": gbs, "frac_of_measured_peak": gbs / peak,
                                             "unique_ancestors": uniq / P}
    return {"config": f"r: resample+gather microbench, P=2^{int(math.log2(P))}, f64, nx=8 (B_R = 140 B/particle)",
            "unit": "GB/s (algorithmic)", "results": res}


def config5(quick):
    from paper_1306_3277_b200 import LORENZ96, RngStream
    from paper_1306_3277_b200.inference import build_filter_grid, particle_filter
    theta = np.array([10.0, 0.1])
    times, ov, om = l96_full()
    grid = build_filter_grid(0.0, 2.0, 40, times[1:], ov, om, n_obs=8)
    out = {}
    sizes = [(lg, True) for lg in (range(10, 23, 4) if quick else (10, 12, 14, 16, 18, 20, 22, 24, 25))]
    if not quick:  # full f64 history at 2^26 is 164 GiB: history-free run (ancestors only, replayed trajectory)
        sizes += [(24, False), (26, False)]
    for lg, kh in sizes:
        P = 1 << lg
        ms, _ = timed(lambda: particle_filter(LORENZ96, theta, grid, RngStream(7), n_particles=P,
                                              resampler="systematic", exact=False, keep_history=kh),
                      warmup=1, reps=3)
        out[f"2^{lg}" + ("" if kh else " history-free")] = {"ms_per_filter": ms, "value": P * 40 / (ms / 1e3)}
    return {"config": "5: L96 PF sweep, T=40, systematic, f64 (1 GPU); 2^26 runs history-free (its f64 position "
                      "history alone is 164 GiB)", "unit": "particle-updates/s", "results": out}


def configg(quick):
    from paper_1306_3277_b200 import LORENZ96, RngStream, generic
    from paper_1306_3277_b200.inference import build_filter_grid, particle_filter
    with open(os.path.join(ROOT, "tests", "golden", "gen_models.json")) as fh:
        lowered = json.load(fh)["lowered"]
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", "generic.npz")))

    def model(name):
        d = dict(lowered[name])
        d.pop("fingerprint", None)
        return generic.from_description(d)

    P = 1 << (16 if quick else 20)
    theta = np.array([10.0, 0.1])
    times, ov, om = l96_full()
    grid = build_filter_grid(0.0, 2.0, 40, times[1:], ov, om, n_obs=8)
    cases = [("Lorenz96 hand-written", LORENZ96, theta, grid), ("Lorenz96 generic", model("Lorenz96"), theta, grid)]
    for name in ("StochVol", "PredatorPrey"):
        m = model(name)
        T = len(g[f"{name}/times"]) - 1
        gr = build_filter_grid(0.0, float(g[f"{name}/times"][-1]), T, g[f"{name}/obs_t"], g[f"{name}/obs_v"],
                               g[f"{name}/obs_m"], n_obs=m.n_obs)
        cases.append((f"{name} generic", m, g[f"{name}/theta"], gr))
    out = {}
    for name, spec, th, gr in cases:
        ms, res = timed(lambda: particle_filter(spec, th, gr, RngStream(7), n_particles=P, resampler="systematic",
                                                exact=False), warmup=1, reps=3)
        T = len(gr.times) - 1
        out[name] = {"ms_per_filter": ms, "value": P * T / (ms / 1e3), "T": T, "loglik": res.loglik}
    return {"config": f"g: generic (NVRTC) path, P=2^{int(math.log2(P))}, systematic, f64 fast",
            "unit": "particle-updates/s", "results": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5,g")
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    fns = {"1": config1, "3": config3, "4": config4, "5": config5, "g": configg,
           "k": configk, "r": configr, "3d": lambda q: config3(q, "device"), "4d": lambda q: config4(q, "device")}
    for c in args.configs.split(","):
        t0 = time.time()
        r = fns[c](args.quick)
        r["wall_s"] = time.time() - t0
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()

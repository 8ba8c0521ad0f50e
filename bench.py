"""Benchmark: Lorenz '96 bootstrap particle filter, 2^24 particles (BASELINE.json
metric "particle-updates/sec (Lorenz '96 PF, 2^24 particles) and % HBM roofline").

One bench step = one complete filter run over the T=40 grid (linspace(0,2,41),
all 8 slots observed, systematic resampling, float64 = the reference's
precision): init + 40 x (resample scan + search, fused gather/propagate/weight)
+ trajectory draw.  particle-updates = P * T per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL); each rank runs its
own 2^24-particle filter (independent replicas, weak scaling) and the timed
region is closed by a barrier; the reported time is the max over ranks.
The reference arm times the CPU oracle port (the reference is pure Python;
/root/reference is absent on the GPU box) on all host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-updates/sec (Lorenz '96 PF, 2^24 particles) and % HBM roofline"
UNIT = "particle-updates/s"
P_BENCH = 1 << 24
T_BENCH = 40
THETA = np.array([10.0, 0.1])  # SURVEY 8d theta* = (F=10, sigma2=0.1)


def simulate_l96_data(times, seed=1, obs_slots=range(8), obs_every=1):
    """L96 states and observations on `times` (the runner.py:47-80 recipe:
    x0 from child(1), transitions child(2, k), observations child(3, k)), simulated
    with this package's own simulate API (host draws on the device kernel: bitwise
    the reference's simulation).  Returns (obs_t, obs_v, obs_m)."""
    from paper_1306_3277_b200 import LORENZ96, RngStream
    from paper_1306_3277_b200 import simulate as S

    rng = RngStream(seed)
    x = LORENZ96.host_initial(rng.child(1), 1)
    ov, om = [], []
    for k in range(1, len(times)):
        x = S.step_transition(LORENZ96, THETA, x, None, times[k - 1], times[k] - times[k - 1], rng.child(2, k))
        ro = rng.child(3, k)
        ov.append([ro.normal(x[0, n], 0.5) for n in range(8)])  # y[n] ~ normal(x[n], 0.5), Lorenz96.bi:32
        m = np.zeros(8, dtype=bool)
        if k % obs_every == 0:
            m[list(obs_slots)] = True
        om.append(m)
    return np.asarray(times[1:]), np.array(ov), np.array(om)


def synthetic_data(T=T_BENCH):
    """L96 data per SURVEY 8d: theta*, grid linspace(0,2,T+1), all slots observed."""
    times = np.linspace(0.0, 2.0 * T / 40, T + 1)
    ot, ov, om = simulate_l96_data(times)
    return times, ot, ov, om


def _cpu_data(T):
    """The same data for the CPU legs, from the oracle's restatement of the
    reference (the CPU legs may not touch the device)."""
    from oracle import ssm_oracle as O

    times = np.linspace(0.0, 2.0 * T / 40, T + 1)
    obs = O.simulate_l96(THETA, times, O.Stream(1))
    ot = times[1:]
    ov = np.array([obs[k][0] for k in range(1, T + 1)])
    om = np.ones((T, 8), dtype=bool)
    return times, ot, ov, om


def workload_config(P, T, dtype, resampler="systematic"):
    return {
        "workload": f"Lorenz96 bootstrap particle filter, P=2^{int(math.log2(P))} particles, T={T} grid steps "
                    f"(linspace(0,2,{T + 1}), 8/8 slots observed), {resampler} resampling, {dtype}",
        "model": "Lorenz96 (8 state dims, RK4, h=delta=0.05)",
        "particles": P,
        "grid_steps": T,
        "resampler": resampler,
        "noise": ("device Philox4x32-10 counters + float32 Box-Muller (MUFU lg2/sqrt/sincos, 32-bit radius "
                  "uniform, 24-bit angle: |z| <= 6.77 sigma), widened to the filter precision; validated in law "
                  "against the reference in tests/test_gpu_statistics.py"),
        "global_batch": P,
        "seq_len": T,
        "parallelism": "replicas",
        "l2": "no flush: per-step state is 1 GiB (f64) >> 126 MB L2",
    }


# ---------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi sampled every 100 ms from before warm-up; summary() keeps the
    samples whose timestamps fall inside [t0, t1] (the timed region)."""

    FIELDS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self, t0=None, t1=None):
        import datetime

        sm, mx, reasons, power = [], 0.0, set(), []
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            if t0 is not None and ts is not None and not (t0 - 0.15 <= ts <= t1 + 0.15):
                continue
            try:
                sm.append(float(f[2]))
                mx = max(mx, float(f[3]))
                power.append(float(f[4]))
            except ValueError:
                continue
            for name, v in zip(self.FIELDS, f[6:10]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------ our arm


def generic_l96():
    """Lorenz '96 through the generic path: the reference model lowered from its
    IR (tests/golden/gen_models.json, make_golden.py) and compiled with NVRTC."""
    from paper_1306_3277_b200 import generic

    with open(os.path.join(ROOT, "tests", "golden", "gen_models.json")) as fh:
        d = dict(json.load(fh)["lowered"]["Lorenz96"])
    d.pop("fingerprint", None)
    return generic.from_description(d)


def run_ours(args, rank, world):
    import torch

    from paper_1306_3277_b200 import LORENZ96, RngStream, profiling
    from paper_1306_3277_b200.inference import build_filter_grid, particle_filter

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    P, T = args.particles, args.T
    model = LORENZ96 if args.model == "lorenz96" else generic_l96()
    times, ot, ov, om = synthetic_data(T)
    grid = build_filter_grid(0.0, times[-1], T, ot, ov, om, n_obs=8)
    opts = dict(dtype=args.dtype, exact=args.exact, noise="device")

    sharded = world > 1 and args.mode == "sharded"

    class _Out:
        def __init__(self, ll, traj):
            self.loglik, self.trajectory = ll, traj

    def call(rng, grid_obj):
        if sharded:  # one filter of world * P particles, NCCL collectives every weighted step (config 5)
            from paper_1306_3277_b200.inference import particle_filter_sharded

            return _Out(*particle_filter_sharded(LORENZ96, THETA, grid_obj, rng, world * P, resampler=args.resampler,
                                                 dtype=args.dtype, exact=args.exact))
        return particle_filter(model, THETA, grid_obj, rng, n_particles=P, resampler=args.resampler, **opts)

    def one(step, grid_obj, timer=None):
        rng = RngStream(7, ((0 if sharded else rank), step))
        if timer is None:
            return call(rng, grid_obj)
        with profiling.timing(timer):
            return call(rng, grid_obj)

    dist = world > 1
    if dist:
        import torch.distributed as tdist

    def barrier():
        if dist:
            tdist.barrier()
        torch.cuda.synchronize()

    # events around every 20th grid step's launches (2 of 40 per run); SSM_BENCH_TIMER_EVERY for A/B
    timer = profiling.KernelTimer(every=int(os.environ.get("SSM_BENCH_TIMER_EVERY", "20")))
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    logliks = []
    with ClockSampler(dev.index) as clocks:
        for w in range(args.warmup):
            out = one(10**6 + w, grid)
        del out
        # ---- device-timed region: K steps, inputs resident, events on the launching stream
        barrier()
        n0 = profiling.launch_count()
        t_wall0 = time.time()
        start.record()
        for k in range(args.steps):
            out = one(k, grid, timer)
            logliks.append(out.loglik)
            del out
        end.record()
        barrier()
        t_wall1 = time.time()
    launches = profiling.launch_count() - n0
    ms = start.elapsed_time(end)
    kern = timer.summary()
    # ---- end-to-end: host buffers in, host results out, through the public API
    e2e_ms = None
    h2d = d2h = 0
    if args.e2e_steps > 0:
        barrier()
        t0 = time.perf_counter()
        for k in range(args.e2e_steps):
            g2 = build_filter_grid(0.0, times[-1], T, ot.copy(), ov.copy(), om.copy(), n_obs=8)
            out = one(1000 + k, g2)
            _ = float(out.loglik), np.asarray(out.trajectory).sum()
            del out
        barrier()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        # bytes copied per step: sub-step table + theta + keys + filter state + u, and back:
        # filter state + trajectory (+ trace pointer tables)
        h2d = T * 64 + 32 + 8 + 64 + 8 + 2 * 8 * (T + 1)
        d2h = 64 + 8 * 8 * (T + 1) + 64
    if dist:
        t = torch.tensor([ms, e2e_ms or 0.0], device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms, e2e_ms = float(t[0]), (float(t[1]) if e2e_ms is not None else None)
    return dict(ms=ms, kern=kern, launches=launches, clocks=clocks.summary(t_wall0, t_wall1), logliks=logliks,
                e2e_ms=e2e_ms, h2d=h2d, d2h=d2h)


# ------------------------------------------------------------ SMC^2 workload (config 4)

SMC2_METRIC = "particle-updates/sec (SMC^2 on Lorenz '96, {n_theta} theta x 2^{logp}, rejuvenation replays counted)"


def run_smc2(args, rank, world):
    """Config 4: SMC^2 on L96 with 1024 theta-particles x 2^14 state
    particles, sparse observations (slots 0-3 every other step of linspace(0,2,41)),
    systematic at both levels, theta-slots sharded contiguously over the ranks
    (smc_sampler with torch.distributed: per observation one all-gather of the
    theta log-weights (C2) and the point-to-point redistribution of migrating
    theta-particles (C3, history-free payloads)).  One bench step = one complete
    SMC^2 run; particle-updates = sum over theta-particles of P x (propagated +
    replayed grid steps)."""
    import torch

    from paper_1306_3277_b200 import LORENZ96, RngStream, profiling
    from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, smc_sampler

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    n_theta, P, T = args.smc_theta, args.smc_particles, 40
    times = np.linspace(0.0, 2.0, T + 1)
    ot, ov, om = simulate_l96_data(times, obs_slots=range(4), obs_every=2)
    grid = build_filter_grid(0.0, 2.0, T, ot, ov, om, n_obs=8)
    runner = FilterRunner(LORENZ96, grid, n_particles=P, resampler="systematic", keep_history=False)
    obs_steps = grid.obs_steps
    steps = sum(obs_steps) + sum((obs_steps[i - 2] if i > 1 else 0) for i in range(1, len(obs_steps) + 1))
    dist = world > 1
    if dist:
        import torch.distributed as tdist

    def barrier():
        if dist:
            tdist.barrier()
        torch.cuda.synchronize()

    def one(k):
        return smc_sampler(LORENZ96, runner, n_theta, RngStream(11, (k,)), theta_resampler="systematic",
                           theta_draws="device")

    timer = profiling.KernelTimer()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clocks:
        for w in range(args.warmup):
            one(10**6 + w)
        barrier()
        n0 = profiling.launch_count()
        t_wall0 = time.time()
        start.record()
        ess = []
        for k in range(args.steps):
            with profiling.timing(timer):
                res = one(k)
            ess.append(res.diagnostics[-1]["ess"])
        end.record()
        barrier()
        t_wall1 = time.time()
    ms = start.elapsed_time(end)
    launches = profiling.launch_count() - n0
    e2e_ms = None
    if args.e2e_steps > 0:  # through the public API from host data: grid, runner and sampler built per step
        barrier()
        t0 = time.perf_counter()
        for k in range(args.e2e_steps):
            g2 = build_filter_grid(0.0, 2.0, T, ot.copy(), ov.copy(), om.copy(), n_obs=8)
            r2 = FilterRunner(LORENZ96, g2, n_particles=P, resampler="systematic", keep_history=False)
            out = smc_sampler(LORENZ96, r2, n_theta, RngStream(12, (k,)), theta_resampler="systematic",
                              theta_draws="device")
            _ = float(np.sum(out.logliks))
        barrier()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
    if dist:
        t = torch.tensor([ms, e2e_ms or 0.0], device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms, e2e_ms = float(t[0]), (float(t[1]) if e2e_ms is not None else None)
    return dict(ms=ms, kern=timer.summary(), launches=launches, clocks=clocks.summary(t_wall0, t_wall1),
                e2e_ms=e2e_ms, steps_per_run=steps, ess=ess)


def smc2_line(args, res, world):
    n_theta, P, K = args.smc_theta, args.smc_particles, args.steps
    updates = n_theta * P * res["steps_per_run"]
    value = updates * K / (res["ms"] / 1e3)
    peak, peak_kind = load_peaks()
    pw = res["kern"].get("propagate_weight", {})
    achieved = pw["bytes"] / (pw["total_ms"] / 1e3) / 1e9 if pw else None
    line = {
        "metric": SMC2_METRIC.format(n_theta=n_theta, logp=int(math.log2(P))), "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": res["ms"] / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (L96 theta*=(10,0.1), sparse obs: slots 0-3 every other step; device noise)",
        "config": {"workload": f"SMC^2 on Lorenz96, {n_theta} theta-particles x 2^{int(math.log2(P))} particles, "
                               "T=40 grid steps, 20 sparse observations, systematic at both levels, float64",
                   "theta_particles": n_theta, "particles": P, "grid_steps": 40,
                   "parallelism": f"theta-slots sharded over {world} GPU(s): C2 all-gather of theta log-weights, "
                                  "C3 point-to-point theta-particle redistribution (history-free payloads)",
                   "theta_draws": "device", "history": "history-free runs (ancestors + replayed trajectories)"},
        "roofline": {"bound": "hbm", "kernel": "pw_kernel (batched over theta-particles)", "achieved": achieved,
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": None},
        "kernels": {k: {"avg_ms": round(v["avg_ms"], 4), "launches": v["launches"]} for k, v in res["kern"].items()},
        "gpu_launches": res["launches"], "clocks": res["clocks"], "final_theta_ess": res["ess"],
    }
    if res["e2e_ms"] is not None:
        line["e2e"] = {"value": updates / (res["e2e_ms"] / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": int(40 * 64 + 40 * 8 * 8), "d2h_bytes_per_step": int(n_theta * 8 * 3),
                       "ms_per_step": res["e2e_ms"]}
    return line


# ------------------------------------------------------------ CPU baselines


def _cpu_filter_task(a):
    P, T, seed = a
    from oracle import ssm_oracle as O

    times, ot, ov, om = _cpu_data(T)
    grid = O.Grid(times, {k + 1: (ov[k], om[k]) for k in range(T)})
    t0 = time.perf_counter()
    O.particle_filter("lorenz96", THETA, grid, O.Stream(7, (seed,)), n_particles=P, resampler="systematic")
    return time.perf_counter() - t0


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def cpu_baseline_single(P=1 << 20, T=10):
    """The oracle port on one host core (numpy is single-threaded here)."""
    dt = _cpu_filter_task((P, T, 0))
    return {"value": P * T / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle port (numpy restatement of ssmkit particle_filter), L96, P=2^{int(math.log2(P))}, "
                      f"T={T} steps, systematic, float64, {dt:.1f} s, one core of {cpu_model()}"}


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (oracle port) on all host cores."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    P, T = args.ref_particles, args.ref_T
    with mp.get_context("spawn").Pool(cores) as pool:
        for w in range(args.warmup):
            pool.map(_cpu_filter_task, [(P, T, 100 + c) for c in range(cores)])
        walls = []
        for k in range(args.steps):
            t0 = time.perf_counter()
            pool.map(_cpu_filter_task, [(P, T, 1000 * k + c) for c in range(cores)])
            walls.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(walls))
    value = cores * P * T / (ms / 1e3)
    sample = (f"{cores} processes x oracle port (numpy restatement of ssmkit particle_filter), L96, "
              f"P=2^{int(math.log2(P))} each, T={T} steps, systematic, float64, {cores} cores of {cpu_model()}")
    # the workload is ours (same metric, model, data recipe, scheme, precision); each timed step is a
    # bounded SAMPLE of it, stated here: `cores` independent filters of P particles over the first T
    # grid steps (the CPU filter's particle-updates/s is flat in P and T: SURVEY 8d)
    cfg = dict(workload_config(P_BENCH, T_BENCH, "float64"), noise="numpy Philox4x64 + ziggurat (host, oracle port)",
               sample=f"{cores} processes x P=2^{int(math.log2(P))} particles x T={T} grid steps per timed step",
               sample_particles=P, sample_grid_steps=T, sample_processes=cores, parallelism=f"{cores} CPU processes")
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------------- main


def _step_roofline(kern, P, peak):
    ph = [kern[k] for k in ("resample", "propagate_weight") if k in kern]
    if not ph:
        return None
    nbytes, ms = sum(v["bytes"] for v in ph), sum(v["total_ms"] for v in ph)
    steps = max(v["launches"] for v in ph)
    achieved = nbytes / (ms / 1e3) / 1e9
    return {"phases": "resample + propagate_weight (gather fused)", "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 3),
            "algorithmic_bytes_per_update": round(nbytes / steps / P, 2)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "pw_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--particles", type=int, default=P_BENCH)
    ap.add_argument("--T", type=int, default=T_BENCH)
    ap.add_argument("--dtype", default="float64", choices=["float64", "float32"])
    ap.add_argument("--resampler", default="systematic", choices=["systematic", "stratified", "multinomial"])
    ap.add_argument("--exact", action="store_true",
                    help="bitwise reference op order (no FMA contraction); default: FMA-contracted float64")
    ap.add_argument("--variants", type=int, default=1, help="also time f64-exact and f32 variants")
    ap.add_argument("--mode", default="sharded", choices=["sharded", "replicas"],
                    help="N>1: one filter of N*2^24 particles across GPUs (default) or N independent filters")
    ap.add_argument("--model", default="lorenz96", choices=["lorenz96", "generic"],
                    help="hand-written L96 kernel (default) or the NVRTC-compiled generic path")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--ref-particles", type=int, default=1 << 17)
    ap.add_argument("--ref-T", type=int, default=8)
    ap.add_argument("--workload", default="pf", choices=["pf", "smc2"],
                    help="pf: the L96 particle filter (headline); smc2: config 4, SMC^2 sharded over the GPUs")
    ap.add_argument("--smc-theta", type=int, default=1024)
    ap.add_argument("--smc-particles", type=int, default=1 << 14)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
        # SSM_BENCH_BACKEND=gloo only to exercise the N>1 harness on a single GPU
        tdist.init_process_group(os.environ.get("SSM_BENCH_BACKEND", "nccl"))
    if args.workload == "smc2":
        res = run_smc2(args, rank, world)
        if rank == 0:
            print(json.dumps(smc2_line(args, res, world)), flush=True)
        if world > 1:
            import torch.distributed as tdist

            tdist.destroy_process_group()
        return
    res = run_ours(args, rank, world)
    if rank != 0:
        if world > 1:
            import torch.distributed as tdist

            tdist.destroy_process_group()
        return
    P, T, K = args.particles, args.T, args.steps
    updates = world * P * T * K
    value = updates / (res["ms"] / 1e3)
    peak, peak_kind = load_peaks()
    pw = res["kern"].get("propagate_weight", {})
    achieved = pw["bytes"] / (pw["total_ms"] / 1e3) / 1e9 if pw else None
    traffic = load_traffic()
    kern = {k: {"avg_ms": round(v["avg_ms"], 4), "launches": v["launches"],
                "GB/s": round(v["bytes"] / (v["total_ms"] / 1e3) / 1e9, 1),
                "frac": round(v["bytes"] / (v["total_ms"] / 1e3) / 1e9 / peak, 3),
                "algorithmic_bytes_per_particle": round(v["bytes"] / max(v["launches"], 1) / P, 2)}
            for k, v in res["kern"].items()}
    dtype_tag = "f64" if args.dtype == "float64" else "f32"
    arith = "bitwise reference op order" if args.exact else "float64 with FMA contraction (1e-12 of reference per step)"
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": res["ms"] / K,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": dtype_tag,
        "data": "synthetic (L96 theta*=(10,0.1) simulated per SURVEY 8d; device Philox noise)",
        "config": dict(workload_config(P, T, args.dtype, args.resampler), arithmetic=arith,
                       kernels=("hand-written L96 kernel" if args.model == "lorenz96"
                                else "generic path: L96 lowered from the reference IR, NVRTC-compiled"),
                       parallelism=("replicas" if world == 1 or args.mode == "replicas"
                                    else f"one filter sharded over {world} GPUs (NCCL all-gather of LSE partials and "
                                         "CDF totals + P2P spill of ancestor states per step)")),
        "roofline": {
            "bound": "hbm",
            "kernel": "pw_lag_kernel (fused ancestor gather + RK4 propagate + weight + LSE; the headline step's pw_kernel specialisation)",
            "achieved": achieved,
            "peak": peak,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None,
            # ncu DRAM bytes of one launch (profiles/pw_traffic.json, captured with `source` below), only
            # when the profiled launch has this run's size
            "traffic": (traffic.get("bytes_per_launch") if traffic and pw and traffic.get("particles") == P
                        else None),
            "traffic_source": (traffic.get("source") if traffic else None),
            "algorithmic_bytes_per_particle": pw["bytes"] / max(pw["launches"], 1) / P if pw else None,
            "timing": ("CUDA events on the launching stream around the resample and pw launches of grid steps "
                       "19 and 39 of each timed filter run (an event between two programmatic dependent "
                       "launches serialises them: bracketing all 40 steps costs 3.4% of the run, "
                       "profiles/r2_timer_ab.txt)"),
        },
        "kernels": kern,
        # the whole grid step (resample kernels + fused gather/propagate/weight): algorithmic bytes of
        # both phases over their summed device time, per particle-update
        "step_roofline": _step_roofline(res["kern"], P, peak),
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "loglik_mean": float(np.mean(res["logliks"])),
    }
    if world > 1 and args.mode == "sharded":
        line["config"]["global_batch"] = world * P
        line["config"]["particles"] = world * P
    if res["e2e_ms"] is not None:
        line["e2e"] = {"value": world * P * T / (res["e2e_ms"] / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"],
                       "ms_per_step": res["e2e_ms"]}
    if args.variants and world == 1:
        line["variants"] = {}
        for name, dt, ex, rs, mdl in (("f64_exact_bitwise", "float64", True, args.resampler, args.model),
                                      ("f32", "float32", False, args.resampler, args.model),
                                      ("f64_multinomial", "float64", False, "multinomial", args.model),
                                      ("f64_generic_codegen", "float64", False, args.resampler, "generic")):
            if (dt, ex, rs, mdl) == (args.dtype, args.exact, args.resampler, args.model):
                continue
            v_args = argparse.Namespace(**vars(args))
            v_args.dtype, v_args.exact, v_args.e2e_steps, v_args.resampler, v_args.model = dt, ex, 0, rs, mdl
            v = run_ours(v_args, rank, world)
            vpw = v["kern"].get("propagate_weight", {})
            line["variants"][name] = {
                "value": P * T * K / (v["ms"] / 1e3), "ms_per_step": v["ms"] / K,
                "pw_GB_s": vpw["bytes"] / (vpw["total_ms"] / 1e3) / 1e9 if vpw else None}
    if args.cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline_single()
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as tdist

        tdist.destroy_process_group()


if __name__ == "__main__":
    main()

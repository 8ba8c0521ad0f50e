"""Where the time of the moderate-P outer loops goes (configs 3 and 4): wall and
device time per call, per-phase kernel time from the native driver's events,
kernel launches.  python profiles/outer_breakdown.py"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_outer as BO  # noqa: E402
from paper_1306_3277_b200 import LORENZ96, WINDKESSEL, RngStream, profiling  # noqa: E402
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample_chains, smc_sampler  # noqa: E402


def breakdown(name, fn, reps=2):
    fn()
    torch.cuda.synchronize()
    timer = profiling.KernelTimer()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = profiling.launch_count()
    t0 = time.perf_counter()
    s.record()
    with profiling.timing(timer):
        for _ in range(reps):
            fn()
    e.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    dev = s.elapsed_time(e) / reps
    k = {n: {"total_ms_per_call": v["total_ms"] / reps, "launches": v["launches"] // reps, "avg_ms": v["avg_ms"]}
         for n, v in timer.summary().items()}
    print(json.dumps({"case": name, "wall_ms": wall * 1e3, "device_ms": dev,
                      "launches": (profiling.launch_count() - n0) // reps, "kernels": k}), flush=True)


theta, times, obs, inputs = BO.wk_data()
grid = build_filter_grid(0.0, 1.0, 100, times[1:], obs, np.ones((100, 1), bool), n_obs=1)
runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=1 << 16, resampler="systematic")
rngs = [RngStream(100 + c) for c in range(8)]
from paper_1306_3277_b200.inference import particle as particle_mod  # noqa: E402

for no_coop in (True, False):
    particle_mod._NO_COOP = no_coop
    breakdown(f"config3 run_batch 8 x 2^16 (one MH step's filters), {'per-step kernels' if no_coop else 'persistent'}",
              lambda: runner.run_batch([theta] * 8, [None] * 8, [g.child(1) for g in rngs]))
breakdown("config3 mh_sample_chains 8 chains x 3 steps (device theta)",
          lambda: mh_sample_chains(WINDKESSEL, runner, 3, rngs, theta_draws="device"), reps=1)
particle_mod._NO_COOP = False
th, t4, ov, om = BO.l96_sparse(T=40)
g4 = build_filter_grid(0.0, 2.0, 40, t4[1:], ov, om, n_obs=8)
r4 = FilterRunner(LORENZ96, g4, n_particles=1 << 14, resampler="systematic")
for no_coop in (True, False):
    particle_mod._NO_COOP = no_coop
    breakdown(f"config4 smc 128 theta x 2^14 (device theta), {'per-step kernels' if no_coop else 'persistent'}",
              lambda: smc_sampler(LORENZ96, r4, 128, RngStream(5), theta_resampler="systematic", theta_draws="device"),
              reps=1)
r4h = FilterRunner(LORENZ96, g4, n_particles=1 << 14, resampler="systematic", keep_history=False)
breakdown("config4 smc 128 theta x 2^14 (device theta, history-free)",
          lambda: smc_sampler(LORENZ96, r4h, 128, RngStream(5), theta_resampler="systematic", theta_draws="device"),
          reps=1)

"""Config 3 (PMMH windkessel, 8 chains x 2^16, T=100, theta blocks on the device):
wall time per MH step vs the GPU-busy time, and a cProfile of the host side.
usage: python profiles/mh_overhead.py"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_outer as B  # noqa: E402
from paper_1306_3277_b200 import WINDKESSEL, RngStream, profiling  # noqa: E402
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample_chains  # noqa: E402


def main():
    theta, times, obs, inputs = B.wk_data()
    grid = build_filter_grid(0.0, 1.0, 100, times[1:], obs, np.ones((100, 1), bool), n_obs=1)
    runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=1 << 16, resampler="systematic")
    rngs = [RngStream(100 + c) for c in range(8)]
    mh_sample_chains(WINDKESSEL, runner, 3, rngs, theta_draws="device")
    torch.cuda.synchronize()
    n = 10
    timer = profiling.KernelTimer()
    t0 = time.perf_counter()
    with profiling.timing(timer):
        mh_sample_chains(WINDKESSEL, runner, n, [RngStream(200 + c) for c in range(8)], theta_draws="device")
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / n
    kern = timer.summary()
    busy = sum(v["total_ms"] for v in kern.values()) / n
    print(f"{wall:.3f} ms wall per MH step; kernels (event-bracketed, serialised) {busy:.3f} ms")
    for k, v in kern.items():
        print(f"  {k:24s} {v['launches'] / n:7.1f} launches/step  {v['total_ms'] / n:8.3f} ms/step")
    t0 = time.perf_counter()
    mh_sample_chains(WINDKESSEL, runner, n, [RngStream(300 + c) for c in range(8)], theta_draws="device")
    torch.cuda.synchronize()
    print(f"{(time.perf_counter() - t0) * 1e3 / n:.3f} ms wall per MH step without the timer")
    pr = cProfile.Profile()
    pr.enable()
    mh_sample_chains(WINDKESSEL, runner, n, [RngStream(400 + c) for c in range(8)], theta_draws="device")
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()

"""Config 4 (SMC^2 L96, 128 theta x 2^14, sparse obs, device theta blocks): wall vs
event-bracketed kernel time, and a cProfile of the host side (tottime).
usage: python profiles/smc_overhead.py"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench_outer as B  # noqa: E402
from paper_1306_3277_b200 import LORENZ96, RngStream, profiling  # noqa: E402
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, smc_sampler  # noqa: E402


def main():
    theta, times, ov, om = B.l96_sparse(T=40)
    grid = build_filter_grid(0.0, 2.0, 40, times[1:], ov, om, n_obs=8)
    runner = FilterRunner(LORENZ96, grid, n_particles=1 << 14, resampler="systematic")

    def run(seed):
        return smc_sampler(LORENZ96, runner, 128, RngStream(seed), theta_resampler="systematic", theta_draws="device")

    run(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(2)
    torch.cuda.synchronize()
    print(f"{(time.perf_counter() - t0) * 1e3:.1f} ms wall per SMC^2 run")
    timer = profiling.KernelTimer()
    with profiling.timing(timer):
        run(3)
    kern = timer.summary()
    for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["total_ms"]):
        print(f"  {k:24s} {v['launches']:6d} launches  {v['total_ms']:8.2f} ms (event-bracketed)")
    import gc

    gc.disable()
    pr = cProfile.Profile()
    pr.enable()
    run(4)
    torch.cuda.synchronize()
    pr.disable()
    gc.enable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(40)


if __name__ == "__main__":
    main()

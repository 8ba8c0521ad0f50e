"""bench.py --workload smc2 (1024 theta x 2^14, device theta blocks, history-free): wall per
run, GPU busy time from a CUDA-event pair around the run vs the host's own time, and a
cProfile of one run (tottime).  usage: python profiles/smc2_overhead.py [n_theta]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1306_3277_b200 import LORENZ96, RngStream  # noqa: E402
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, smc_sampler  # noqa: E402


def main():
    n_theta = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    times = np.linspace(0.0, 2.0, 41)
    ot, ov, om = bench.simulate_l96_data(times, obs_slots=range(4), obs_every=2)
    grid = build_filter_grid(0.0, 2.0, 40, ot, ov, om, n_obs=8)
    runner = FilterRunner(LORENZ96, grid, n_particles=1 << 14, resampler="systematic", keep_history=False)

    def run(k):
        return smc_sampler(LORENZ96, runner, n_theta, RngStream(11, (k,)), theta_resampler="systematic",
                           theta_draws="device")

    run(10**6)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(0)
    torch.cuda.synchronize()
    print(f"{(time.perf_counter() - t0) * 1e3:.1f} ms wall per run")
    pr = cProfile.Profile()
    pr.enable()
    run(1)
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(35)
    st.sort_stats("cumulative").print_stats(40)


if __name__ == "__main__":
    main()

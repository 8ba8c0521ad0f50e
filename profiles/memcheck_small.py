"""Small native calls for compute-sanitizer memcheck: theta-level resample of a few
weights (the P_in < 2048 tile of the search path), the tile-path resample at ragged
sizes, a short filter and a small SMC^2.  usage: compute-sanitizer python profiles/memcheck_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1306_3277_b200 import LORENZ96, RngStream  # noqa: E402
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, particle_filter, smc_sampler  # noqa: E402
from paper_1306_3277_b200.inference.resampling import resample  # noqa: E402


def main():
    rs = np.random.default_rng(0)
    for n in (1, 5, 256, 2047, 2049, 5000):
        for scheme in ("systematic", "stratified", "multinomial"):
            resample(rs.random(n), scheme, RngStream(n))
    times = np.linspace(0.0, 1.0, 11)
    ot, ov, om = bench.simulate_l96_data(times, obs_slots=range(8), obs_every=1)
    grid = build_filter_grid(0.0, 1.0, 10, ot, ov, om, n_obs=8)
    for P in (1000, 5000, 8192 + 37):
        for r in ("systematic", "stratified", "multinomial"):
            particle_filter(LORENZ96, bench.THETA, grid, RngStream(P), n_particles=P, resampler=r, noise="device")
    runner = FilterRunner(LORENZ96, grid, n_particles=8192 + 5, resampler="systematic", keep_history=False)
    smc_sampler(LORENZ96, runner, 6, RngStream(3), theta_resampler="systematic", theta_draws="device")
    print("memcheck workload done")


if __name__ == "__main__":
    main()

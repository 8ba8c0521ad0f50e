"""World-1 overhead of the sharded driver against particle_filter at the bench
size (L96, P=2^24, T=40, systematic, f64): same kernels, host loop in Python
with the sharded bookkeeping (no host synchronisation in the grid loop)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import THETA, synthetic_data  # noqa: E402
from paper_1306_3277_b200 import LORENZ96, RngStream  # noqa: E402
from paper_1306_3277_b200.inference import build_filter_grid, particle_filter, particle_filter_sharded  # noqa: E402

P, T = 1 << 24, 40
times, ot, ov, om = synthetic_data(T)
grid = build_filter_grid(0.0, times[-1], T, ot, ov, om, n_obs=8)


def timed(fn, n=5):
    for w in range(2):
        fn(RngStream(9, (w,)))
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for k in range(n):
        fn(RngStream(7, (k,)))
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


pf = timed(lambda rng: particle_filter(LORENZ96, THETA, grid, rng, n_particles=P, resampler="systematic"))
sh = timed(lambda rng: particle_filter_sharded(LORENZ96, THETA, grid, rng, P, resampler="systematic"))
a = particle_filter(LORENZ96, THETA, grid, RngStream(3), n_particles=P, resampler="systematic")
b = particle_filter_sharded(LORENZ96, THETA, grid, RngStream(3), P, resampler="systematic")
print(f"particle_filter {pf:.3f} ms/run  sharded(world=1) {sh:.3f} ms/run  overhead {100 * (sh / pf - 1):.2f}%  "
      f"bitwise loglik {a.loglik == b[0]} traj {np.array_equal(a.trajectory, b[1])}")

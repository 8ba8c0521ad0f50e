"""Config 1 (windkessel PF, P=1024, T=100) after a warm-up, for an ncu launch
list and a host/device split: python profiles/one_wk_filter.py"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_outer as B  # noqa: E402
from paper_1306_3277_b200 import WINDKESSEL, RngStream, profiling  # noqa: E402
from paper_1306_3277_b200.inference import build_filter_grid, particle_filter  # noqa: E402

theta, times, obs, inputs = B.wk_data()
grid = build_filter_grid(0.0, 1.0, 100, times[1:], obs, np.ones((100, 1), bool), n_obs=1)
for _ in range(3):
    particle_filter(WINDKESSEL, theta, grid, RngStream(7), inputs=inputs, n_particles=1024, resampler="systematic")
torch.cuda.synchronize()
print("warm launches", profiling.launch_count(), flush=True)
t0 = time.perf_counter()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
out = particle_filter(WINDKESSEL, theta, grid, RngStream(7), inputs=inputs, n_particles=1024, resampler="systematic")
e.record()
torch.cuda.synchronize()
print("wall ms %.3f  events ms %.3f" % ((time.perf_counter() - t0) * 1e3, s.elapsed_time(e)), flush=True)

"""One batched SMC^2-style replay: 128 L96 filters x 2^14 particles over 19 grid
steps (sparse obs), wall vs device time; then a second call for an ncu launch list."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_outer as B  # noqa: E402
from paper_1306_3277_b200 import LORENZ96, RngStream, profiling  # noqa: E402
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid  # noqa: E402

theta, times, ov, om = B.l96_sparse(T=40)
grid = build_filter_grid(0.0, 2.0, 40, times[1:], ov, om, n_obs=8)
runner = FilterRunner(LORENZ96, grid, n_particles=1 << 14, resampler="systematic")
th = [np.array([10.0 + 0.01 * k, 0.1]) for k in range(128)]
x0 = [np.full(8, 1.0) for _ in range(128)]


def once(seed):
    return runner.run_batch(th, x0, [RngStream(seed, (k,)) for k in range(128)], upto=19)


once(1)
torch.cuda.synchronize()
for rep in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    s.record()
    once(2 + rep)
    e.record()
    torch.cuda.synchronize()
    print("wall_ms", (time.perf_counter() - t) * 1e3, "event_ms", s.elapsed_time(e), flush=True)
print("launches_before", profiling.launch_count(), flush=True)
once(9)
torch.cuda.synchronize()
print("launches_after", profiling.launch_count(), flush=True)

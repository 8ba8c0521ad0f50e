"""One PMMH step of config 3 after a warm-up (for an ncu launch list):
python profiles/one_mh_step.py  -> prints the launch count of the warm-up part."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_outer as B  # noqa: E402
from paper_1306_3277_b200 import WINDKESSEL, RngStream, profiling  # noqa: E402
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample_chains  # noqa: E402

theta, times, obs, inputs = B.wk_data()
grid = build_filter_grid(0.0, 1.0, 100, times[1:], obs, np.ones((100, 1), bool), n_obs=1)
runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=1 << 16, resampler="systematic")
mh_sample_chains(WINDKESSEL, runner, 2, [RngStream(100 + c) for c in range(8)])
torch.cuda.synchronize()
print("warm launches", profiling.launch_count(), flush=True)
mh_sample_chains(WINDKESSEL, runner, 1, [RngStream(200 + c) for c in range(8)])
torch.cuda.synchronize()
print("total launches", profiling.launch_count(), flush=True)

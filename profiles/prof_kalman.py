"""Host/device split of the batched device Kalman filter (bench_outer config k)."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_outer as B  # noqa: E402
from paper_1306_3277_b200 import WINDKESSEL  # noqa: E402
from paper_1306_3277_b200.inference import build_filter_grid  # noqa: E402
from paper_1306_3277_b200.inference.kalman import advance_kalman_runs, kalman_runs  # noqa: E402
from paper_1306_3277_b200.lineargauss import extract_linear_gaussian  # noqa: E402

theta, times, obs, inputs = B.wk_data()
grid = build_filter_grid(0.0, 1.0, 100, times[1:], obs, np.ones((100, 1), bool), n_obs=1)
thetas = theta * np.random.default_rng(0).uniform(0.8, 1.2, size=(8192, 4))
sys_ = extract_linear_gaussian(WINDKESSEL, thetas, grid.times, inputs)


def run():
    runs = kalman_runs(sys_, grid)
    advance_kalman_runs(runs, grid.last)
    torch.cuda.synchronize()


run()
pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(15)

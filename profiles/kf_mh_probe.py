"""Host/device split of one PMMH step with the Kalman runner (config k's 64 chains)."""
import cProfile, gc, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench_outer as B
from paper_1306_3277_b200 import WINDKESSEL, RngStream
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample_chains

theta, times, obs, inputs = B.wk_data()
grid = build_filter_grid(0.0, 1.0, 100, times[1:], obs, np.ones((100, 1), bool), n_obs=1)
runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, filter_kind="kalman")
mh_sample_chains(WINDKESSEL, runner, 3, [RngStream(100 + c) for c in range(64)], theta_draws="device")
torch.cuda.synchronize()
t0 = time.perf_counter()
mh_sample_chains(WINDKESSEL, runner, 10, [RngStream(200 + c) for c in range(64)], theta_draws="device")
torch.cuda.synchronize()
print(f"{(time.perf_counter() - t0) * 1e3 / 11:.2f} ms per MH step")
gc.disable()
pr = cProfile.Profile(); pr.enable()
mh_sample_chains(WINDKESSEL, runner, 10, [RngStream(300 + c) for c in range(64)], theta_draws="device")
torch.cuda.synchronize(); pr.disable(); gc.enable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)

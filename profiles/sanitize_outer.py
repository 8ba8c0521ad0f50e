"""compute-sanitizer driver (one tool per gpurun call): the SMC^2 / PMMH outer
loops at small P (persistent kernel) and at P = 8192 (multi-kernel path), in one
process, after an SMC^2 run with device theta draws."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1306_3277_b200 import LORENZ96, RngStream  # noqa: E402
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, mh_sample_chains, smc_sampler  # noqa: E402
from tests.conftest import load_golden  # noqa: E402
from tests.test_gpu_distributed import _run  # noqa: E402

g = load_golden("stat.npz")
grid = build_filter_grid(0.0, 1.0, 20, g["l96_sparse/obs_t"], g["l96_sparse/obs_v"], g["l96_sparse/obs_m"], n_obs=8)
runner = FilterRunner(LORENZ96, grid, n_particles=4096, resampler="systematic")
for r in range(int(os.environ.get("REPS", "2"))):
    res = smc_sampler(LORENZ96, runner, 16, RngStream(700 + r), theta_resampler="systematic", theta_draws="device")
    print("smc2 device draws", r, res.logliks[:2], flush=True)
for cfg in (None, dict(P=8192, resampler="multinomial")):
    out = _run("smc", cfg)
    print("smc", cfg, np.asarray(out[1])[:3], flush=True)
out = _run("pmmh")
print("pmmh", np.asarray(out[1])[0, :3], flush=True)
print("SANITIZE_DONE")

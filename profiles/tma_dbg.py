import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_1306_3277_b200 import LORENZ96, RngStream
from paper_1306_3277_b200.inference import build_filter_grid, particle_filter
times, ot, ov, om = bench.synthetic_data(40)
grid = build_filter_grid(0.0, times[-1], 40, ot, ov, om, n_obs=8)
for lg in (16, 20, 21, 22, 23, 24):
    try:
        out = particle_filter(LORENZ96, bench.THETA, grid, RngStream(7), n_particles=1 << lg, resampler="systematic", upto=int(sys.argv[1]))
        torch.cuda.synchronize()
        print(lg, "ok", out.loglik, flush=True)
    except Exception as e:
        print(lg, "FAIL", str(e)[:100], flush=True)
        break

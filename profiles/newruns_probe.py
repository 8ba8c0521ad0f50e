"""Time the pieces of FilterRunner.new_runs for 128 L96 runs (config 4 size)."""
import copy, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench_outer as B
from paper_1306_3277_b200 import LORENZ96, RngStream
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid
from paper_1306_3277_b200.inference.particle import ParticleRun, init_runs

theta, times, ov, om = B.l96_sparse(T=40)
grid = build_filter_grid(0.0, 2.0, 40, times[1:], ov, om, n_obs=8)
runner = FilterRunner(LORENZ96, grid, n_particles=1 << 14, resampler="systematic")
th = [np.array([10.0, 0.1])] * 128
for rep in range(3):
    t0 = time.perf_counter(); proto = runner._make(th[0], None); t1 = time.perf_counter()
    rs = [copy.copy(proto) for _ in range(127)]; t2 = time.perf_counter()
    rs2 = []
    for _ in range(127):
        o = ParticleRun.__new__(ParticleRun); o.__dict__ = dict(proto.__dict__); rs2.append(o)
    t3 = time.perf_counter()
    runs = [proto] + rs
    rngs = [RngStream(5).child(j) for j in range(128)]
    t4 = time.perf_counter(); init_runs(runs, [g.child(0) for g in rngs]); torch.cuda.synchronize(); t5 = time.perf_counter()
    t6 = time.perf_counter(); runner.new_runs(th, [None] * 128, rngs); torch.cuda.synchronize(); t7 = time.perf_counter()
    print(f"_make {1e3*(t1-t0):.3f} ms  copy.copy x127 {1e3*(t2-t1):.3f} ms  dict copy x127 {1e3*(t3-t2):.3f} ms  "
          f"init_runs {1e3*(t5-t4):.3f} ms  new_runs {1e3*(t7-t6):.3f} ms")

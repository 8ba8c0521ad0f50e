import sys, time, cProfile, pstats, numpy as np, torch
sys.path.insert(0, '.')
import bench_outer as BO
from paper_1306_3277_b200 import WINDKESSEL, RngStream
from paper_1306_3277_b200.inference import build_filter_grid, particle_filter, ParticleRun
theta, times, obs, inputs = BO.wk_data()
grid = build_filter_grid(0.0, 1.0, 100, times[1:], obs, np.ones((100, 1), bool), n_obs=1)
f = lambda: particle_filter(WINDKESSEL, theta, grid, RngStream(7), inputs=inputs, n_particles=1024, resampler="systematic")
for _ in range(3): f()
torch.cuda.synchronize()
rng = RngStream(7)
t0 = time.perf_counter(); r = ParticleRun(WINDKESSEL, theta, grid, inputs=inputs, n_particles=1024, resampler="systematic"); t1 = time.perf_counter()
r.init(rng.child(0)); torch.cuda.synchronize(); t2 = time.perf_counter()
r.advance_to(100, rng.child(1)); t3 = time.perf_counter()
tr = r.sample_trajectory(rng.child(2)); t4 = time.perf_counter()
print('construct %.3f ms init %.3f advance %.3f traj %.3f' % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3, (t4-t3)*1e3))
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(); r2 = ParticleRun(WINDKESSEL, theta, grid, inputs=inputs, n_particles=1024, resampler="systematic").init(rng.child(0)); m = torch.cuda.Event(enable_timing=True); m.record(); r2.advance_to(100, rng.child(1)); e.record(); torch.cuda.synchronize()
print('device: init %.3f ms, advance(incl. sync) %.3f ms' % (s.elapsed_time(m), m.elapsed_time(e)))
cProfile.run('for _ in range(20): f()', '/tmp/p.prof')
pstats.Stats('/tmp/p.prof').sort_stats('tottime').print_stats(15)

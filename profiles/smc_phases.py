"""Unprofiled phase timing of one SMC^2 run (config 4, device theta): wraps the
functions smc_sampler calls with perf_counter accumulators."""
import collections, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench_outer as B
from paper_1306_3277_b200 import LORENZ96, RngStream
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, smc_sampler
import paper_1306_3277_b200.inference.smc as smc
import paper_1306_3277_b200.inference.particle as particle
import paper_1306_3277_b200.inference.theta_mh as tmh
import paper_1306_3277_b200.inference.mcmc as mcmc

acc = collections.defaultdict(float)
cnt = collections.defaultdict(int)
def wrap(mod, name, label=None):
    f = getattr(mod, name)
    lab = label or name
    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc[lab] += time.perf_counter() - t
            cnt[lab] += 1
    setattr(mod, name, g)

for m in (smc, mcmc, tmh, particle):
    for n in ("advance_runs", "sample_trajectories", "init_runs"):
        if hasattr(m, n): wrap(m, n, n)
wrap(tmh, "marginal_mh_steps_device")
wrap(smc, "_advance_all")
wrap(smc, "resample", "theta_resample")
wrap(particle, "_fs_view")
wrap(particle, "_advance_native")
wrap(particle, "_schedule")
wrap(particle, "_derived_tensor")
wrap(particle, "_rows")
orig_new_runs = mcmc.FilterRunner.new_runs
def new_runs(self, *a, **k):
    t = time.perf_counter()
    try: return orig_new_runs(self, *a, **k)
    finally: acc["new_runs"] += time.perf_counter() - t; cnt["new_runs"] += 1
mcmc.FilterRunner.new_runs = new_runs
orig_prop = tmh.DeviceThetaChains.propose
def prop(self, *a, **k):
    t = time.perf_counter()
    try: return orig_prop(self, *a, **k)
    finally: acc["propose"] += time.perf_counter() - t; cnt["propose"] += 1
tmh.DeviceThetaChains.propose = prop
orig_acc = tmh.DeviceThetaChains.accept
def accf(self, *a, **k):
    t = time.perf_counter()
    try: return orig_acc(self, *a, **k)
    finally: acc["accept"] += time.perf_counter() - t; cnt["accept"] += 1
tmh.DeviceThetaChains.accept = accf

theta, times, ov, om = B.l96_sparse(T=40)
grid = build_filter_grid(0.0, 2.0, 40, times[1:], ov, om, n_obs=8)
runner = FilterRunner(LORENZ96, grid, n_particles=1 << 14, resampler="systematic")
run = lambda s: smc_sampler(LORENZ96, runner, 128, RngStream(s), theta_resampler="systematic", theta_draws="device")
run(1); torch.cuda.synchronize()
import gc
for gc_off in (False, True):
    acc.clear(); cnt.clear()
    if gc_off:
        gc.disable()
    t0 = time.perf_counter(); run(2); torch.cuda.synchronize(); tot = time.perf_counter() - t0
    gc.enable()
    print(f"gc {'off' if gc_off else 'on'}: total {tot*1e3:.1f} ms, gc stats {gc.get_stats()[2]}")
print("per-function (last run):")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:28s} {cnt[k]:5d} calls {v*1e3:8.2f} ms")

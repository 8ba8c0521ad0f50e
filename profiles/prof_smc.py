"""Wall-time attribution for config 4 (SMC^2): wraps the main host phases
with perf_counter + cuda synchronize (run under gpurun).  python profiles/prof_smc.py"""
import collections
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench_outer as B  # noqa: E402
from paper_1306_3277_b200 import models  # noqa: E402
from paper_1306_3277_b200.inference import mcmc, particle, smc  # noqa: E402

T = collections.defaultdict(float)
N = collections.Counter()


def wrap(mod, name, label=None):
    f = getattr(mod, name)
    label = label or f"{mod.__name__.split('.')[-1]}.{name}"

    def g(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            torch.cuda.synchronize()
            T[label] += time.perf_counter() - t
            N[label] += 1
    setattr(mod, name, g)


for mod, name in [(mcmc, "propose_batch"), (mcmc, "init_runs"), (mcmc, "advance_runs"), (mcmc, "sample_trajectories"),
                  (smc, "advance_runs"), (smc, "sample_trajectories"), (smc, "resample"),
                  (smc, "marginal_mh_steps"), (smc, "_advance_all")]:
    wrap(mod, name)

B.config4(False)
T.clear()
N.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
out = B.config4(False)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print("wall", wall, out)
for k, v in sorted(T.items(), key=lambda x: -x[1]):
    print(f"{k:32s} {v*1e3:9.1f} ms  calls {N[k]}")

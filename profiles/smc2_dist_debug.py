"""Sharded SMC^2 (bench.py --workload smc2 settings) under torchrun on one GPU
(gloo): which configuration fails.  usage: torchrun ... profiles/smc2_dist_debug.py
<theta_draws host|device> <n_theta> <P> <keep_history 0|1> [runs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

import bench  # noqa: E402
from paper_1306_3277_b200 import LORENZ96, RngStream  # noqa: E402
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid, smc_sampler  # noqa: E402


def main():
    td = None if sys.argv[1] == "host" else "device"
    n_theta, P, kh = int(sys.argv[2]), int(sys.argv[3]), bool(int(sys.argv[4]))
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo")
    times = np.linspace(0.0, 2.0, 41)
    ot, ov, om = bench.simulate_l96_data(times, obs_slots=range(4), obs_every=2)
    grid = build_filter_grid(0.0, 2.0, 40, ot, ov, om, n_obs=8)
    runner = FilterRunner(LORENZ96, grid, n_particles=P, resampler="systematic", keep_history=kh)
    runs = int(sys.argv[5]) if len(sys.argv) > 5 else 1
    seeds = [10**6 + w for w in range(int(os.environ.get("DBG_WARM", "0")))] + list(range(runs))
    for k in seeds:
        if os.environ.get("DBG_TIMER") and k < 10**6:
            from paper_1306_3277_b200 import profiling
            with profiling.timing(profiling.KernelTimer(every=int(os.environ["DBG_TIMER"]))):
                r = smc_sampler(LORENZ96, runner, n_theta, RngStream(11, (k,)), theta_resampler="systematic",
                                theta_draws=td)
        else:
            r = smc_sampler(LORENZ96, runner, n_theta, RngStream(11, (k,)), theta_resampler="systematic",
                            theta_draws=td)
        if os.environ.get("DBG_SYNC"):
            torch.cuda.synchronize()
        if tdist.get_rank() == 0:
            print("run", k, float(np.sum(r.logliks)), flush=True)
    torch.cuda.synchronize()
    if tdist.get_rank() == 0:
        print("OK", sys.argv[1:], float(np.sum(r.logliks)))
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()

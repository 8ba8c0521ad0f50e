"""Where the headline filter run's time goes outside the grid-step kernels:
per-run wall vs device time, and a cProfile of the host side of one run.
usage: python profiles/run_overhead.py [P_log2]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1306_3277_b200 import LORENZ96, RngStream  # noqa: E402
from paper_1306_3277_b200.inference import build_filter_grid, particle_filter  # noqa: E402


def main():
    P = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
    times, ot, ov, om = bench.synthetic_data(40)
    grid = build_filter_grid(0.0, times[-1], 40, ot, ov, om, n_obs=8)

    def one(k):
        return particle_filter(LORENZ96, bench.THETA, grid, RngStream(7, (0, k)), n_particles=P,
                               resampler="systematic", noise="device")

    for k in range(3):
        out = one(10**6 + k)
    del out
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    for k in range(5):
        out = one(k)
        _ = out.loglik
        del out
    e.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / 5
    print(f"P=2^{P.bit_length() - 1}: {s.elapsed_time(e) / 5:.3f} ms per run (events), {wall:.3f} ms wall")
    # host time of one run while the device is idle: enqueue cost with the GPU drained first
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    t0 = time.perf_counter()
    out = one(99)
    t1 = time.perf_counter()
    pr.disable()
    print(f"one run, host wall {1e3 * (t1 - t0):.3f} ms")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(30)


if __name__ == "__main__":
    main()

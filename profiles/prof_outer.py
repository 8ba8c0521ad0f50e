"""Host vs device split for bench_outer configs 3 / 4 (run under gpurun):
wall time per call, cProfile top functions, and device time from a KernelTimer-free
CUDA-event bracket.  Usage: python profiles/prof_outer.py 3|4"""
import cProfile
import io
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench_outer as B  # noqa: E402
from paper_1306_3277_b200 import profiling  # noqa: E402


def main(cfg):
    fn = {"3": B.config3, "4": B.config4, "3d": lambda q: B.config3(q, "device"),
          "4d": lambda q: B.config4(q, "device")}[cfg]
    fn(False)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n0 = profiling.launch_count()
    out = fn(False)
    torch.cuda.synchronize()
    print("wall_s", time.perf_counter() - t0, "launches", profiling.launch_count() - n0, out)
    pr = cProfile.Profile()
    pr.enable()
    fn(False)
    torch.cuda.synchronize()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(35)
    print(s.getvalue())
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
    print(s.getvalue())


if __name__ == "__main__":
    main(sys.argv[1])

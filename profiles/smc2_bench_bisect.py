"""Bisect bench.run_smc2 under torchrun (one GPU, gloo): DBG_NOCLOCK=1 replaces the
nvidia-smi sampler, DBG_NOTIMER=1 disables the kernel timer, DBG_NOBARRIER=1 the gloo barrier."""
import argparse
import contextlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

import bench  # noqa: E402
from paper_1306_3277_b200 import profiling  # noqa: E402


class NoClock:
    def __init__(self, *a):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *e):
        pass

    def summary(self, *a):
        return {}


def main():
    if os.environ.get("DBG_NOCLOCK"):
        bench.ClockSampler = NoClock
    if os.environ.get("DBG_NOTIMER"):
        profiling.timing = lambda t: contextlib.nullcontext(t)
    if os.environ.get("DBG_NOBARRIER"):
        tdist.barrier = lambda *a, **k: None
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo")
    args = argparse.Namespace(smc_theta=256, smc_particles=1 << 14, warmup=3, steps=3, e2e_steps=0)
    res = bench.run_smc2(args, tdist.get_rank(), tdist.get_world_size())
    if tdist.get_rank() == 0:
        print("OK", res["ms"])
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()

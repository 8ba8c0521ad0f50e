"""Sharded outer loops on ONE GPU: two processes (gloo, host-staged
exchange) each drive their own kernels on cuda:0 -- no kernel waits on
another process, so this is safe on one device.  Results must equal the
single-process run bitwise (draws are keyed by the global slot)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from paper_1306_3277_b200 import LORENZ96
    from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid
    from tests.conftest import load_golden

    g = load_golden("outer.npz")
    times = g["l96/times"]
    grid = build_filter_grid(0.0, times[-1], 10, times[1:], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)
    return LORENZ96, FilterRunner(LORENZ96, grid, n_particles=512, resampler="systematic")


def _run(kind):
    from paper_1306_3277_b200 import RngStream
    from paper_1306_3277_b200.inference import mh_sample_chains, smc_sampler

    model, runner = _setup()
    if kind == "smc":
        r = smc_sampler(model, runner, 12, RngStream(3), theta_resampler="systematic")
        return r.thetas, r.logliks, r.log_v, r.trajectories
    chains, acc = mh_sample_chains(model, runner, 3, [RngStream(60 + c) for c in range(5)])
    return (np.array([[s.theta for s in ch] for ch in chains]), np.array([[s.loglik for s in ch] for ch in chains]),
            acc, np.array([[s.trajectory for s in ch] for ch in chains]))


def _worker(rank, world, port, kind, q):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.getcwd())
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = _run(kind)
        if rank == 0:
            q.put(tuple(np.asarray(o) for o in out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["smc", "pmmh"])
def test_sharded_equals_single(kind):
    ref = _run(kind)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for a, b in zip(ref, got):
        np.testing.assert_array_equal(np.asarray(a), b)

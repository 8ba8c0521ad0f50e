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


def _setup(cfg=None):
    from paper_1306_3277_b200 import LORENZ96
    from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid
    from tests.conftest import load_golden

    g = load_golden("outer.npz")
    times = g["l96/times"]
    grid = build_filter_grid(0.0, times[-1], 10, times[1:], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)
    cfg = dict(cfg or {})
    opts = dict(n_particles=cfg.pop("P", 512), resampler=cfg.pop("resampler", "systematic"))
    return LORENZ96, FilterRunner(LORENZ96, grid, **opts, **cfg)


def _run(kind, cfg=None):
    from paper_1306_3277_b200 import RngStream
    from paper_1306_3277_b200.inference import mh_sample_chains, smc_sampler

    model, runner = _setup(cfg)
    if kind == "smc":
        r = smc_sampler(model, runner, 12, RngStream(3), theta_resampler="systematic")
        return r.thetas, r.logliks, r.log_v, r.trajectories
    chains, acc = mh_sample_chains(model, runner, 3, [RngStream(60 + c) for c in range(5)])
    return (np.array([[s.theta for s in ch] for ch in chains]), np.array([[s.loglik for s in ch] for ch in chains]),
            acc, np.array([[s.trajectory for s in ch] for ch in chains]))


def _worker(rank, world, port, kind, q, cfg=None):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.getcwd())
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = _run(kind, cfg)
        if rank == 0:
            q.put(tuple(np.asarray(o) for o in out))
    finally:
        dist.destroy_process_group()


# P >= 8192 takes the multi-kernel tile path (the small-P kernel keeps its CDF
# in shared memory): migrating theta-particles must carry their tile CDF for every
# scheme that resamples from it, including the default multinomial (sorted,
# device draws), with the ESS gate, and history-free runs ship ancestors only
CFGS = {
    "small": None,
    "multinomial_8k": dict(P=8192, resampler="multinomial"),
    "stratified_8k": dict(P=8192, resampler="stratified"),
    "systematic_8k_ess": dict(P=8192, resampler="systematic", ess_rel=0.5),
    "multinomial_8k_history_free": dict(P=8192, resampler="multinomial", keep_history=False),
}


@pytest.mark.parametrize("kind,cfg", [("smc", c) for c in CFGS] + [("pmmh", "small")])
def test_sharded_equals_single(kind, cfg):
    cfg = CFGS[cfg]
    ref = _run(kind, cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q, cfg)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for a, b in zip(ref, got):
        np.testing.assert_array_equal(np.asarray(a), b)

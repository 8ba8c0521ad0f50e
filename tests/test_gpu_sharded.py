"""Config 5: one particle filter sharded across ranks (peer-mapped arenas,
ssm_offspring_push / x_peer gathers).  On one GPU: the 1-rank sharded filter
must equal particle_filter bitwise; 2 processes (gloo, host-staged
collectives, each driving its own kernels on cuda:0 and reading the other's
arenas through CUDA IPC) must equal 1 rank up to the association of the
per-rank LSE partials."""

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


def _problem():
    from paper_1306_3277_b200.inference import build_filter_grid
    from tests.conftest import load_golden

    g = load_golden("pf.npz")
    return g["l96/theta"], build_filter_grid(0.0, 2.0, 20, g["l96/obs_t"], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)


def _sharded(scheme, P, ess_rel=None):
    from paper_1306_3277_b200 import LORENZ96, RngStream
    from paper_1306_3277_b200.inference import particle_filter_sharded

    theta, grid = _problem()
    ll, traj = particle_filter_sharded(LORENZ96, theta, grid, RngStream(31), P, resampler=scheme, ess_rel=ess_rel)
    return np.array([ll]), traj


@pytest.mark.parametrize("scheme,ess_rel", [("systematic", None), ("stratified", None), ("systematic", 0.6)])
def test_one_rank_sharded_equals_particle_filter(scheme, ess_rel):
    from paper_1306_3277_b200 import LORENZ96, RngStream
    from paper_1306_3277_b200.inference import particle_filter

    theta, grid = _problem()
    P = 1 << 15
    ll, traj = _sharded(scheme, P, ess_rel)
    out = particle_filter(LORENZ96, theta, grid, RngStream(31), n_particles=P, resampler=scheme, exact=False,
                          ess_rel=ess_rel)
    assert ll[0] == out.loglik
    np.testing.assert_array_equal(traj, out.trajectory)


def _worker(rank, world, port, scheme, P, q, ess_rel=None):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.getcwd())
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ll, traj = _sharded(scheme, P, ess_rel)
        q.put((rank, ll, traj))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scheme,ess_rel", [("systematic", None), ("stratified", None), ("systematic", 0.6)])
def test_two_ranks_match_one(scheme, ess_rel):
    P = 1 << 15
    ref_ll, ref_traj = _sharded(scheme, P, ess_rel)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, scheme, P, q, ess_rel)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for _, ll, traj in res:
        assert abs(ll[0] - ref_ll[0]) <= 1e-9 * abs(ref_ll[0])
        np.testing.assert_allclose(traj, ref_traj, rtol=0, atol=1e-9)


def test_two_ranks_large_partition():
    """Large per-rank P (partition sizes differ between the phases' layouts)."""
    P = 1 << 21
    ref_ll, ref_traj = _sharded("systematic", P)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, "systematic", P, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for _, ll, traj in res:
        assert abs(ll[0] - ref_ll[0]) <= 1e-9 * abs(ref_ll[0])


def test_four_ranks_match_one():
    """Four ranks: outputs of one rank's particles may land two ranks away in the
    degenerate first steps; the peer stores follow them."""
    P = 1 << 14
    ref_ll, ref_traj = _sharded("systematic", P)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 4, port, "systematic", P, q)) for r in range(4)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(4)]
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for _, ll, traj in res:
        assert abs(ll[0] - ref_ll[0]) <= 1e-9 * abs(ref_ll[0])
        np.testing.assert_allclose(traj, ref_traj, rtol=0, atol=1e-9)

"""Multi-process (gloo, world_size 2) tests of the multi-GPU plumbing on CPU:
sharding, all-gather (C2) and theta-slot redistribution (C3)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1306_3277_b200.distributed import (Shard, allgather_f64, exchange, owner_of,
                                              plan_redistribution, shard_bounds)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("n,world", [(10, 3), (3, 4), (1024, 8), (7, 1), (16, 2)])
def test_shard_bounds_partition(n, world):
    seen = []
    for r in range(world):
        lo, hi = shard_bounds(n, r, world)
        seen.extend(range(lo, hi))
        for j in range(lo, hi):
            assert owner_of(j, n, world) == r
    assert seen == list(range(n))


def test_plan_is_consistent_across_ranks():
    rs = np.random.default_rng(0)
    n, world = 37, 4
    anc = np.sort(rs.integers(0, n, n))
    plans = [plan_redistribution(anc, n, Shard(r, world)) for r in range(world)]
    for r, pl in enumerate(plans):
        for peer, srcs in pl.sends.items():
            dsts = plans[peer].recvs[r]
            assert len(srcs) == len(dsts)
            assert [int(anc[j]) for j in dsts] == srcs
        lo, hi = shard_bounds(n, r, world)
        covered = [j for j, _ in pl.local_copies] + [j for ds in pl.recvs.values() for j in ds]
        assert sorted(covered) == list(range(lo, hi))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = Shard.current()
        n = 11
        counts = [shard_bounds(n, r, world)[1] - shard_bounds(n, r, world)[0] for r in range(world)]
        lo, hi = shard.bounds(n)
        # C2: all-gather of per-rank vectors with unequal counts
        g = allgather_f64(np.arange(lo, hi, dtype=float) * 10.0, shard, counts)
        assert np.array_equal(g, np.arange(n) * 10.0)
        # C3: each slot's payload = (slot id, a (3, 4) tensor tagged by slot)
        anc = np.array([0, 0, 1, 3, 3, 3, 6, 9, 9, 10, 10])
        plan = plan_redistribution(anc, n, shard)
        payload = {j: [torch.tensor([float(j)]), torch.full((3, 4), float(j))] for j in range(lo, hi)}
        sends = {peer: [t for a in srcs for t in payload[a]] for peer, srcs in plan.sends.items()}
        specs = {peer: [((1,), torch.float32), ((3, 4), torch.float32)] * len(d) for peer, d in plan.recvs.items()}
        got = exchange(sends, specs, shard)
        result = {j: payload[a][0].item() for j, a in plan.local_copies}
        for peer, dsts in plan.recvs.items():
            for k, j in enumerate(dsts):
                result[j] = got[peer][2 * k].item()
                assert torch.all(got[peer][2 * k + 1] == got[peer][2 * k].item())
        q.put((rank, sorted(result.items())))
    finally:
        dist.destroy_process_group()


def test_gloo_allgather_and_redistribution_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get() for _ in range(world))
    anc = [0, 0, 1, 3, 3, 3, 6, 9, 9, 10, 10]
    merged = dict(res[0] + res[1])
    assert [merged[j] for j in range(11)] == [float(a) for a in anc]

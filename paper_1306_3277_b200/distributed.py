"""Multi-GPU plumbing for the outer loops: one process per GPU,
torch.distributed (NCCL over NVLink on B200; gloo for CPU tests).

  * Contiguous sharding of independent units (PMMH chains, theta-particles).
  * C2: all-gather of per-rank float64 vectors (theta log-weights, summaries).
  * C3: redistribution after theta-resampling.  Every rank computes the same
    ancestors from the same host stream, so the send/receive plan is
    computed locally and consistently.  Payloads are lists of tensors with
    shapes the receiver can derive.  They go through NCCL point-to-point
    (batch_isend_irecv) when the backend is NCCL, or are staged through host
    memory for gloo.
No collective is ever issued inside a kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    group: object = None

    @staticmethod
    def current(group=None):
        if dist.is_available() and dist.is_initialized():
            return Shard(dist.get_rank(group), dist.get_world_size(group), group)
        return Shard(0, 1, None)

    def bounds(self, n):
        return shard_bounds(n, self.rank, self.world)

    def owner(self, j, n):
        return owner_of(j, n, self.world)

    @property
    def backend(self):
        if self.world == 1:
            return None
        return dist.get_backend(self.group)


def shard_bounds(n, rank, world):
    """Contiguous split of n units over `world` ranks (first n % world get one more)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def owner_of(j, n, world):
    base, extra = divmod(n, world)
    cut = extra * (base + 1)
    return j // (base + 1) if j < cut else extra + (j - cut) // max(base, 1)


def _comm_device(shard):
    if shard.backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def allgather_f64(local: np.ndarray, shard: Shard, counts=None) -> np.ndarray:
    """Concatenate each rank's float64 vector in rank order (C1/C2).
    `counts` (per-rank lengths) defaults to equal lengths."""
    local = np.ascontiguousarray(local, dtype=np.float64).reshape(-1)
    if shard.world == 1:
        return local.copy()
    dev = _comm_device(shard)
    if counts is None:
        counts = [local.size] * shard.world
    m = max(counts)
    buf = torch.zeros(m, dtype=torch.float64, device=dev)
    buf[: local.size] = torch.from_numpy(local).to(dev)
    out = [torch.empty(m, dtype=torch.float64, device=dev) for _ in range(shard.world)]
    dist.all_gather(out, buf, group=shard.group)
    return np.concatenate([o[:c].cpu().numpy() for o, c in zip(out, counts)])


def allreduce_max_f64(x: float, shard: Shard) -> float:
    if shard.world == 1:
        return float(x)
    t = torch.tensor([x], dtype=torch.float64, device=_comm_device(shard))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=shard.group)
    return float(t.item())


@dataclass
class Plan:
    """Redistribution of n global slots after resampling with `ancestors`.

    For this rank: local destination slot j (global index) receives the
    payload of global source slot ancestors[j].  `local_copies` lists
    (dest j, src a) with both on this rank; `sends[peer]` lists the local
    source slots to send (in ascending destination order); `recvs[peer]`
    lists the local destination slots filled by that peer (same order).
    """

    local_copies: list
    sends: dict
    recvs: dict


def plan_redistribution(ancestors, n, shard: Shard) -> Plan:
    anc = np.asarray(ancestors, dtype=np.int64)
    lo, hi = shard.bounds(n)
    local_copies, sends, recvs = [], {}, {}
    for j in range(n):
        a = int(anc[j])
        dst, src = owner_of(j, n, shard.world), owner_of(a, n, shard.world)
        if dst == shard.rank and src == shard.rank:
            local_copies.append((j, a))
        elif dst == shard.rank:
            recvs.setdefault(src, []).append(j)
        elif src == shard.rank:
            sends.setdefault(dst, []).append(a)
    return Plan(local_copies, sends, recvs)


def exchange(send_payloads: dict, recv_specs: dict, shard: Shard) -> dict:
    """Point-to-point exchange.  send_payloads[peer] = list of tensors;
    recv_specs[peer] = list of (shape, dtype) for the tensors to receive.
    Returns recv[peer] = list of tensors on the payload device."""
    out = {}
    if shard.world == 1:
        return out
    dev = _comm_device(shard)
    ops, keep = [], []
    for peer in sorted(set(send_payloads) | set(recv_specs)):
        for t in send_payloads.get(peer, []):
            tt = t.detach().contiguous().to(dev)
            keep.append(tt)
            ops.append(dist.P2POp(dist.isend, tt, peer, group=shard.group))
        bufs = [torch.empty(shape, dtype=dt, device=dev) for shape, dt in recv_specs.get(peer, [])]
        out[peer] = bufs
        for b in bufs:
            ops.append(dist.P2POp(dist.irecv, b, peer, group=shard.group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return out

"""SMC over parameters with MH rejuvenation -- SMC^2 with the device particle
filter inside (the reference's inference/smc.py:67-171 API).

The reference maps rejuvenation and propagation over theta-particles with a
GIL-bound thread pool (smc.py:60-64).  Here every phase is one batched
device launch per grid step over the theta-particles a rank owns:
  * theta-resampling: `resample` on the device, identical on every rank;
    local clones share history (ParticleRun.clone is copy-on-advance);
  * rejuvenation: all proposals replayed from t0 to the previous observation
    in ONE batched filter (the O(T^2) part, smc.py:100-122);
  * propagation: all attached filters advanced together (smc.py:125-134).
Multi-GPU: theta slots are sharded contiguously over
ranks.  Per observation step there is one all-gather of the theta
log-weights (C2) and one redistribution of the theta-particles whose
ancestor lives on another rank (C3: host fields + filter state + history,
NCCL point-to-point).  Draws are keyed by the global slot index
(step_rng.child(...)), so results do not depend on the number of ranks,
just as the reference's do not depend on nthreads.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .. import _lib
from ..distributed import Shard, allgather_f64, exchange, plan_redistribution
from ..errors import DegenerateEnsembleError, UnsupportedModelError
from ..models import resolve_model
from .mcmc import _chain_log_priors, marginal_mh_steps
from .particle import _dtype_info, advance_runs, sample_trajectories
from .resampling import resample


def _logsumexp(a):
    a = np.asarray(a, dtype=float)
    m = np.max(a)
    if np.isnan(m):
        return float("nan")
    if not np.isfinite(m):
        return float(m)
    return float(m + np.log(np.sum(np.exp(a - m))))


@dataclass
class ThetaParticle:
    theta: np.ndarray
    log_prior: float
    loglik: float = 0.0
    trajectory: np.ndarray = None
    init_state: np.ndarray = None
    run: object = None

    def clone(self):
        return ThetaParticle(theta=self.theta, log_prior=self.log_prior, loglik=self.loglik,
                             trajectory=self.trajectory, init_state=self.init_state,
                             run=self.run.clone() if self.run is not None else None)


@dataclass
class SmcResult:
    thetas: np.ndarray
    log_v: np.ndarray
    logliks: np.ndarray
    trajectories: np.ndarray
    particles: list = field(default_factory=list)  # this rank's theta-particles
    diagnostics: list = field(default_factory=list)


class _Children:
    """parent.child(a, j, b) on demand, indexed by j (a dict of them, built lazily)."""

    __slots__ = ("parent", "a", "b")

    def __init__(self, parent, a, b):
        self.parent, self.a, self.b = parent, a, b

    def __getitem__(self, j):
        return self.parent.child(self.a, j, self.b)


def _advance_all(runner, particles, js, upto, run_rngs, init_rngs, traj_rngs):
    """Create missing runs, advance all to `upto` in batches by position, refresh trajectories."""
    missing = [j for j in js if particles[j].run is None]
    if missing:
        runs = runner.new_runs([particles[j].theta for j in missing],
                               [particles[j].init_state for j in missing],
                               [init_rngs[j] for j in missing])
        for j, r in zip(missing, runs):
            particles[j].run = r
    incr = {}
    if runner.filter_kind == "kalman":  # device Kalman runs (kalman.py): exact increments, host backward draws
        from .kalman import advance_kalman_runs, sample_kalman_trajectories

        inc = advance_kalman_runs([particles[j].run for j in js], upto)
        for j, v in zip(js, inc):
            incr[j] = float(v)
        if traj_rngs is not None and js:
            trajs = sample_kalman_trajectories([particles[j].run for j in js], [traj_rngs[j] for j in js])
            for j, t in zip(js, trajs):
                particles[j].trajectory = t
        return incr
    by_pos = {}
    for j in js:
        by_pos.setdefault(particles[j].run.pos, []).append(j)
    for _, group in sorted(by_pos.items()):
        inc = advance_runs([particles[j].run for j in group], upto, [run_rngs[j] for j in group])
        for j, v in zip(group, inc):
            incr[j] = float(v)
    if traj_rngs is not None and js:
        trajs = sample_trajectories([particles[j].run for j in js], [traj_rngs[j] for j in js])
        for j, t in zip(js, trajs):
            particles[j].trajectory = t
    return incr


# ---------------------------------------------------------------- C3 payloads
#
# A theta-particle travels as one float64 host vector (theta, prior, loglik,
# trajectory, x0, run position / weighting state and, for history-free runs,
# the per-step Philox keys) plus its filter's device tensors:
#   keep_history=True : positions x_0..x_pos [pos+1, nx, P], ancestors [pos, P]
#   keep_history=False: current positions [nx, P] and ancestors [pos, P] only
#                       (the trajectory replay regenerates the line,
#                       ssm_replay_path) -- ~10x less than the stacked history
# then the unnormalised log-weights, the 64-byte filter state and, whenever the
# run carries the fused kernel's tile CDF (systematic / stratified and the
# device-noise sorted multinomial), cdf_local and the warp-tile records.


@dataclass(frozen=True)
class _Layout:
    have_run: bool
    traj_len: int
    pos: int
    has_a: bool
    has_tiles: bool
    keep_history: bool


def _host_len(spec, L):
    n = spec.n_param + 2 + L.traj_len * spec.nx + (spec.nx if spec.has_proposal_initial else 0) + 3
    if L.have_run and not L.keep_history:
        n += 2 * (L.pos + 1)  # Philox key (2 x uint32, exact in float64) per grid index
    return n


def _payload_specs(spec, L, P, tdtype):
    specs = [((_host_len(spec, L),), torch.float64)]
    if L.have_run:
        xs = (L.pos + 1, spec.nx, P) if L.keep_history else (spec.nx, P)
        specs += [(xs, tdtype), ((max(L.pos, 1), P), torch.int32), ((P,), tdtype), ((64,), torch.uint8)]
        if L.has_tiles:
            specs += [((P,), torch.int64), (((P + 31) // 32, 2), torch.float64)]
    return specs


def _pack(spec, L, p):
    host = [p.theta, [p.log_prior, p.loglik]]
    host.append(p.trajectory.reshape(-1) if L.traj_len else [])
    if spec.has_proposal_initial:
        host.append(p.init_state)
    r = p.run
    host.append([float(r.pos) if r else 0.0, float(r.weights_uniform) if r else 1.0,
                 float(r._maybe_nonuniform) if r else 0.0])
    if r is not None and not L.keep_history:
        host.append(np.asarray(r._kk, dtype=np.uint32).reshape(-1).astype(np.float64))
    out = [torch.from_numpy(np.concatenate([np.asarray(h, dtype=np.float64).reshape(-1) for h in host]))]
    if r is not None:
        P = r.n_particles
        ar = torch.arange(P, dtype=torch.int32, device=r.device)
        hist = [v for seg, b in r._segs for v in seg.views(b)]  # (x_i | None, anc_i | None) per grid index
        xs = torch.stack([h[0] for h in hist]) if L.keep_history else r._x
        ancs = [h[1] for h in hist[1:]]
        ha = torch.stack([a if a is not None else ar for a in ancs]) if r.pos > 0 else ar[None]
        a = r._a if r._a is not None else torch.zeros(P, dtype=r.tdtype, device=r.device)
        out += [xs, ha, a, r._fs.contiguous()]
        if L.has_tiles:
            out += [r._cdf if r._cdf is not None else torch.zeros(P, dtype=torch.int64, device=r.device),
                    r._trec if r._trec is not None else torch.zeros(((P + 31) // 32, 2), dtype=torch.float64,
                                                                    device=r.device)]
    return out


def _unpack(spec, runner, tensors, L):
    host = tensors[0].cpu().numpy()
    k = 0
    theta = host[k : k + spec.n_param].copy()
    k += spec.n_param
    log_prior, loglik = float(host[k]), float(host[k + 1])
    k += 2
    traj = host[k : k + L.traj_len * spec.nx].reshape(L.traj_len, spec.nx).copy() if L.traj_len else None
    k += L.traj_len * spec.nx
    init = None
    if spec.has_proposal_initial:
        init = host[k : k + spec.nx].copy()
        k += spec.nx
    pos, uniform, maybe = int(host[k]), bool(host[k + 1]), bool(host[k + 2])
    k += 3
    p = ThetaParticle(theta=theta, log_prior=log_prior, loglik=loglik, trajectory=traj, init_state=init)
    if len(tensors) > 1:
        run = runner._make(theta, init)
        dev = run.device
        xs = tensors[1].to(dev)
        ha = tensors[2].to(dev)
        if L.keep_history:
            run._set_history(xs, ha[:pos])
            run._x = xs[pos]
        else:
            keys = host[k : k + 2 * (pos + 1)].astype(np.uint32).reshape(pos + 1, 2)
            run._set_history(None, ha[:pos], keys)
            run._x = xs
        run._a = tensors[3].to(dev) if L.has_a else None
        run._fs = tensors[4].to(dev)
        if L.has_tiles:
            run._cdf = tensors[5].to(dev)
            run._trec = tensors[6].to(dev)
        run.pos, run.loglik, run.weights_uniform, run._maybe_nonuniform = pos, loglik, uniform, maybe
        fsv = run._fs.cpu().numpy().view(_lib.FILTER_STATE_DTYPE)[0]
        run.loglik = float(fsv["loglik"])
        p.run = run
    return p


def _redistribute(spec, runner, particles, anc, n, shard, lo):
    """particles: this rank's slots [lo, hi) (list); returns the new local list."""
    plan = plan_redistribution(anc, n, shard)
    local_src = {lo + i: p for i, p in enumerate(particles)}
    probe = particles[0] if particles else None
    have_run = probe is not None and probe.run is not None
    traj_len = 0 if probe is None or probe.trajectory is None else probe.trajectory.shape[0]
    # every rank holds particles in the same state, but a rank may own none: share the layout
    r = probe.run if have_run else None
    info = allgather_f64(np.array([float(have_run), float(traj_len), float(r.pos) if have_run else -1.0,
                                   float(r._a is not None) if have_run else 0.0,
                                   float(r._cdf is not None) if have_run else 0.0,
                                   float(r.keep_history) if have_run else 1.0]), shard).reshape(shard.world, 6)
    ref = info[np.argmax(info[:, 2])]
    L = _Layout(bool(ref[0]), int(ref[1]), int(ref[2]), bool(ref[3]), bool(ref[4]), bool(ref[5]))
    sends = {peer: [t for a in srcs for t in _pack(spec, L, local_src[a])] for peer, srcs in plan.sends.items()}
    P = runner.n_particles
    _, tdtype, _ = _dtype_info(runner.device_opts.get("dtype", "float64"))
    one = _payload_specs(spec, L, P, tdtype)
    recv_specs = {peer: one * len(dsts) for peer, dsts in plan.recvs.items()}
    got = exchange(sends, recv_specs, shard)
    new = {}
    for j, a in plan.local_copies:
        new[j] = local_src[a].clone()
    per = len(one)
    for peer, dsts in plan.recvs.items():
        ts = got[peer]
        for q, j in enumerate(dsts):
            new[j] = _unpack(spec, runner, ts[q * per : (q + 1) * per], L)
    hi = lo + len(particles)
    return [new[j] for j in range(lo, hi)]


# ---------------------------------------------------------------- the sampler


def smc_sampler(ir, runner, n_theta, rng, theta_resampler="multinomial", nthreads=1, shard=None,
                theta_draws=None):
    """smc.py:67-171 on the GPU.  `nthreads` is accepted for API compatibility
    (the batch is the parallelism); `shard` (paper_1306_3277_b200.distributed.Shard)
    spreads theta-particles over ranks, default: torch.distributed if initialised.
    `theta_draws` ("host" | "device") runs the rejuvenation move's theta-level
    blocks on the device (theta_mh.py); None keeps them on the host."""
    if n_theta < 2:
        raise ValueError("smc sampler needs n_theta >= 2")
    from ..profiling import gc_paused

    with gc_paused():
        return _smc_sampler(ir, runner, n_theta, rng, theta_resampler, shard, theta_draws)


def _smc_sampler(ir, runner, n_theta, rng, theta_resampler, shard, theta_draws):
    shard = shard or Shard.current()
    if runner.filter_kind == "kalman" and shard.world > 1:
        raise UnsupportedModelError("sharded SMC^2 moves particle-filter state; use the bootstrap filter")
    spec = resolve_model(ir)
    grid = runner.grid
    use_init = spec.has_proposal_initial
    lo, hi = shard.bounds(n_theta)
    J = list(range(lo, hi))
    # prior draws: the full ensemble's streams, sliced (identical on every rank)
    thetas = spec.sample_parameter(rng.child(0), size=n_theta)
    init_states = spec.sample_initial(thetas, rng.child(1), size=n_theta) if use_init else None
    local = []
    lps = _chain_log_priors(spec, [thetas[j] for j in J], [init_states[j] for j in J] if use_init else None)
    for j, lp in zip(J, lps):
        local.append(ThetaParticle(theta=thetas[j], log_prior=lp, init_state=init_states[j] if use_init else None))
    log_v = np.full(n_theta, -np.log(n_theta))
    counts = [shard_bounds_count(n_theta, r, shard.world) for r in range(shard.world)]
    diagnostics = []
    obs_steps = grid.obs_steps
    for i, grid_idx in enumerate(obs_steps, start=1):
        step_rng = rng.child(2, i)
        prev_idx = obs_steps[i - 2] if i > 1 else 0
        # theta-resample (smc.py:96-98): same ancestors on every rank
        anc = resample(np.exp(log_v - _logsumexp(log_v)), theta_resampler, step_rng.child(0))
        if shard.world == 1:
            # the old list is dropped: each ancestor's first copy can be the particle itself
            seen = bytearray(len(local))
            picked = []
            for a in anc:
                if seen[a]:
                    picked.append(local[a].clone())
                else:
                    seen[a] = 1
                    picked.append(local[a])
            local = picked
        else:
            local = _redistribute(spec, runner, local, anc, n_theta, shard, lo)
        particles = dict(zip(J, local))
        # rejuvenate: one marginal MH move each, one batched replay (smc.py:101-122)
        # the MH step reads theta, init_state, loglik and log_prior of each chain state:
        # the theta-particles themselves serve (MhChainState duck type, read only)
        chains = local
        # the rejuvenated filters' trajectories are redrawn by the propagation below: not drawn here
        if theta_draws is None:
            outs = marginal_mh_steps(ir, chains, runner, [step_rng.child(1, j) for j in J], upto=prev_idx,
                                     trajectories=False)
        else:
            from .theta_mh import marginal_mh_steps_device

            outs, _ = marginal_mh_steps_device(ir, chains, runner, [step_rng.child(1, j) for j in J], upto=prev_idx,
                                               draws=theta_draws, step=i, trajectories=False)
        accepted = []
        for p, (new, ok, run) in zip(local, outs):
            if ok:
                p.theta, p.log_prior, p.loglik = new.theta, new.log_prior, new.loglik
                p.trajectory, p.init_state, p.run = new.trajectory, new.init_state, run
            accepted.append(ok)
        # propagate and weight (smc.py:125-134)
        rr = {j: step_rng.child(2, j, 1) for j in J}
        ir_ = _Children(step_rng, 2, 0)  # only the theta-particles without a run draw from these
        # only the last step's trajectories reach the result (each draws from its own stream,
        # smc.py:131, so skipping the intermediate ones leaves every other draw unchanged)
        tr = {j: step_rng.child(3, j) for j in J} if i == len(obs_steps) else None
        incr = _advance_all(runner, particles, J, grid_idx, run_rngs=rr, init_rngs=ir_, traj_rngs=tr)
        for j in J:
            particles[j].loglik += incr[j]
        log_v = allgather_f64(np.array([incr[j] for j in J]), shard, counts)  # C2
        acc_all = allgather_f64(np.array(accepted, dtype=float), shard, counts)
        lse = _logsumexp(log_v)
        if not np.isfinite(lse):
            t = float(grid.times[grid_idx])
            raise DegenerateEnsembleError(f"all theta-weights vanished at t={t:g}", time=t)
        norm = np.exp(log_v - lse)
        diagnostics.append({"time": float(grid.times[grid_idx]), "ess": float(1.0 / np.sum(norm ** 2)),
                            "acceptance": float(np.mean(acc_all))})

    # finalize (smc.py:150-161)
    particles = dict(zip(J, local))
    need_new = [j for j in J if particles[j].run is None]
    if need_new:
        runs = runner.new_runs([particles[j].theta for j in need_new],
                               [particles[j].init_state for j in need_new],
                               [rng.child(3, j, 0) for j in need_new])
        for j, r in zip(need_new, runs):
            particles[j].run = r
    behind = [j for j in J if particles[j].run.pos < grid.last]
    if behind:
        _advance_all(runner, particles, behind, grid.last, run_rngs={j: rng.child(3, j, 1) for j in behind},
                     init_rngs=None, traj_rngs={j: rng.child(3, j, 2) for j in behind})
    stale = [j for j in J if particles[j].trajectory is None]
    if stale:
        trajs = sample_trajectories([particles[j].run for j in stale], [rng.child(3, j, 2) for j in stale])
        for j, t in zip(stale, trajs):
            particles[j].trajectory = t
    log_v = log_v - _logsumexp(log_v)
    S1 = grid.last + 1
    th = allgather_f64(np.concatenate([particles[j].theta for j in J]) if J else np.zeros(0), shard,
                       [c * spec.n_param for c in counts]).reshape(n_theta, spec.n_param)
    ll = allgather_f64(np.array([particles[j].loglik for j in J]), shard, counts)
    tj = allgather_f64(np.concatenate([particles[j].trajectory.reshape(-1) for j in J]) if J else np.zeros(0),
                       shard, [c * S1 * spec.nx for c in counts]).reshape(n_theta, S1, spec.nx)
    return SmcResult(thetas=th, log_v=log_v, logliks=ll, trajectories=tj,
                     particles=[particles[j] for j in J], diagnostics=diagnostics)


def shard_bounds_count(n, rank, world):
    from ..distributed import shard_bounds

    lo, hi = shard_bounds(n, rank, world)
    return hi - lo

"""SMC over parameters with MH rejuvenation -- SMC^2 with the device particle
filter inside (the reference's inference/smc.py:67-171 API).

The reference maps rejuvenation and propagation over theta-particles with a
GIL-bound thread pool (smc.py:60-64).  Here every phase is one batched
device launch per grid step over all theta-particles:
  * theta-resampling: `resample` on the device; clones share history
    (ParticleRun.clone is copy-on-advance);
  * rejuvenation: all proposals replayed from t0 to the previous
    observation in ONE batched filter (the O(T^2) part, smc.py:100-122);
  * propagation: all attached filters advanced together (smc.py:125-134).
Draws use the reference's stream keys (step_rng.child(...)) so the result is
independent of batching, like the reference's independence of nthreads.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ..errors import DegenerateEnsembleError
from ..models import resolve_model
from .mcmc import MhChainState, _chain_log_prior, marginal_mh_steps
from .particle import advance_runs, sample_trajectories
from .resampling import resample


def _logsumexp(a):
    a = np.asarray(a, dtype=float)
    m = np.max(a)
    if not np.isfinite(m):
        return float(m) if m == np.inf else float("-inf") if np.all(a == -np.inf) else float("nan")
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
    particles: list = field(default_factory=list)
    diagnostics: list = field(default_factory=list)


def _advance_all(runner, particles, js, upto, run_rngs, init_rngs, traj_rngs):
    """Create missing runs, advance all to `upto` in one batch, refresh trajectories."""
    missing = [j for j in js if particles[j].run is None]
    if missing:
        runs = runner.new_runs([particles[j].theta for j in missing],
                               [particles[j].init_state for j in missing],
                               [init_rngs[j] for j in missing])
        for j, r in zip(missing, runs):
            particles[j].run = r
    # group by position (all equal in practice)
    incr = {}
    by_pos = {}
    for j in js:
        by_pos.setdefault(particles[j].run.pos, []).append(j)
    for _, group in sorted(by_pos.items()):
        inc = advance_runs([particles[j].run for j in group], upto, [run_rngs[j] for j in group])
        for j, v in zip(group, inc):
            incr[j] = float(v)
    if traj_rngs is not None:
        trajs = sample_trajectories([particles[j].run for j in js], [traj_rngs[j] for j in js])
        for j, t in zip(js, trajs):
            particles[j].trajectory = t
    return incr


def smc_sampler(ir, runner, n_theta, rng, theta_resampler="multinomial", nthreads=1):
    """smc.py:67-171 on the GPU (nthreads is accepted for API compatibility;
    the batch is the parallelism)."""
    if n_theta < 2:
        raise ValueError("smc sampler needs n_theta >= 2")
    spec = resolve_model(ir)
    grid = runner.grid
    use_init = spec.has_proposal_initial
    thetas = spec.sample_parameter(rng.child(0), size=n_theta)
    init_states = spec.sample_initial(thetas, rng.child(1), size=n_theta) if use_init else None
    particles = []
    for j in range(n_theta):
        ist = init_states[j] if use_init else None
        particles.append(ThetaParticle(theta=thetas[j], log_prior=_chain_log_prior(spec, thetas[j], ist),
                                       init_state=ist))
    log_v = np.full(n_theta, -np.log(n_theta))
    diagnostics = []
    obs_steps = grid.obs_steps
    J = list(range(n_theta))
    for i, grid_idx in enumerate(obs_steps, start=1):
        step_rng = rng.child(2, i)
        prev_idx = obs_steps[i - 2] if i > 1 else 0
        # theta-resample (smc.py:96-98)
        anc = resample(np.exp(log_v - _logsumexp(log_v)), theta_resampler, step_rng.child(0))
        particles = [particles[a].clone() for a in anc]
        # rejuvenate: one marginal MH move each, batched replays (smc.py:101-122)
        chains = [MhChainState(theta=p.theta, trajectory=p.trajectory, loglik=p.loglik,
                               log_prior=p.log_prior, init_state=p.init_state) for p in particles]
        outs = marginal_mh_steps(ir, chains, runner, [step_rng.child(1, j) for j in J], upto=prev_idx)
        accepted = []
        for p, (new, ok, run) in zip(particles, outs):
            if ok:
                p.theta, p.log_prior, p.loglik = new.theta, new.log_prior, new.loglik
                p.trajectory, p.init_state, p.run = new.trajectory, new.init_state, run
            accepted.append(ok)
        # propagate and weight (smc.py:125-134)
        incr = _advance_all(runner, particles, J, grid_idx,
                            run_rngs=[step_rng.child(2, j, 1) for j in J],
                            init_rngs=[step_rng.child(2, j, 0) for j in J],
                            traj_rngs=[step_rng.child(3, j) for j in J])
        for j in J:
            particles[j].loglik += incr[j]
        log_v = np.array([incr[j] for j in J])
        lse = _logsumexp(log_v)
        if not np.isfinite(lse):
            t = float(grid.times[grid_idx])
            raise DegenerateEnsembleError(f"all theta-weights vanished at t={t:g}", time=t)
        norm = np.exp(log_v - lse)
        diagnostics.append({"time": float(grid.times[grid_idx]), "ess": float(1.0 / np.sum(norm ** 2)),
                            "acceptance": float(np.mean(accepted))})

    # finalize (smc.py:150-161)
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
    return SmcResult(thetas=np.stack([p.theta for p in particles]), log_v=log_v,
                     logliks=np.array([p.loglik for p in particles]),
                     trajectories=np.stack([p.trajectory for p in particles]),
                     particles=particles, diagnostics=diagnostics)

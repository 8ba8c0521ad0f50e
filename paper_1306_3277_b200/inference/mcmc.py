"""Marginal Metropolis-Hastings over parameters (PMMH) with the device
particle filter inside -- the reference's inference/mcmc.py:28-180 API.

`FilterRunner` is the drop-in factory (mcmc.py:54-108): `new_run` /
`run` build a `ParticleRun` on the GPU.  `run_batch` advances many filters
in one launch per step; `mh_sample_chains` uses it to run C independent
PMMH chains in lock-step (config 3: 64 chains), giving exactly the draws of
C serial `mh_sample` calls with streams rngs[c].  theta-level proposals and
priors run on the host by default, or on the device with
`theta_draws=` (theta_mh.py).
"""

from __future__ import annotations


from dataclasses import dataclass

import numpy as np

from ..models import propose_batch, resolve_model
from .particle import ParticleRun, advance_runs, init_runs, sample_trajectories
from .timegrid import as_filter_grid

_FILTER_KEY = 7  # mcmc.py:25


def metropolis_accept(log_ratio, rng):
    """Accept iff u <= exp(log_ratio), u ~ U(0,1)  (mcmc.py:28-33)."""
    if np.isnan(log_ratio) or log_ratio == -np.inf:
        return False
    u = rng.uniform()
    return bool(u <= np.exp(min(log_ratio, 0.0)))


@dataclass
class MhChainState:
    theta: np.ndarray
    trajectory: np.ndarray
    loglik: float
    log_prior: float
    init_state: np.ndarray = None


class FilterRunner:
    """Builds and runs the bootstrap filter on the GPU for a given theta."""

    def __init__(self, ir, grid, inputs=None, filter_kind="bootstrap", n_particles=1024,
                 resampler="multinomial", ess_rel=None, check_finite=True, **device_opts):
        if filter_kind not in ("kalman", "bootstrap"):
            raise ValueError(f"unknown filter {filter_kind!r}")
        self.ir = ir
        self.spec = resolve_model(ir)
        self.grid = as_filter_grid(grid)
        self.inputs = inputs
        self.filter_kind = filter_kind
        self.n_particles = n_particles
        self.resampler = resampler
        self.ess_rel = ess_rel
        self.check_finite = check_finite
        self.device_opts = dict(device_opts)

    def _systems(self, thetas, init_states):
        """Linear-Gaussian systems of a batch (mcmc.py:81-87): x0 proposals pin the initial state."""
        from ..lineargauss import extract_linear_gaussian

        src = self.spec if isinstance(self.ir, str) else self.ir
        sys_ = extract_linear_gaussian(src, np.asarray(thetas, dtype=float).reshape(len(thetas), -1),
                                       self.grid.times, self.inputs)
        for k, st in enumerate(init_states):
            if st is not None:
                sys_.mu0[k] = np.asarray(st, dtype=float)
                sys_.P0[k] = 0.0
        return sys_

    def _make(self, theta, init_state):
        return ParticleRun(self.spec, theta, self.grid, inputs=self.inputs, n_particles=self.n_particles,
                           resampler=self.resampler, ess_rel=self.ess_rel, initial_state=init_state,
                           check_finite=self.check_finite, **self.device_opts)

    def new_run(self, theta, init_state, rng):
        """Fresh, initialised (not yet advanced) filter run (mcmc.py:79-100)."""
        if self.filter_kind == "kalman":
            return self.new_runs([theta], [init_state], [rng])[0]
        return self._make(theta, init_state).init(rng.child(0))

    def new_runs(self, thetas, init_states, rngs):
        # one validated run, then per-theta shallow copies (the constructor's checks
        # and lookups are per runner, not per theta; SMC^2 builds ~100 runs per step)
        if not thetas:
            return []
        if self.filter_kind == "kalman":
            from .kalman import kalman_runs

            return kalman_runs(self._systems(thetas, init_states), self.grid, self.device_opts.get("device"))
        proto = self._make(thetas[0], init_states[0])
        runs = [proto]
        base = proto.__dict__
        cls = type(proto)
        for t, st in zip(thetas[1:], init_states[1:]):
            r = cls.__new__(cls)  # a shallow copy of the validated prototype
            d = dict(base)
            d["theta"] = np.asarray(t, dtype=float).reshape(1, -1)
            d["initial_state"] = st
            d["_derived"] = None
            d["_segs"] = []  # init_runs installs the history and pointer arrays
            r.__dict__ = d
            runs.append(r)
        init_runs(runs, [g.child(0) for g in rngs])
        return runs

    def trajectories(self, runs, rngs):
        """sample_trajectory for a batch of this runner's runs (each from its own stream)."""
        if not runs:
            return []
        if self.filter_kind == "kalman":
            from .kalman import sample_kalman_trajectories

            return sample_kalman_trajectories(runs, rngs)
        return sample_trajectories(runs, rngs)

    def run(self, theta, init_state, rng, upto=None):
        """(loglik, trajectory, run) over grid steps 1..upto (mcmc.py:102-108)."""
        out = self.run_batch([theta], [init_state], [rng], upto=upto)
        return out[0]

    def run_batch(self, thetas, init_states, rngs, upto=None, trajectories=True):
        """Batched FilterRunner.run: one launch per step for all filters.
        trajectories=False skips the trajectory draws (their slot is None): a
        caller that discards them (SMC^2 rejuvenation, whose trajectories are
        redrawn at the propagation) saves a trace and a read-back."""
        upto = self.grid.last if upto is None else upto
        if not thetas:
            return []
        runs = self.new_runs(thetas, init_states, rngs)
        if self.filter_kind == "kalman":
            from .kalman import advance_kalman_runs, sample_kalman_trajectories

            advance_kalman_runs(runs, upto)
            trajs = (sample_kalman_trajectories(runs, [g.child(2) for g in rngs]) if trajectories
                     else [None] * len(runs))
            return [(r.loglik, t, r) for r, t in zip(runs, trajs)]
        advance_runs(runs, upto, [g.child(1) for g in rngs])
        trajs = sample_trajectories(runs, [g.child(2) for g in rngs]) if trajectories else [None] * len(runs)
        return [(r.loglik, t, r) for r, t in zip(runs, trajs)]


def _chain_log_prior(spec, theta, init_state):
    lp = spec.parameter_logpdf(theta)
    if init_state is not None:
        lp += spec.initial_logpdf(theta, init_state)
    return lp


def _chain_log_priors(spec, thetas, init_states):
    """_chain_log_prior for a batch of chains (SMC^2's theta-particles): the
    hand-written models' densities evaluated column-wise over the batch with the
    scalar path's addition order (bitwise the same values); other models per chain."""
    from ..models import ModelSpec, d_gauss_logpdf, d_uniform_logpdf, parameter_logpdf_batch

    n = len(thetas)
    if not isinstance(spec, ModelSpec) or n == 0:
        return [_chain_log_prior(spec, thetas[k], None if init_states is None else init_states[k]) for k in range(n)]
    lp = parameter_logpdf_batch(spec, np.asarray(thetas, dtype=float))
    if init_states is not None:
        X0 = np.atleast_2d(np.asarray(init_states, dtype=float))
        tot = np.zeros(n)
        if spec.name == "Lorenz96":
            for i in range(8):
                tot = tot + d_uniform_logpdf(X0[:, i], -1.0, 3.0)
        else:
            tot = tot + d_gauss_logpdf(X0[:, 0], 90.0, 15.0)
        lp = lp + tot
    return [float(v) for v in lp]


def init_chain(ir, runner, rng, upto=None):
    """mcmc.py:118-132."""
    return init_chains(ir, runner, [rng], upto)[0]


def init_chains(ir, runner, rngs, upto=None):
    spec = resolve_model(ir)
    thetas, inits = [], []
    for rng in rngs:
        theta = spec.sample_parameter(rng, size=1)[0]
        init_state = None
        if spec.has_proposal_initial:
            init_state = spec.sample_initial(theta, rng, size=1)[0]
        thetas.append(theta)
        inits.append(init_state)
    res = runner.run_batch(thetas, inits, [g.child(_FILTER_KEY) for g in rngs], upto=upto)
    return [
        MhChainState(theta=th, trajectory=traj, loglik=ll, log_prior=_chain_log_prior(spec, th, ist),
                     init_state=ist)
        for th, ist, (ll, traj, _) in zip(thetas, inits, res)
    ]


def _propose(spec, chain, rng):
    theta_new, logq_fwd = spec.propose_parameters(chain.theta, rng)
    logq_rev = spec.proposal_parameter_logpdf(theta_new, chain.theta)
    init_new = None
    if chain.init_state is not None:
        init_new, lq = spec.propose_initial(theta_new, chain.init_state, rng)
        logq_fwd += lq
        logq_rev += spec.proposal_initial_logpdf(chain.theta, init_new, chain.init_state)
    log_prior_new = _chain_log_prior(spec, theta_new, init_new)
    return theta_new, init_new, logq_fwd, logq_rev, log_prior_new


def marginal_mh_step(ir, chain, runner, rng, upto=None, reference=None):
    """One marginal MH transition (mcmc.py:135-166); returns (state, accepted, run)."""
    return marginal_mh_steps(ir, [chain], runner, [rng], upto, [reference])[0]


def marginal_mh_steps(ir, chains, runner, rngs, upto=None, references=None, trajectories=True):
    """Lock-step marginal MH over independent chains: host proposals, one
    batched device filter run for every chain inside the prior support,
    then per-chain accept/reject with the chain's own stream.
    trajectories=False: accepted states carry trajectory None (see run_batch)."""
    spec = resolve_model(ir)
    references = references or [None] * len(chains)
    if not chains:
        return []
    # vectorised over chains; per-stream draws in the reference's order (bit-identical to _propose)
    th_new, x0_new, lq_f, lq_r, lp_new = propose_batch(
        spec, [c.theta for c in chains], [c.init_state for c in chains] if chains[0].init_state is not None else None,
        rngs)
    props = [(th_new[k], x0_new[k], float(lq_f[k]), float(lq_r[k]), float(lp_new[k])) for k in range(len(chains))]
    todo = [k for k, p in enumerate(props) if p[4] != -np.inf]
    # the filters first, trajectories only for the accepted proposals (each draws from its
    # own stream, so skipping the rejected ones changes no other draw)
    res = runner.run_batch([props[k][0] for k in todo], [props[k][1] for k in todo],
                           [rngs[k].child(_FILTER_KEY) for k in todo], upto=upto, trajectories=False)
    by_k = dict(zip(todo, res))
    out = []
    accepted = []
    for k, (chain, rng) in enumerate(zip(chains, rngs)):
        theta_new, init_new, logq_fwd, logq_rev, log_prior_new = props[k]
        if k not in by_k:
            out.append((chain, False, None))  # outside the prior support: auto-reject
            continue
        loglik_new, _, run = by_k[k]
        current = chain.loglik if references[k] is None else references[k]
        log_ratio = (loglik_new + log_prior_new + logq_rev) - (current + chain.log_prior + logq_fwd)
        if metropolis_accept(log_ratio, rng):
            out.append((MhChainState(theta=theta_new, trajectory=None, loglik=loglik_new,
                                     log_prior=log_prior_new, init_state=init_new), True, run))
            accepted.append(k)
        else:
            out.append((chain, False, None))
    if trajectories and accepted:
        trajs = runner.trajectories([by_k[k][2] for k in accepted],
                                    [rngs[k].child(_FILTER_KEY).child(2) for k in accepted])
        for k, t in zip(accepted, trajs):
            out[k][0].trajectory = t
    return out


def mh_sample(ir, runner, n_samples, rng):
    """mcmc.py:169-180: (list of MhChainState, acceptance count)."""
    chains, acc = mh_sample_chains(ir, runner, n_samples, [rng])
    return chains[0], int(acc[0])


def mh_sample_chains(ir, runner, n_samples, rngs, upto=None, on_step=None, shard=None, theta_draws=None):
    """C independent PMMH chains advanced in lock-step (batched filters).
    Chain c reproduces mh_sample(ir, runner, n_samples, rngs[c]).

    `theta_draws` moves the theta-level blocks (proposal walk, densities,
    prior, accept) onto the device (theta_mh.py): "host"
    injects the reference's draws (parity mode), "device" draws with Philox;
    None keeps them on the host.

    Multi-GPU (config 3): with a `Shard` (default: torch.distributed
    if initialised) each rank runs its contiguous block of chains as
    independent replicas; the samples are all-gathered at the end (C4), so
    every rank returns all C chains."""
    from ..profiling import gc_paused

    with gc_paused():
        return _mh_sample_chains(ir, runner, n_samples, rngs, upto, on_step, shard, theta_draws)


def _mh_sample_chains(ir, runner, n_samples, rngs, upto, on_step, shard, theta_draws):
    from ..distributed import Shard, allgather_f64, shard_bounds

    shard = shard or Shard.current()
    C = len(rngs)
    lo, hi = shard.bounds(C)
    mine = list(rngs[lo:hi])
    samples = [[] for _ in mine]
    accepted = np.zeros(len(mine), dtype=int)
    if mine:
        states = init_chains(ir, runner, [g.child(0) for g in mine], upto=upto)
        dev = None
        for step in range(1, n_samples + 1):
            if theta_draws is None:
                outs = marginal_mh_steps(ir, states, runner, [g.child(step) for g in mine], upto=upto)
            else:
                from .theta_mh import marginal_mh_steps_device

                outs, dev = marginal_mh_steps_device(ir, states, runner, [g.child(step) for g in mine], upto=upto,
                                                     draws=theta_draws, dev=dev, step=step)
            for c, (st, ok, _) in enumerate(outs):
                states[c] = st
                accepted[c] += int(ok)
                samples[c].append(st)
            if on_step is not None:
                on_step(step, states)
    if shard.world == 1:
        return samples, accepted
    # C4: gather every chain's record (theta, loglik, log_prior, x0, trajectory) to every rank
    spec = resolve_model(ir)
    S1 = runner.grid.last + 1 if upto is None else upto + 1
    nx0 = spec.nx if spec.has_proposal_initial else 0
    rec = spec.n_param + 2 + nx0 + S1 * spec.nx
    flat = []
    for ch in samples:
        for st in ch:
            parts = [st.theta, [st.loglik, st.log_prior]]
            if nx0:
                parts.append(st.init_state)
            parts.append(st.trajectory.reshape(-1))
            flat.append(np.concatenate([np.asarray(q, dtype=float).reshape(-1) for q in parts]))
    counts = [(shard_bounds(C, r, shard.world)[1] - shard_bounds(C, r, shard.world)[0]) * n_samples * rec
              for r in range(shard.world)]
    allrec = allgather_f64(np.concatenate(flat) if flat else np.zeros(0), shard, counts).reshape(C, n_samples, rec)
    acc_all = allgather_f64(accepted.astype(float), shard,
                            [shard_bounds(C, r, shard.world)[1] - shard_bounds(C, r, shard.world)[0]
                             for r in range(shard.world)]).astype(int)
    out = []
    for c in range(C):
        chain = []
        for k in range(n_samples):
            v = allrec[c, k]
            th = v[: spec.n_param].copy()
            q = spec.n_param
            ll, lp = float(v[q]), float(v[q + 1])
            q += 2
            x0 = v[q : q + nx0].copy() if nx0 else None
            q += nx0
            chain.append(MhChainState(theta=th, trajectory=v[q:].reshape(S1, spec.nx).copy(), loglik=ll,
                                      log_prior=lp, init_state=x0))
        out.append(chain)
    return out, acc_all

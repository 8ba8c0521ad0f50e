"""Theta-level marginal MH on the device.

The reference proposes, scores and accepts each chain on the host
(mcmc.py:_propose 138-148, marginal_mh_step 151-166, metropolis_accept 28-33;
simulate.py:220-352).  Here `ssm_theta_propose` draws the proposal walk of
every chain (theta, and x0 when the model has proposal_initial), its forward
and reverse proposal log-densities and the prior of the proposal in one
launch, and `ssm_theta_accept` applies the MH accept to all chains in a
second launch after the batched filter.  The chain state (theta, x0, loglik,
log prior) stays resident on the device between MH steps.

Draws:
  * ``draws="device"``: Philox keyed by each chain's per-step stream (fresh
    streams, independent of batching); statistically equivalent to the
    reference, not stream-identical.
  * ``draws="host"``: the reference's own numpy draws from each chain's stream,
    in its order (the uniforms of the truncated-Gaussian statements, the gamma
    variate of the inverse-gamma statement, the x0 uniforms, then the accept
    uniform), injected.  This is the parity mode: the result equals
    `marginal_mh_steps` up to normcdf/normcdfinv rounding (~1e-15 relative).

Generic models (codegen.py) run the same two launches: the generated
`Theta` walks (`ssm_gen_theta_propose`, ssm_gen_rt.cuh) and the shared accept.
Their injected draws are the standard variates of the reference's own
numpy calls, recorded while its walk runs on each chain's stream
(`_RecordingStream`).
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _lib
from ..errors import DistributionParameterError, UnsupportedModelError
from ..models import resolve_model
from ..rng import device_keys, prime_streams
from .mcmc import _FILTER_KEY, MhChainState

DRAW_MODES = ("device", "host")


class _RecordingStream:
    """Stands in for a chain's RngStream while the reference's walk draws from it
    (generic.GenericModel.propose_parameters / propose_initial): every draw is
    taken as a standard variate from the stream -- the same generator calls,
    so the stream advances exactly as under the reference -- recorded, and
    scaled the way numpy's own distribution functions scale it (loc + scale z,
    low + (high - low) u, scale * standard_gamma)."""

    def __init__(self, rng):
        self.rng = rng
        self.draws = []

    def normal(self, loc=0.0, scale=1.0, size=None):
        z = np.asarray(self.rng.normal(0.0, 1.0, size=size), dtype=float)
        self.draws.extend(np.ravel(z).tolist())
        return np.asarray(loc, dtype=float) + np.asarray(scale, dtype=float) * z

    def uniform(self, low=0.0, high=1.0, size=None):
        u = np.asarray(self.rng.uniform(0.0, 1.0, size=size), dtype=float)
        self.draws.extend(np.ravel(u).tolist())
        lo = np.asarray(low, dtype=float)
        return lo + (np.asarray(high, dtype=float) - lo) * u

    def gamma(self, shape, scale=1.0, size=None):
        g = np.asarray(self.rng.gamma(shape, 1.0, size=size), dtype=float)
        self.draws.extend(np.ravel(g).tolist())
        return np.asarray(scale, dtype=float) * g


class DeviceThetaChains:
    """Device-resident state of C chains plus the proposal buffers."""

    def __init__(self, ir, states, device=None):
        spec = resolve_model(ir)
        self.generic = spec.kernel == _lib.SSM_MODEL_GENERIC
        if not self.generic and spec.kernel not in (_lib.SSM_MODEL_LORENZ96, _lib.SSM_MODEL_WINDKESSEL):
            raise UnsupportedModelError(f"{spec.name}: no device theta-level blocks")
        self.has_init = bool(states and states[0].init_state is not None)
        if self.generic:
            from .. import codegen

            if not codegen.theta_supported(spec.desc):
                raise UnsupportedModelError(f"{spec.name}: a theta-level statement the device walk cannot sample")
        elif self.has_init and not spec.has_proposal_initial:
            raise UnsupportedModelError(f"{spec.name} has no proposal_initial block")
        _lib.require_cuda()
        self.spec = spec
        self.device = torch.device(device if device is not None else "cuda")
        self.C = len(states)
        f64 = dict(dtype=torch.float64, device=self.device)
        C, npar, nx = self.C, spec.n_param, spec.nx
        # one pinned host block, one asynchronous copy (no stream synchronisation)
        q = C * npar + (C * nx if self.has_init else 0)
        host = np.empty(q + 2 * C)
        host[: C * npar] = np.array([s.theta for s in states], dtype=float).reshape(-1)
        if self.has_init:
            host[C * npar : q] = np.array([s.init_state for s in states], dtype=float).reshape(-1)
        host[q : q + C] = [float(s.loglik) for s in states]
        host[q + C :] = [float(s.log_prior) for s in states]
        dev_all = _lib.h2d(host, self.device)
        self.theta = dev_all[: C * npar].view(C, npar)
        self.x0 = dev_all[C * npar : q].view(C, nx) if self.has_init else None
        self.loglik = dev_all[q : q + C]
        self.log_prior = dev_all[q + C :]
        self.theta_new = torch.empty(C, npar, **f64)
        self.x0_new = torch.empty(C, nx, **f64) if self.has_init else None
        self.lq_f = torch.empty(C, **f64)
        self.lq_r = torch.empty(C, **f64)
        self.lp_new = torch.empty(C, **f64)
        self.ll_new = torch.empty(C, **f64)
        self.accepted = torch.empty(C, dtype=torch.int32, device=self.device)
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        if self.generic:
            self._handle = spec.handle(self.device)
            self.u_stride = _lib.lib().ssm_gen_theta_draws(self._handle, int(self.has_init))
        else:
            self.u_stride = _lib.lib().ssm_theta_draws(spec.kernel, int(self.has_init))
        self._inj = None
        self._keys = None

    def _args(self, step=0):
        a = _lib.ThetaArgs()
        a.model, a.n_chains, a.n_param, a.nx = self.spec.kernel, self.C, self.spec.n_param, self.spec.nx
        a.has_init, a.u_stride, a.step = int(self.has_init), self.u_stride, int(step)
        p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        a.keys = p(self._keys)
        a.theta, a.x0, a.theta_new, a.x0_new = p(self.theta), p(self.x0), p(self.theta_new), p(self.x0_new)
        a.logq_fwd, a.logq_rev, a.log_prior_new = p(self.lq_f), p(self.lq_r), p(self.lp_new)
        a.loglik, a.log_prior, a.loglik_new = p(self.loglik), p(self.log_prior), p(self.ll_new)
        a.accepted, a.err = p(self.accepted), p(self.err)
        if self._inj is not None:
            a.u_in, a.g_in, a.u_acc_in = (p(t) for t in self._inj)
        return a

    def _host_draws_generic(self, rngs):
        """The reference's walk on each chain's stream with the draws recorded
        (GenericModel.propose_batch order), then the accept uniform."""
        spec, C = self.spec, self.C
        th = self.theta.cpu().numpy()
        x0 = self.x0.cpu().numpy() if self.has_init else None
        u = np.zeros((C, self.u_stride))
        ua = np.zeros(C)
        prime_streams(rngs)
        for c, rng in enumerate(rngs):
            rec = _RecordingStream(rng)
            th_new, _ = spec.propose_parameters(th[c], rec)
            if self.has_init:
                spec.propose_initial(th_new, x0[c], rec)
            if len(rec.draws) != self.u_stride - 1:
                raise UnsupportedModelError(f"{spec.name}: {len(rec.draws)} theta-level draws, "
                                            f"expected {self.u_stride - 1}")
            u[c, : self.u_stride - 1] = rec.draws
            ua[c] = rng.uniform()
        return u, np.zeros(C), ua

    def host_draws(self, rngs):
        """The reference's draws from each chain stream, in its order (models.propose_batch,
        then metropolis_accept): (u [C][u_stride], g [C], u_acc [C])."""
        if self.generic:
            return self._host_draws_generic(rngs)
        spec, C = self.spec, self.C
        n_tg = 1 if spec.kernel == _lib.SSM_MODEL_LORENZ96 else 3
        ig = n_tg
        th = self.theta.cpu().numpy()
        u = np.zeros((C, self.u_stride))
        g = np.zeros(C)
        ua = np.zeros(C)
        scale = 1.0 / (3.0 * th[:, ig])
        prime_streams(rngs)
        for c, rng in enumerate(rngs):
            u[c, :n_tg] = rng.uniform(size=n_tg)
            g[c] = rng.gamma(2.0, np.asarray(scale[c]), size=1)[0]
            if self.has_init:
                u[c, n_tg : n_tg + spec.nx] = rng.uniform(size=spec.nx)
            ua[c] = rng.uniform()
        return u, g, ua

    def propose(self, rngs, step, draws="device", stream=None):
        """One ssm_theta_propose launch; returns host copies (theta_new, x0_new, lq_f, lq_r, lp_new)."""
        if draws not in DRAW_MODES:
            raise ValueError(f"draws must be one of {DRAW_MODES}")
        if draws == "host":
            self._inj = tuple(_lib.h2d(np.ascontiguousarray(v, dtype=np.float64), self.device)
                              for v in self.host_draws(rngs))
            self._keys = None
        else:
            self._inj = None
            keys = np.ascontiguousarray(device_keys(rngs), dtype=np.uint32).view(np.int32)  # bit pattern kept
            self._keys = _lib.h2d(keys, self.device)
        self.err.zero_()
        with torch.cuda.device(self.device):
            if self.generic:
                _lib.check(_lib.lib().ssm_gen_theta_propose(self._handle, self._args(step), _lib.stream_ptr(stream)),
                           "ssm_gen_theta_propose")
            else:
                _lib.check(_lib.lib().ssm_theta_propose(self._args(step), _lib.stream_ptr(stream)),
                           "ssm_theta_propose")
        packed = torch.cat([self.theta_new.reshape(-1)] + ([self.x0_new.reshape(-1)] if self.has_init else []) +
                           [self.lq_f, self.lq_r, self.lp_new, self.err.to(torch.float64)]).cpu().numpy()
        if packed[-1] != 0:
            raise DistributionParameterError("theta proposal: invalid distribution parameter")
        C, npar, nx = self.C, self.spec.n_param, self.spec.nx
        q = C * npar
        th = packed[:q].reshape(C, npar)
        x0 = None
        if self.has_init:
            x0 = packed[q : q + C * nx].reshape(C, nx)
            q += C * nx
        return th, x0, packed[q : q + C], packed[q + C : q + 2 * C], packed[q + 2 * C : q + 3 * C]

    def accept(self, loglik_new, step, stream=None):
        """One ssm_theta_accept launch over all chains; returns the accepted flags (host)."""
        self.ll_new.copy_(_lib.h2d(np.asarray(loglik_new, dtype=float), self.device))
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().ssm_theta_accept(self._args(step), _lib.stream_ptr(stream)), "ssm_theta_accept")
        return self.accepted.cpu().numpy().astype(bool)


def marginal_mh_steps_device(ir, chains, runner, rngs, upto=None, draws="device", dev=None, step=0,
                             trajectories=True):
    """marginal_mh_steps with the theta-level blocks on the device: one propose
    launch, one batched filter over the chains inside the prior support, one
    accept launch.  `dev` carries the chain state between calls (built from
    `chains` when None).  Returns (outs, dev) with outs as marginal_mh_steps."""
    if not chains:
        return [], dev
    dev = dev or DeviceThetaChains(ir, chains, device=runner.device_opts.get("device"))
    th, x0, lq_f, lq_r, lp = dev.propose(rngs, step, draws)
    todo = [k for k in range(len(chains)) if lp[k] != -np.inf]
    res = runner.run_batch([th[k] for k in todo], [x0[k] if x0 is not None else None for k in todo],
                           [rngs[k].child(_FILTER_KEY) for k in todo], upto=upto, trajectories=False)
    ll_new = np.full(len(chains), -np.inf)
    by_k = dict(zip(todo, res))
    for k, (ll, _, _) in by_k.items():
        ll_new[k] = ll
    ok = dev.accept(ll_new, step)
    # trajectories for the accepted proposals only (per-stream draws: the others are unaffected)
    acc_k = [k for k in range(len(chains)) if ok[k]]
    trajs = {}
    if trajectories and acc_k:
        trajs = dict(zip(acc_k, runner.trajectories([by_k[k][2] for k in acc_k],
                                                    [rngs[k].child(_FILTER_KEY).child(2) for k in acc_k])))
    outs = []
    for k, chain in enumerate(chains):
        if ok[k]:
            ll, _, run = by_k[k]
            outs.append((MhChainState(theta=th[k].copy(), trajectory=trajs.get(k), loglik=ll, log_prior=float(lp[k]),
                                      init_state=None if x0 is None else x0[k].copy()), True, run))
        else:
            outs.append((chain, False, None))
    return outs, dev

"""CPU oracle for the bootstrap-particle-filter hot path (TEST INFRASTRUCTURE).

This module is a plain-numpy restatement of the reference `ssmkit` algorithm
for the two models the B200 kernels implement (Lorenz '96 and the
three-element windkessel).  It is the *checker*: only `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of
`bench.py` may import it.  The product path (`paper_1306_3277_b200`) never
imports, links or executes anything in here.

Parity pinning: every function below is checked against golden vectors that
were produced by running the reference itself (`tests/golden/make_golden.py`,
which imports `/root/reference/pkg/src` in a subprocess) -- see
`tests/test_oracle_golden.py`.

Reference anchors (all paths under /root/reference/pkg/src/ssmkit):
  substep_schedule ............ core/simulate.py:28-38
  RK4 integrator .............. core/simulate.py:71-93
  Wiener / sample statements .. core/simulate.py:50-60
  step_transition ............. core/simulate.py:132-163
  observe_logpdf .............. core/simulate.py:166-193 + distributions.py:94-101
  resample .................... inference/resampling.py:15-36
  ParticleRun / particle_filter inference/particle.py:28-185
  RngStream ................... core/rng.py:16-57
  logsumexp ................... scipy.special.logsumexp (scipy 1.18.1 form:
                                max elements split out, log1p of the rest)
"""

from __future__ import annotations

import math

import numpy as np

LOG_SQRT_2PI = 0.5 * np.log(2.0 * np.pi)  # distributions.py:15

# Lorenz96.bi:7 (const h = 0.05), :21 (x ~ U(-1,3)), :32 (obs sd 0.5)
L96_H = 0.05
L96_NX = 8
L96_OBS_SD = 0.5
# Windkessel.bi:5 (const h = 0.01), :24 (Pp ~ N(90,15)), :33 (obs sd 2)
WK_H = 0.01
WK_OBS_SD = 2.0


class OracleError(Exception):
    """Raised where the reference raises NonFinite/Degenerate errors."""

    def __init__(self, kind, time):
        self.kind = kind
        self.time = time
        super().__init__(f"{kind} at t={time:g}")


# --------------------------------------------------------------------------
# randomness (core/rng.py:16-57): numpy Philox keyed by SeedSequence
# --------------------------------------------------------------------------


class Stream:
    """Same (seed, key path) -> numpy Philox contract as rng.py:16-34."""

    def __init__(self, seed, key=()):
        self.seed = int(seed)
        self.key = tuple(int(k) for k in key)
        self._g = None

    @property
    def gen(self):
        if self._g is None:
            ss = np.random.SeedSequence(entropy=self.seed, spawn_key=self.key)
            self._g = np.random.Generator(np.random.Philox(ss))
        return self._g

    def child(self, *key):
        return Stream(self.seed, self.key + tuple(key))

    def uniform(self, low=0.0, high=1.0, size=None):
        return self.gen.uniform(low, high, size)

    def normal(self, loc=0.0, scale=1.0, size=None):
        return self.gen.normal(loc, scale, size)


# --------------------------------------------------------------------------
# time stepping helpers
# --------------------------------------------------------------------------


def substep_schedule(t, dt, delta):
    """simulate.py:28-38: ceil(dt/delta - 1e-9) sub-steps, the last shortened."""
    if delta is None:
        return [(t, dt)]
    n = max(1, int(np.ceil(dt / delta - 1e-9)))
    t_end = t + dt
    out = []
    for k in range(n):
        start = t + k * delta
        out.append((start, min(delta, t_end - start)))
    return out


def rk4_lengths(duration, h):
    """simulate.py:85-87: RK4 step lengths s_k = min(h, duration - k*h)."""
    n = max(1, int(np.ceil(duration / h - 1e-9)))
    return [min(h, duration - k * h) for k in range(n)]


# --------------------------------------------------------------------------
# Lorenz '96 (Lorenz96.bi:24-33)
# --------------------------------------------------------------------------


def l96_deriv(x, F, noise_term):
    """Slot n: ((((x[n-1]*(x[n+1]-x[n-2])) - x[n]) + F) + noise_term[n]),
    the exact association of the compiled lambda (ir.py:188-214)."""
    out = np.empty_like(x)
    for n in range(L96_NX):
        xm1 = x[:, (n - 1) % L96_NX]
        xp1 = x[:, (n + 1) % L96_NX]
        xm2 = x[:, (n - 2) % L96_NX]
        out[:, n] = (((xm1 * (xp1 - xm2)) - x[:, n]) + F) + noise_term[:, n]
    return out


def l96_transition(theta, x, t, dt, wiener):
    """One grid step of the L96 SDE (simulate.py:132-163 with the RK4 ODE
    op of simulate.py:71-93).  `wiener(k, d)` returns the (P, 8) Wiener
    increments W for sub-step k of length d (slot-major draws, sd sqrt(d)).
    Returns (x_new, t_fail) with t_fail the first sub-step end time at which
    the state is non-finite (None if all finite)."""
    F, sigma2 = float(theta[0]), float(theta[1])
    X = np.array(x, dtype=float, copy=True)
    t_fail = None
    for k, (t_k, d) in enumerate(substep_schedule(t, dt, L96_H)):
        W = wiener(k, d)
        noise_term = (np.sqrt(sigma2) * W) / L96_H  # ((sqrt(T1) * W) / 0.05)
        for s in rk4_lengths(d, L96_H):
            y0 = X.copy()
            k1 = l96_deriv(y0, F, noise_term)
            k2 = l96_deriv(y0 + 0.5 * s * k1, F, noise_term)
            k3 = l96_deriv(y0 + 0.5 * s * k2, F, noise_term)
            k4 = l96_deriv(y0 + s * k3, F, noise_term)
            X = y0 + (s / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
        if t_fail is None and not np.all(np.isfinite(X)):
            t_fail = t_k + d
    return X, t_fail


def l96_obs_logpdf(x, y, mask):
    """observe_logpdf (simulate.py:166-193): sum over present slots in slot
    order of the Gaussian logpdf (distributions.py:98-101), mean x_n, sd 0.5."""
    total = np.zeros(x.shape[0])
    log_sd = np.log(L96_OBS_SD)
    for n in range(L96_NX):
        if not mask[n]:
            continue
        z = (y[n] - x[:, n]) / L96_OBS_SD
        total = total + (-0.5 * z * z - log_sd - LOG_SQRT_2PI)
    return total


# --------------------------------------------------------------------------
# windkessel (Windkessel.bi:27-34)
# --------------------------------------------------------------------------


def wk_coeffs(theta):
    """exp(-h/(R*C)) and R*(1-exp(-h/(R*C))) exactly as the compiled lambda
    evaluates them: ((-0.01) / (R * C)) then np.exp."""
    R, C = float(theta[0]), float(theta[1])
    a = np.exp(np.array([(-WK_H) / (R * C)]))[0]
    b = R * (1.0 - a)
    return a, b


def wk_transition(theta, x, t, dt, xi_draw, input_at):
    """Pp <- a*Pp + b*(F + xi) per sub-step, xi ~ N(0, h*sqrt(sigma2))
    (simulate.py:63-68 + Windkessel.bi:28-29).  `xi_draw(k, sd)` returns
    the (P,) noise for sub-step k; `input_at(t)` the input F at time t."""
    a, b = wk_coeffs(theta)
    X = np.array(x, dtype=float, copy=True)
    t_fail = None
    for k, (t_k, d) in enumerate(substep_schedule(t, dt, WK_H)):
        F = float(input_at(t_k))
        sd = WK_H * np.sqrt(np.array([float(theta[3])]))[0]
        xi = xi_draw(k, sd)
        X = (a * X) + (b * (F + xi[:, None] if xi.ndim == 1 else F + xi))
        if t_fail is None and not np.all(np.isfinite(X)):
            t_fail = t_k + d
    return X, t_fail


def wk_obs_logpdf(theta, x, F_obs, y, mask):
    """Pa ~ gaussian(Pp + Z*F, 2.0) (Windkessel.bi:33)."""
    total = np.zeros(x.shape[0])
    if not mask[0]:
        return total
    mean = x[:, 0] + float(theta[2]) * float(F_obs)
    z = (y[0] - mean) / WK_OBS_SD
    return total + (-0.5 * z * z - np.log(WK_OBS_SD) - LOG_SQRT_2PI)


# --------------------------------------------------------------------------
# reductions and resampling
# --------------------------------------------------------------------------


def logsumexp(a):
    """scipy 1.18.1 logsumexp for a 1-D real array: the maximal elements are
    split out of the sum (count m), result log1p(s/m) + log(m) + a_max."""
    a = np.asarray(a, dtype=float)
    a_max = np.max(a)
    is_max = a == a_max
    m = float(np.sum(is_max))
    rest = np.where(is_max, -np.inf, a)
    with np.errstate(invalid="ignore"):
        s = float(np.sum(np.exp(rest - a_max)))
    if s != 0:
        s = s / m
    if m == 0:  # all-NaN input
        return float("nan")
    return float(np.log1p(s) + np.log(m) + a_max)


def ess(logw):
    """ParticleRun.ess (particle.py:83-85)."""
    w = np.exp(logw - logsumexp(logw))
    return 1.0 / float(np.sum(w * w))


def cumulative(weights):
    """resampling.py:22-27: cum = cumsum(w / sum(w)), cum[-1] = 1."""
    w = np.asarray(weights, dtype=float)
    cum = np.cumsum(w / w.sum())
    cum[-1] = 1.0
    return cum


def queries(scheme, u, P):
    """resampling.py:28-33: the query points for each scheme given the raw
    uniforms `u` (P draws for multinomial/stratified, 1 for systematic)."""
    if scheme == "multinomial":
        return np.asarray(u, dtype=float)
    if scheme == "stratified":
        return (np.arange(P) + np.asarray(u, dtype=float)) / P
    if scheme == "systematic":
        return (np.arange(P) + float(np.asarray(u).reshape(-1)[0])) / P
    raise ValueError(scheme)


def search(cum, q):
    """resampling.py:36: searchsorted(cum, q, 'right') clipped to [0, P-1]."""
    return np.searchsorted(cum, q, side="right").clip(0, len(cum) - 1)


def resample_with(weights, scheme, u, size=None):
    w = np.asarray(weights, dtype=float)
    P = w.size if size is None else int(size)
    return search(cumulative(w), queries(scheme, u, P))


def draw_uniforms(scheme, rng, P):
    """The draws `resample` consumes (resampling.py:28-33)."""
    if scheme == "systematic":
        return np.array([rng.uniform()])
    return rng.uniform(size=P)


# --------------------------------------------------------------------------
# the particle filter (particle.py:28-185)
# --------------------------------------------------------------------------


class Grid:
    """Minimal FilterGrid (timegrid.py:31-49): times plus per-step obs."""

    def __init__(self, times, obs):
        self.times = np.asarray(times, dtype=float)
        self.obs = obs  # dict: grid index -> (y, mask)

    @property
    def last(self):
        return len(self.times) - 1


class OracleFilter:
    """Bootstrap PF following ParticleRun (particle.py:28-153) for the two
    hand-written models.  `model` is "lorenz96" or "windkessel"; `inputs`
    is a callable t -> F for the windkessel."""

    def __init__(self, model, theta, grid, n_particles, resampler="multinomial",
                 ess_rel=None, initial_state=None, inputs=None, check_finite=True):
        if n_particles < 2:
            raise ValueError("particle filter needs n_particles >= 2")
        self.model = model
        self.theta = np.asarray(theta, dtype=float)
        self.grid = grid
        self.P = int(n_particles)
        self.resampler = resampler
        self.ess_rel = ess_rel
        self.initial_state = initial_state
        self.inputs = inputs
        self.check_finite = check_finite
        self.loglik = 0.0
        self.pos = 0
        self.nx = L96_NX if model == "lorenz96" else 1

    # particle.py:61-71 ; simulate.py:111-129 (slot-major draws)
    def init(self, rng):
        P = self.P
        if self.initial_state is not None:
            self.x = np.tile(np.asarray(self.initial_state, dtype=float), (P, 1))
        elif self.model == "lorenz96":
            self.x = np.zeros((P, L96_NX))
            for n in range(L96_NX):
                self.x[:, n] = rng.uniform(-1.0, 3.0, size=P)
        else:
            self.x = np.zeros((P, 1))
            self.x[:, 0] = rng.normal(90.0, 15.0, size=P)
        self.logw = np.full(P, -np.log(P))
        self.uniform = True
        self.history = [(self.x, None)]
        return self

    def advance_to(self, upto, rng):
        start = self.loglik
        for i in range(self.pos + 1, upto + 1):
            self.step(i, rng.child(i))
        self.pos = max(self.pos, upto)
        return self.loglik - start

    def _maybe_resample(self, rng):
        P = self.P
        if self.uniform:
            return np.arange(P)
        if self.ess_rel is not None and ess(self.logw) >= self.ess_rel * P:
            return np.arange(P)
        w = np.exp(self.logw)
        anc = resample_with(w, self.resampler, draw_uniforms(self.resampler, rng, P))
        self.x = self.x[anc]
        self.logw = np.full(P, -np.log(P))
        self.uniform = True
        return anc

    def transition(self, x, t, dt, rng):
        P = self.P
        if self.model == "lorenz96":
            def wiener(k, d):
                sd = math.sqrt(d)
                W = np.zeros((P, L96_NX))
                for n in range(L96_NX):
                    W[:, n] = rng.normal(0.0, sd, size=P)
                return W
            return l96_transition(self.theta, x, t, dt, wiener)

        def xi_draw(k, sd):
            return rng.normal(0.0, np.array([sd]), size=P)
        return wk_transition(self.theta, x, t, dt, xi_draw, self.inputs)

    def obs_logpdf(self, x, t, y, mask):
        if self.model == "lorenz96":
            return l96_obs_logpdf(x, y, mask)
        return wk_obs_logpdf(self.theta, x, self.inputs(t), y, mask)

    def step(self, i, rng_i):
        anc = self._maybe_resample(rng_i.child(0))
        t0, t1 = self.grid.times[i - 1], self.grid.times[i]
        self.x, t_fail = self.transition(self.x, t0, t1 - t0, rng_i.child(1))
        if self.check_finite and t_fail is not None:
            raise OracleError("nonfinite", t_fail)
        obs = self.grid.obs.get(i)
        if obs is not None and np.any(obs[1]):
            g = self.obs_logpdf(self.x, t1, obs[0], obs[1])
            a = self.logw + g
            incr = logsumexp(a)
            if not np.isfinite(incr):
                raise OracleError("degenerate", t1)
            self.loglik += incr
            self.logw = a - incr
            self.uniform = False
        self.history.append((self.x, anc))

    # particle.py:137-149
    def sample_trajectory(self, rng):
        j = int(resample_with(np.exp(self.logw), "multinomial", rng.uniform(size=1), size=1)[0])
        out = np.empty((self.pos + 1, self.nx))
        for i in range(self.pos, 0, -1):
            xs, anc = self.history[i]
            out[i] = xs[j]
            j = int(anc[j])
        out[0] = self.history[0][0][j]
        return out


def particle_filter(model, theta, grid, rng, n_particles=1024, resampler="multinomial",
                    ess_rel=None, initial_state=None, inputs=None, check_finite=True, upto=None):
    """particle.py:156-185: init(child 0) -> advance(child 1) -> trajectory(child 2)."""
    f = OracleFilter(model, theta, grid, n_particles, resampler, ess_rel, initial_state,
                     inputs, check_finite)
    f.init(rng.child(0))
    f.advance_to(grid.last if upto is None else upto, rng.child(1))
    traj = f.sample_trajectory(rng.child(2))
    return f.loglik, traj, f


# --------------------------------------------------------------------------
# synthetic data (runner.py:47-80 recipe)
# --------------------------------------------------------------------------


def windkessel_flow(t, f_max=500.0, t_s=0.3, t_d=0.5):
    """Eq. (5) of the paper: F(t) = Fmax sin^2(pi t'/Ts)
    for t' = mod(t, Ts+Td) < Ts, else 0."""
    tp = np.mod(t, t_s + t_d)
    return np.where(tp < t_s, f_max * np.sin(np.pi * tp / t_s) ** 2, 0.0)


def simulate_l96(theta, times, rng, obs_slots=range(8), obs_every=1):
    """Forward-simulate L96 states and observations on `times`
    (runner.py:47-80: x0 from child(1), transitions child(2,k), obs child(3,k))."""
    P = 1
    x = np.zeros((P, L96_NX))
    r1 = rng.child(1)
    for n in range(L96_NX):
        x[:, n] = r1.uniform(-1.0, 3.0, size=P)
    obs = {}
    for k in range(1, len(times)):
        rk = rng.child(2, k)

        def wiener(kk, d, rk=rk):
            W = np.zeros((P, L96_NX))
            for n in range(L96_NX):
                W[:, n] = rk.normal(0.0, math.sqrt(d), size=P)
            return W
        x, _ = l96_transition(theta, x, times[k - 1], times[k] - times[k - 1], wiener)
        ro = rng.child(3, k)
        y = np.array([ro.normal(x[0, n], L96_OBS_SD) for n in range(L96_NX)])
        mask = np.zeros(L96_NX, dtype=bool)
        if k % obs_every == 0:
            mask[list(obs_slots)] = True
        obs[k] = (y, mask)
    return obs

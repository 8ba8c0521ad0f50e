"""Linear-Gaussian structure of a model, for the device Kalman filter
(the reference's lineargauss.py:292-316).

The model's lowered blocks (codegen.lower) are executed symbolically with
every quantity an affine form  c + ax . x + sum_j az_j z_j  over the state
slots x and the standard-normal draws z behind the Gaussian / Wiener samples,
exactly as the reference's _Extractor does (lineargauss.py:29-260): any step
that leaves the affine family (a product of two state-dependent terms, a
function of a state-dependent argument, a state-dependent divisor or sd, a
non-Gaussian sample) raises NonlinearModelError.  Sub-stepping, RK4 and input
look-up follow simulate.step_transition.  Unlike the reference, the forms are
vectorised over a batch of parameter vectors (every coefficient is a (B,)
array), so one symbolic pass builds the systems of all theta-particles or
chains of a batched filter.  One deliberate difference: a transition `sample`
of a state slot writes that state (as the simulator does), where the
reference's extractor files it under noise.

Result convention (not the reference's transposed F / square-root factors):
  x_s = A_s x_{s-1} + b_s + N(0, Q_s),   y_s = H_s x_s + c_s + N(0, diag(r_sd_s^2)),
  x_0 ~ N(mu0, P0).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import NonlinearModelError


class _Aff:
    __slots__ = ("c", "ax", "az")

    def __init__(self, c, ax, az=None):
        self.c = c  # (B,)
        self.ax = ax  # (B, nx)
        self.az = {} if az is None else az  # j -> (B,)

    def is_const(self):
        return not self.az and not np.any(self.ax)

    def copy(self):
        return _Aff(self.c.copy(), self.ax.copy(), {k: v.copy() for k, v in self.az.items()})


class _Walker:
    def __init__(self, desc, thetas, inputs):
        self.desc = desc
        self.T = np.atleast_2d(np.asarray(thetas, dtype=float))
        self.B = self.T.shape[0]
        c = desc["counts"]
        self.nx, self.n_noise, self.n_input = c["state"], c["noise"], c["input"]
        self.inputs = inputs
        self.U = np.zeros(max(self.n_input, 1))
        self.n_z = 0

    # affine arithmetic (lineargauss.py:54-90)
    def const(self, v):
        return _Aff(np.broadcast_to(np.asarray(v, dtype=float), (self.B,)).copy(), np.zeros((self.B, self.nx)))

    def unit(self, k):
        a = self.const(0.0)
        a.ax[:, k] = 1.0
        return a

    def fresh_z(self, coef):
        a = self.const(0.0)
        a.az[self.n_z] = np.broadcast_to(np.asarray(coef, dtype=float), (self.B,)).copy()
        self.n_z += 1
        return a

    def add(self, a, b):
        out = a.copy()
        out.c = out.c + b.c
        out.ax = out.ax + b.ax
        for k, v in b.az.items():
            out.az[k] = out.az[k] + v if k in out.az else v.copy()
        return out

    def scale(self, a, s):
        s = np.asarray(s, dtype=float)
        return _Aff(a.c * s, a.ax * s[..., None] if s.ndim else a.ax * s, {k: v * s for k, v in a.az.items()})

    def mul(self, a, b, where):
        if a.is_const():
            return self.scale(b, a.c)
        if b.is_const():
            return self.scale(a, b.c)
        raise NonlinearModelError(f"product of state-dependent terms in {where}")

    def div(self, a, b, where):
        if not b.is_const():
            raise NonlinearModelError(f"state-dependent divisor in {where}")
        return self.scale(a, 1.0 / b.c)

    def eval(self, e, state, noise, where):
        t = e[0]
        if t == "num":
            return self.const(e[1])
        if t == "T":
            return self.const(self.T[:, e[1]])
        if t == "U":
            return self.const(self.U[..., e[1]])  # (width,) or per row (rows, width)
        if t == "X":
            return state[e[1]].copy()
        if t == "W":
            if noise is None:
                raise NonlinearModelError(f"noise read in {where}")
            return noise[e[1]].copy()
        if t == "neg":
            return self.scale(self.eval(e[1], state, noise, where), -1.0)
        if t == "bin":
            a = self.eval(e[2], state, noise, where)
            b = self.eval(e[3], state, noise, where)
            op = e[1]
            if op == "+":
                return self.add(a, b)
            if op == "-":
                return self.add(a, self.scale(b, -1.0))
            if op == "*":
                return self.mul(a, b, where)
            return self.div(a, b, where)
        if t == "call":
            args = [self.eval(a, state, noise, where) for a in e[2]]
            if any(not a.is_const() for a in args):
                raise NonlinearModelError(f"nonlinear function {e[1]} of a state-dependent argument in {where}")
            v = [a.c for a in args]
            if e[1] == "mod":
                return self.const(v[0] - v[1] * np.floor(v[0] / v[1]))  # lineargauss.py:117-118
            fn = {"exp": np.exp, "sqrt": np.sqrt, "sin": np.sin, "pow": np.power}[e[1]]
            return self.const(fn(*v))
        raise ValueError(e)

    def sample(self, op, i, state, noise, where, wiener_sd=None):
        """mean + sd * fresh z of one sampled slot (lineargauss.py:132-146)."""
        if op["kind"] == "wiener":
            return self.fresh_z(wiener_sd)
        if op["kind"] != "gaussian":
            raise NonlinearModelError(f"non-Gaussian sample in {where}")
        mean = self.eval(op["args"][i][0], state, noise, where)
        sd = self.eval(op["args"][i][1], state, noise, where)
        if not sd.is_const():
            raise NonlinearModelError(f"state-dependent sd in {where}")
        return self.add(mean, self.fresh_z(sd.c))

    def initial(self):
        state = [self.const(0.0) for _ in range(self.nx)]
        for op in self.desc["initial"]:
            if op["op"] == "sample":
                for i, slot in enumerate(op["slots"]):
                    state[slot] = self.sample(op, i, state, None, "initial")
            elif op["op"] == "assign":
                vals = [self.eval(e, state, None, "initial") for e in op["exprs"]]
                for slot, v in zip(op["slots"], vals):
                    state[slot] = v
            else:
                raise NonlinearModelError("ode in initial block")
        return state

    def interval(self, t, dt, state):
        """Affine state over (t, t+dt] (lineargauss.py:171-193)."""
        from .inference.particle import substep_schedule
        from .simulate import _input_row

        noise = [self.const(0.0) for _ in range(self.n_noise)]
        delta = self.desc["delta"]
        for t_k, d in substep_schedule(t, dt, delta):
            self.U = _input_row(self.inputs, t_k, self.n_input, max(self.n_input, 1))
            for op in self.desc["transition"]:
                if op["op"] == "sample":
                    vals = [self.sample(op, i, state, noise, "transition", wiener_sd=math.sqrt(d))
                            for i in range(len(op["slots"]))]
                    dst = state if op["role"] == "state" else noise
                    for slot, v in zip(op["slots"], vals):
                        dst[slot] = v
                elif op["op"] == "assign":
                    vals = [self.eval(e, state, noise, "transition") for e in op["exprs"]]
                    dst = noise if op["role"] == "noise" else state
                    for slot, v in zip(op["slots"], vals):
                        dst[slot] = v
                else:
                    self.rk4(op, state, noise, d)
        return state

    def interval_rows(self, sched, u_rows, state):
        """interval() for rows that share one sub-step schedule `sched` (durations
        d_k) but have their own inputs u_rows[k] (rows, width) at sub-step k: the
        batch is (theta x grid step), so one symbolic pass serves many steps."""
        noise = [self.const(0.0) for _ in range(self.n_noise)]
        for k, d in enumerate(sched):
            self.U = u_rows[k]
            for op in self.desc["transition"]:
                if op["op"] == "sample":
                    vals = [self.sample(op, i, state, noise, "transition", wiener_sd=math.sqrt(d))
                            for i in range(len(op["slots"]))]
                    dst = state if op["role"] == "state" else noise
                    for slot, v in zip(op["slots"], vals):
                        dst[slot] = v
                elif op["op"] == "assign":
                    vals = [self.eval(e, state, noise, "transition") for e in op["exprs"]]
                    dst = noise if op["role"] == "noise" else state
                    for slot, v in zip(op["slots"], vals):
                        dst[slot] = v
                else:
                    self.rk4(op, state, noise, d)
        return state

    def rk4(self, op, state, noise, duration):
        """simulate.py:71-93 on affine forms (lineargauss.py:195-221)."""
        slots = op["slots"]

        def deriv(stage):
            full = list(state)
            for slot, v in zip(slots, stage):
                full[slot] = v
            return [self.eval(e, full, noise, "transition") for e in op["exprs"]]

        h = op["h"]
        n_steps = max(1, int(np.ceil(duration / h - 1e-9)))
        for k in range(n_steps):
            s = min(h, duration - k * h)
            y0 = [state[slot].copy() for slot in slots]
            k1 = deriv(y0)
            k2 = deriv([self.add(y, self.scale(q, 0.5 * s)) for y, q in zip(y0, k1)])
            k3 = deriv([self.add(y, self.scale(q, 0.5 * s)) for y, q in zip(y0, k2)])
            k4 = deriv([self.add(y, self.scale(q, s)) for y, q in zip(y0, k3)])
            for i, slot in enumerate(slots):
                incr = self.add(self.add(k1[i], self.scale(k2[i], 2.0)), self.add(self.scale(k3[i], 2.0), k4[i]))
                state[slot] = self.add(y0[i], self.scale(incr, s / 6.0))

    def observation(self, t, u_rows=None):
        """(H, c, r_sd) over all obs slots at time t (lineargauss.py:223-260);
        u_rows: per-row inputs (rows of a theta x step batch) instead of t's."""
        from .simulate import _input_row

        self.U = _input_row(self.inputs, t, self.n_input, max(self.n_input, 1)) if u_rows is None else u_rows
        ny = self.desc["counts"]["obs"]
        H = np.zeros((self.B, ny, self.nx))
        c = np.zeros((self.B, ny))
        r = np.zeros((self.B, ny))
        state = [self.unit(k) for k in range(self.nx)]
        for op in self.desc["observation"]:
            if op["kind"] != "gaussian":
                raise NonlinearModelError("non-Gaussian observation")
            for i, slot in enumerate(op["slots"]):
                mean = self.eval(op["args"][i][0], state, None, "observation")
                sd = self.eval(op["args"][i][1], state, None, "observation")
                if not sd.is_const():
                    raise NonlinearModelError("state-dependent sd in observation")
                H[:, slot, :] = mean.ax
                c[:, slot] = mean.c
                r[:, slot] = sd.c
        return H, c, r


def _to_gaussian(state, n_z, B):
    nx = len(state)
    mu = np.stack([a.c for a in state], axis=1)  # (B, nx)
    A = np.stack([a.ax for a in state], axis=1)  # (B, nx, nx): row k = coefficients of x_k
    L = np.zeros((B, nx, n_z))
    for k, a in enumerate(state):
        for j, v in a.az.items():
            L[:, k, j] = v
    return mu, A, L


@dataclass
class LinearGaussianSystems:
    """B systems along one time grid (steps 1..S)."""

    times: np.ndarray
    mu0: np.ndarray  # (B, nx)
    P0: np.ndarray  # (B, nx, nx)
    A: np.ndarray  # (B, S, nx, nx)
    b: np.ndarray  # (B, S, nx)
    Q: np.ndarray  # (B, S, nx, nx)
    H: np.ndarray  # (B, S, ny, nx)
    c: np.ndarray  # (B, S, ny)
    r_sd: np.ndarray  # (B, S, ny)

    @property
    def B(self):
        return self.mu0.shape[0]

    def row(self, k):
        return LinearGaussianSystems(self.times, *(getattr(self, f)[k : k + 1] for f in
                                                   ("mu0", "P0", "A", "b", "Q", "H", "c", "r_sd")))


def description_of(ir):
    """The lowered description of a model (hand-written specs carry theirs)."""
    from . import codegen
    from .generic import GenericModel
    from .models import ModelSpec

    if isinstance(ir, GenericModel):
        return ir.desc
    if isinstance(ir, ModelSpec):
        return _builtin_description(ir)
    if isinstance(ir, dict):
        return ir
    return codegen.lower(ir)


def _builtin_description(spec):
    """Windkessel.bi / Lorenz96.bi as lowered descriptions (the statements the
    hand-written kernels implement)."""
    num = lambda v: ["num", v]  # noqa: E731
    T = lambda k: ["T", k]  # noqa: E731
    X = lambda k: ["X", k]  # noqa: E731
    bn = lambda op, a, b: ["bin", op, a, b]  # noqa: E731
    if spec.name == "Windkessel":
        a = ["call", "exp", [bn("/", ["neg", num(0.01)], bn("*", T(0), T(1)))]]
        return {
            "name": "Windkessel", "counts": spec.counts, "delta": spec.delta,
            "initial": [{"op": "sample", "role": "state", "kind": "gaussian", "slots": [0],
                         "args": [[num(90.0), num(15.0)]]}],
            "transition": [
                {"op": "sample", "role": "noise", "kind": "gaussian", "slots": [0],
                 "args": [[num(0.0), bn("*", num(0.01), ["call", "sqrt", [T(3)]])]]},
                {"op": "assign", "role": "state", "slots": [0],
                 "exprs": [bn("+", bn("*", a, X(0)),
                              bn("*", bn("*", T(0), bn("-", num(1.0), a)), bn("+", ["U", 0], ["W", 0])))]},
            ],
            "observation": [{"op": "sample", "role": "obs", "kind": "gaussian", "slots": [0],
                             "args": [[bn("+", X(0), bn("*", T(2), ["U", 0])), num(2.0)]]}],
        }
    raise NonlinearModelError(f"{spec.name} is not linear-Gaussian")


def extract_linear_gaussian(ir, thetas, times, inputs=None) -> LinearGaussianSystems:
    """The linear-Gaussian systems of `ir` at each row of `thetas` along `times`
    (lineargauss.py:292-316); raises NonlinearModelError otherwise."""
    desc = description_of(ir)
    times = np.asarray(times, dtype=float)
    w = _Walker(desc, thetas, inputs)
    B, nx = w.B, w.nx
    st0 = w.initial()
    mu0, A0, L0 = _to_gaussian(st0, w.n_z, B)
    if np.any(A0):
        raise NonlinearModelError("initial state mean must not depend on the state")
    P0 = L0 @ L0.transpose(0, 2, 1)
    S = len(times) - 1
    ny = desc["counts"]["obs"]
    out = dict(A=np.zeros((B, S, nx, nx)), b=np.zeros((B, S, nx)), Q=np.zeros((B, S, nx, nx)),
               H=np.zeros((B, S, ny, nx)), c=np.zeros((B, S, ny)), r_sd=np.zeros((B, S, ny)))
    # grid steps that share a sub-step schedule (the same durations; inputs may differ)
    # are evaluated together: one symbolic pass over a (theta x step) batch per schedule
    from .inference.particle import substep_schedule
    from .simulate import _input_row

    width = max(w.n_input, 1)
    groups = {}
    for i in range(1, S + 1):
        sched = substep_schedule(times[i - 1], times[i] - times[i - 1], desc["delta"])
        groups.setdefault(tuple(d for _, d in sched), []).append((i, [t_k for t_k, _ in sched]))
    thetas2 = np.atleast_2d(np.asarray(thetas, dtype=float))
    per = max(1, 65536 // B)  # steps per pass: ~64K rows keep the numpy temporaries cache-sized
    chunks = [(ds, members[k : k + per]) for ds, members in groups.items() for k in range(0, len(members), per)]
    for ds, members in chunks:
        steps = np.array([i for i, _ in members])
        n = len(steps)
        # rows theta-major: row = b * n + j (step steps[j]); inputs per step, repeated over theta
        wg = _Walker(desc, np.repeat(thetas2, n, axis=0), inputs)
        u_sub = [np.tile(np.stack([_input_row(inputs, tk[k], wg.n_input, width) for _, tk in members]), (B, 1))
                 for k in range(len(ds))]
        st = wg.interval_rows(ds, u_sub, [wg.unit(k) for k in range(nx)])
        b, A, L = _to_gaussian(st, wg.n_z, B * n)
        out["A"][:, steps - 1] = A.reshape(B, n, nx, nx)
        out["b"][:, steps - 1] = b.reshape(B, n, nx)
        Lr = L.reshape(B, n, nx, -1)
        out["Q"][:, steps - 1] = Lr @ Lr.transpose(0, 1, 3, 2)
        u_obs = np.tile(np.stack([_input_row(inputs, times[i], wg.n_input, width) for i in steps]), (B, 1))
        H, c, r = wg.observation(None, u_rows=u_obs)
        out["H"][:, steps - 1] = H.reshape(B, n, ny, nx)
        out["c"][:, steps - 1] = c.reshape(B, n, ny)
        out["r_sd"][:, steps - 1] = r.reshape(B, n, ny)
    return LinearGaussianSystems(times=times, mu0=mu0, P0=P0, **out)

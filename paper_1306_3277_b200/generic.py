"""`GenericModel`: the device path for any reference model that has no
hand-written kernel.

A reference `ModelIr` (or its lowered description, codegen.lower) becomes a
model spec with the interface the filter host code uses (`ModelSpec`'s slot
counts, `derived`, `host_initial`, `host_noise`), backed by an NVRTC-compiled
kernel set (csrc/ssm_gen.cu, one compile per model and device, cached).

Host-side draws follow the reference exactly, so `noise="host"` runs are
parity runs:
  * initial block (simulate.py:111-129): the reference's statements evaluated
    with numpy on the host, in its draw order;
  * transition noise (simulate.py:50-60): per sub-step, statement and slot,
    the standard variate numpy's normal / uniform consume (z with
    rng.normal(loc, scale) = loc + scale z; U with rng.uniform(lo, hi) =
    lo + (hi - lo) U), which the kernel maps exactly as numpy does.
    Gamma / inverse-gamma transition noise has no such form: device draws only.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib, codegen
from .errors import DistributionParameterError, UnsupportedModelError
from .models import (d_gamma_logpdf, d_gamma_sample, d_gauss_logpdf, d_invgamma_logpdf, d_invgamma_sample,
                     d_tgauss_logpdf, d_tgauss_sample, d_uniform_logpdf, d_uniform_sample)

_INJECTABLE = {"wiener": "normal", "gaussian": "normal", "uniform": "uniform", "truncated_gaussian": "uniform"}
_CACHE = {}
_LOCK = threading.Lock()


def _sample_host(kind, args, size, rng):
    """distributions.sample (distributions.py:73-91)."""
    if kind == "gaussian":
        if not np.all(np.asarray(args[1]) > 0):
            raise DistributionParameterError("gaussian sd must be > 0")
        return rng.normal(args[0], args[1], size=size)
    if kind == "uniform":
        return d_uniform_sample(rng, args[0], args[1], size)
    if kind == "truncated_gaussian":
        return d_tgauss_sample(rng, args[0], args[1], args[2], args[3], size)
    if kind == "gamma":
        if not (np.all(np.asarray(args[0]) > 0) and np.all(np.asarray(args[1]) > 0)):
            raise DistributionParameterError("gamma shape and scale must be > 0")
        return d_gamma_sample(rng, args[0], args[1], size)
    if kind == "inverse_gamma":
        return d_invgamma_sample(rng, args[0], args[1], size)
    raise UnsupportedModelError(f"cannot sample {kind} on the host")


def _check_params(kind, args):
    """distributions.py:53-69"""
    def req(ok, msg):
        if not np.all(ok):
            raise DistributionParameterError(msg)

    if kind in ("gaussian", "truncated_gaussian"):
        req(np.asarray(args[1]) > 0, f"{kind} sd must be > 0")
        if kind == "truncated_gaussian":
            req(np.asarray(args[2]) < np.asarray(args[3]), "truncated_gaussian needs lower < upper")
    elif kind in ("gamma", "inverse_gamma"):
        req(np.asarray(args[0]) > 0, f"{kind} shape must be > 0")
        req(np.asarray(args[1]) > 0, f"{kind} scale must be > 0")
    elif kind == "uniform":
        req(np.asarray(args[0]) < np.asarray(args[1]), "uniform needs lower < upper")


def _logpdf_host(kind, args, x):
    """distributions.logpdf (distributions.py:94-123)."""
    _check_params(kind, args)
    if kind == "gaussian":
        return d_gauss_logpdf(x, args[0], args[1])
    if kind == "truncated_gaussian":
        return d_tgauss_logpdf(x, *args)
    if kind == "gamma":
        return d_gamma_logpdf(x, args[0], args[1])
    if kind == "inverse_gamma":
        return d_invgamma_logpdf(x, args[0], args[1])
    if kind == "uniform":
        return d_uniform_logpdf(x, args[0], args[1])
    raise UnsupportedModelError(f"cannot evaluate {kind}")


class GenericModel:
    """Model spec for the NVRTC-compiled generic kernels (SSM_MODEL_GENERIC)."""

    kernel = _lib.SSM_MODEL_GENERIC
    h = 0.0  # RK4 steps are split in the kernel (the sub-step table's s[] is unused)
    obs_sd = 1.0  # unused: the observation density is generated code
    has_ode = False

    def __init__(self, desc: dict):
        self.desc = desc
        c = desc["counts"]
        self.name = desc["name"]
        self.n_param, self.n_state, self.n_noise = c["param"], c["state"], c["noise"]
        self.n_input, self.n_obs = c["input"], c["obs"]
        self.delta = desc["delta"]
        self.source = codegen.cuda_source(desc)
        self.digest = codegen.source_digest(self.source)
        self.draw_kinds = codegen.transition_draws(desc)
        self.theta_stride = max(self.n_param, 1)
        self._handles = {}
        self._fns = {}
        self.has_proposal_initial = desc.get("proposal_initial") is not None
        self.ode_h = [float(op["h"]) for op in desc["transition"] if op["op"] == "ode"]

    @property
    def nx(self):
        return self.n_state

    @property
    def counts(self):
        return dict(self.desc["counts"])

    def block(self, name):
        if name in ("initial", "transition", "observation"):
            return True
        return True if self.desc.get(name) is not None else None

    def __repr__(self):
        return f"GenericModel({self.name!r}, digest={self.digest})"

    # ---- device kernels ---------------------------------------------------
    def handle(self, device) -> int:
        """Compiled kernel set on `device` (NVRTC, once per process)."""
        import torch

        key = torch.device(device).index or 0
        h = self._handles.get(key)
        if h is None:
            with _LOCK:
                h = self._handles.get(key)
                if h is None:
                    with torch.cuda.device(key):
                        out = C.c_void_p()
                        log = C.create_string_buffer(1 << 16)
                        st = _lib.lib().ssm_gen_compile(self.source.encode(), codegen.include_dir().encode(),
                                                        C.byref(out), log, len(log))
                        if st != _lib.SSM_OK:
                            raise UnsupportedModelError(
                                f"{self.name}: NVRTC compile / load failed ({_lib.lib().ssm_status_string(st).decode()}: "
                                f"{_lib.lib().ssm_last_cuda_error().decode()}):\n"
                                f"{log.value.decode(errors='replace')[:4000]}")
                        h = out.value
                    self._handles[key] = h
        return h

    def check_compiles(self) -> str:
        """NVRTC compile only (no device needed); returns the log."""
        log = C.create_string_buffer(1 << 16)
        st = _lib.lib().ssm_gen_check(self.source.encode(), codegen.include_dir().encode(), log, len(log))
        if st != _lib.SSM_OK:
            raise UnsupportedModelError(f"{self.name}: NVRTC compile failed:\n{log.value.decode(errors='replace')}")
        return log.value.decode(errors="replace")

    # ---- per-filter constants ----------------------------------------------
    def derived(self, thetas) -> np.ndarray:
        """(B, theta_stride) float64: the parameters themselves."""
        th = np.atleast_2d(np.asarray(thetas, dtype=float))
        out = np.zeros((th.shape[0], self.theta_stride))
        out[:, : self.n_param] = th[:, : self.n_param]
        return out

    # ---- host draws (noise="host") -----------------------------------------
    def _block_fns(self, name):
        """Statements of a block with host (numpy) expression functions."""
        if name not in self._fns:
            ops = []
            for op in self.desc.get(name) or ():
                if op["op"] == "sample":
                    ops.append(("sample", op["kind"], op["slots"],
                                [[codegen.numpy_fn(a) for a in row] for row in op["args"]]))
                elif op["op"] == "assign":
                    ops.append(("assign", None, op["slots"], [codegen.numpy_fn(e) for e in op["exprs"]]))
            self._fns[name] = ops
        return self._fns[name]

    def host_initial(self, rng, P, theta=None):
        """simulate.sample_initial (simulate.py:111-129) for one filter: (P, nx)."""
        T = np.atleast_2d(np.asarray(theta if theta is not None else np.zeros(self.n_param), dtype=float))
        X = np.zeros((P, self.n_state))
        W = np.zeros((P, 0))
        U = np.zeros(self.n_input)
        for what, kind, slots, fns in self._block_fns("initial"):
            if what == "sample":
                args_all = [tuple(f(T, X, W, U) for f in row) for row in fns]
                for slot, args in zip(slots, args_all):
                    X[:, slot] = _sample_host(kind, args, P, rng)
            else:
                vals = [f(T, X, W, U) for f in fns]
                for slot, v in zip(slots, vals):
                    X[:, slot] = v
        return X

    def check_host_noise(self):
        bad = sorted({k for k in self.draw_kinds if k not in _INJECTABLE})
        if bad:
            raise UnsupportedModelError(f"{self.name}: noise='host' cannot inject {bad} draws (device noise only)")

    def host_noise(self, rng, subs, P, derived_row):
        """Standard variates of every transition draw in the reference's order
        (per sub-step, statement, slot): (n_sub, KDRAW, P)."""
        self.check_host_noise()
        K = max(len(self.draw_kinds), 1)
        out = np.zeros((len(subs), K, P))
        for k in range(len(subs)):
            for j, kind in enumerate(self.draw_kinds):
                if _INJECTABLE[kind] == "normal":
                    out[k, j] = rng.normal(0.0, 1.0, size=P)
                else:
                    out[k, j] = rng.uniform(0.0, 1.0, size=P)
        return out


    # ---- theta-level blocks on the host (simulate.py:96-108, 219-352) --------
    def sample_parameter(self, rng, size=1):
        T = np.zeros((size, self.n_param))
        X, W, U = np.zeros((size, 0)), np.zeros((size, 0)), np.zeros(self.n_input)
        for what, kind, slots, fns in self._block_fns("parameter"):
            if what != "sample":
                continue
            args_all = [tuple(f(T, X, W, U) for f in row) for row in fns]
            for slot, args in zip(slots, args_all):
                T[:, slot] = _sample_host(kind, args, size, rng)
        return T

    def sample_initial(self, thetas, rng, size=None):
        T = np.atleast_2d(np.asarray(thetas, dtype=float))
        return self.host_initial(rng, T.shape[0] if size is None else size, T)

    def parameter_logpdf(self, theta):
        theta = np.asarray(theta, dtype=float)
        T, X, W, U = theta[None, :], np.zeros((1, 0)), np.zeros((1, 0)), np.zeros(self.n_input)
        total = 0.0
        for what, kind, slots, fns in self._block_fns("parameter"):
            for slot, row in zip(slots, fns):
                args = tuple(f(T, X, W, U) for f in row)
                total += float(np.sum(_logpdf_host(kind, args, theta[slot])))
        return total

    def initial_logpdf(self, theta, x0):
        theta, x0 = np.asarray(theta, dtype=float), np.asarray(x0, dtype=float)
        T, X, W, U = theta[None, :], x0[None, :], np.zeros((1, 0)), np.zeros(self.n_input)
        total = 0.0
        for what, kind, slots, fns in self._block_fns("initial"):
            if what != "sample":
                continue
            for slot, row in zip(slots, fns):
                args = tuple(f(T, X, W, U) for f in row)
                total += float(np.sum(_logpdf_host(kind, args, x0[slot])))
        return total

    def _apply_initial_assigns(self, theta, x0):
        X = np.array(x0, dtype=float, copy=True)[None, :]
        T, W, U = np.atleast_2d(np.asarray(theta, dtype=float)), np.zeros((1, 0)), np.zeros(self.n_input)
        for what, _, slots, fns in self._block_fns("initial"):
            if what == "assign":
                vals = [f(T, X, W, U) for f in fns]
                for slot, v in zip(slots, vals):
                    X[:, slot] = v
        return X[0]

    def _walk(self, block, fallback, T, X, env, values_from, values_to, rng):
        """simulate._walk_proposal (simulate.py:264-299): sequential overwrite."""
        name = block if self.desc.get(block) is not None else fallback
        W, U = np.zeros((1, 0)), np.zeros(self.n_input)
        logq = 0.0
        out = np.array(values_from, dtype=float, copy=True)
        for what, kind, slots, fns in self._block_fns(name):
            if what != "sample":
                continue
            args_all = [tuple(f(T, X, W, U) for f in row) for row in fns]
            for slot, args in zip(slots, args_all):
                if values_to is None:
                    value = float(_sample_host(kind, args, 1, rng)[0])
                else:
                    value = float(values_to[slot])
                logq += float(np.sum(_logpdf_host(kind, args, value)))
                out[slot] = value
                env[0, slot] = value
        return out, logq

    def propose_parameters(self, theta, rng):
        theta = np.asarray(theta, dtype=float)
        T, X = theta[None, :].copy(), np.zeros((1, self.n_state))
        return self._walk("proposal_parameter", "parameter", T, X, T, theta, None, rng)

    def proposal_parameter_logpdf(self, theta_from, theta_to):
        theta_from = np.asarray(theta_from, dtype=float)
        T, X = theta_from[None, :].copy(), np.zeros((1, self.n_state))
        return self._walk("proposal_parameter", "parameter", T, X, T, theta_from, theta_to, None)[1]

    def propose_initial(self, theta, x0, rng):
        x0 = np.asarray(x0, dtype=float)
        T, X = np.atleast_2d(np.asarray(theta, dtype=float)).copy(), x0[None, :].copy()
        out, logq = self._walk("proposal_initial", "initial", T, X, X, x0, None, rng)
        return self._apply_initial_assigns(theta, out), logq

    def proposal_initial_logpdf(self, theta, x_from, x_to):
        x_from = np.asarray(x_from, dtype=float)
        T, X = np.atleast_2d(np.asarray(theta, dtype=float)).copy(), x_from[None, :].copy()
        return self._walk("proposal_initial", "initial", T, X, X, x_from, x_to, None)[1]

    def propose_batch(self, thetas, inits, rngs):
        """models.propose_batch for a generic model: the reference's marginal MH
        proposal (mcmc.py:140-147), chain by chain in its draw order."""
        C = len(rngs)
        new = np.zeros((C, self.n_param))
        x0s, lq_f, lq_r, lp = [None] * C, np.zeros(C), np.zeros(C), np.zeros(C)
        for c, rng in enumerate(rngs):
            th = np.asarray(thetas[c], dtype=float)
            th_new, f = self.propose_parameters(th, rng)
            r = self.proposal_parameter_logpdf(th_new, th)
            x_new = None
            if inits is not None and inits[c] is not None:
                x_new, lq = self.propose_initial(th_new, inits[c], rng)
                f += lq
                r += self.proposal_initial_logpdf(th, x_new, inits[c])
            p = self.parameter_logpdf(th_new)
            if x_new is not None:
                p += self.initial_logpdf(th_new, x_new)
            new[c], x0s[c], lq_f[c], lq_r[c], lp[c] = th_new, x_new, f, r, p
        return new, x0s, lq_f, lq_r, lp


def from_description(desc: dict) -> GenericModel:
    key = codegen.dumps(desc)
    with _LOCK:
        m = _CACHE.get(key)
        if m is None:
            m = GenericModel(desc)
            _CACHE[key] = m
    return m


def from_ir(ir) -> GenericModel:
    return from_description(codegen.lower(ir))

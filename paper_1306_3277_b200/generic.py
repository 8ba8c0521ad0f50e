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
from .models import d_gamma_sample, d_invgamma_sample, d_tgauss_sample, d_uniform_sample

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


class GenericModel:
    """Model spec for the NVRTC-compiled generic kernels (SSM_MODEL_GENERIC)."""

    kernel = _lib.SSM_MODEL_GENERIC
    h = 0.0  # RK4 steps are split in the kernel (the sub-step table's s[] is unused)
    obs_sd = 1.0  # unused: the observation density is generated code
    has_ode = False
    has_proposal_initial = False

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
        self._init_fns = None

    @property
    def nx(self):
        return self.n_state

    @property
    def counts(self):
        return dict(self.desc["counts"])

    def block(self, name):
        return True if name in ("initial", "transition", "observation") else None

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
    def _initial_fns(self):
        if self._init_fns is None:
            ops = []
            for op in self.desc["initial"]:
                if op["op"] == "sample":
                    ops.append(("sample", op["kind"], op["slots"],
                                [[codegen.numpy_fn(a) for a in row] for row in op["args"]]))
                else:
                    ops.append(("assign", None, op["slots"], [codegen.numpy_fn(e) for e in op["exprs"]]))
            self._init_fns = ops
        return self._init_fns

    def host_initial(self, rng, P, theta=None):
        """simulate.sample_initial (simulate.py:111-129) for one filter: (P, nx)."""
        T = np.atleast_2d(np.asarray(theta if theta is not None else np.zeros(self.n_param), dtype=float))
        X = np.zeros((P, self.n_state))
        W = np.zeros((P, 0))
        U = np.zeros(self.n_input)
        for what, kind, slots, fns in self._initial_fns():
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

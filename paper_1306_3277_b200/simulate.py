"""Model-block kernels behind the reference's simulate API
(core/simulate.py:132-193): one grid step of the transition and the
observation log-density, batched over particles, on the device.

These are thin single-step entry points over the same fused kernel the
filter uses (ssm_propagate_weight); the filter itself never calls them.
  step_transition(ir, theta, x, inputs, t, dt, rng, check_finite)
      rng: an RngStream -> the reference's own draws, in its order
           (slot-major normal(0, sqrt(d), P) per sub-step), injected;
      or noise=array (n_sub, n_noise, P) of noise-variable values.
  observe_logpdf(ir, theta, x, inputs, y, mask)
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import DistributionParameterError, NonFiniteStateError
from .inference.particle import _dtype_info, _fs_init, substep_schedule
from .models import LOG_SQRT_2PI, resolve_model


def _input_row(inputs, t, n_input, width):
    """Input values (a provider at t, or a value vector), zero-padded to width."""
    out = np.zeros(width)
    if inputs is not None and n_input:
        v = inputs.at(t) if hasattr(inputs, "at") else inputs
        out[:n_input] = np.asarray(v, dtype=float).reshape(-1)[:n_input]
    return out


def _subs(spec, t, dt, inputs):
    if dt <= 0:
        raise ValueError("step_transition requires dt > 0")
    subs = substep_schedule(t, dt, spec.delta)
    arr = np.zeros(len(subs), dtype=_lib.SUBSTEP_DTYPE)
    for k, (t_k, d) in enumerate(subs):
        arr[k]["d"] = d
        arr[k]["sd"] = np.sqrt(d)
        if spec.n_input:
            arr[k]["u_in"] = float(np.asarray(inputs.at(t_k) if hasattr(inputs, "at") else inputs).reshape(-1)[0])
        if spec.has_ode:
            n_ode = max(1, int(np.ceil(d / spec.h - 1e-9)))
            for m in range(n_ode):
                arr[k]["s"][m] = min(spec.h, d - m * spec.h)
            arr[k]["n_ode"] = n_ode
    return subs, arr


def _run_pw(spec, theta, x, arr, noise, obs, dtype, exact, check_finite, device, y_vec=None, u_vec=None):
    _lib.require_cuda()
    L = _lib.lib()
    _, tdt, dt_id = _dtype_info(dtype)
    X = np.atleast_2d(np.asarray(x, dtype=float))
    P = X.shape[0]
    dev = device or torch.device("cuda", torch.cuda.current_device())
    xin = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev, tdt)
    xout = torch.empty_like(xin)
    th = torch.from_numpy(spec.derived(np.asarray(theta, dtype=float).reshape(1, -1))).to(dev)
    subs_t = torch.from_numpy(arr.view(np.uint8).copy()).to(dev) if len(arr) else None
    noise_t = torch.from_numpy(np.ascontiguousarray(noise)).to(dev, tdt) if noise is not None else None
    fs = _fs_init(1, dev)
    ws = torch.empty(L.ssm_pw_workspace_bytes(1, P), dtype=torch.uint8, device=dev)
    a_out = torch.empty(P, dtype=tdt, device=dev) if obs is not None else None
    A = _lib.PwArgs()
    A.model, A.dtype, A.B, A.P = spec.kernel, dt_id, 1, P
    A.step, A.n_sub = 1, len(arr)
    A.exact, A.check_finite = int(bool(exact)), int(bool(check_finite))
    A.log_w0 = 0.0  # a_out = 0.0 + g = g exactly
    A.obs_log_sd = float(np.log(spec.obs_sd))
    A.log_sqrt_2pi = float(LOG_SQRT_2PI)
    A.ess_rel = -1.0
    A.x_in, A.x_out = xin.data_ptr(), xout.data_ptr()
    A.theta = th.data_ptr()
    A.subs = subs_t.data_ptr() if subs_t is not None else None
    A.noise = noise_t.data_ptr() if noise_t is not None else None
    A.fs, A.workspace = fs.data_ptr(), ws.data_ptr()
    keep = []
    if spec.kernel == _lib.SSM_MODEL_GENERIC:
        A.gen, A.theta_stride = spec.handle(dev), spec.theta_stride
        for name, v in (("y_vec", y_vec), ("u_vec", u_vec)):
            if v is not None:
                t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(dev)
                keep.append(t)
                setattr(A, name, t.data_ptr())
    if obs is not None:
        bits, yy, u_obs = obs
        A.has_obs, A.obs_mask, A.u_obs = 1, bits, u_obs
        for n in range(8):
            A.y[n] = float(yy[n])
        A.a_out = a_out.data_ptr()
    _lib.check(L.ssm_propagate_weight(A, _lib.stream_ptr()), "ssm_propagate_weight")
    st = fs.cpu().numpy().reshape(-1).view(_lib.FILTER_STATE_DTYPE)[0]
    if int(st["err_param"]) != _lib.INT32_MAX:
        raise DistributionParameterError(f"{spec.name}: invalid distribution argument")
    return xout, a_out, st


def step_transition(ir, theta, x, inputs, t, dt, rng=None, check_finite=True, *, noise=None,
                    dtype="float64", exact=True, device=None):
    """Advance x (P, nx) over (t, t+dt] on the device; returns (P, nx) float64."""
    spec = resolve_model(ir)
    subs, arr = _subs(spec, t, dt, inputs)
    P = np.atleast_2d(x).shape[0]
    if noise is None:
        if rng is None:
            raise ValueError("step_transition needs rng or noise")
        noise = spec.host_noise(rng, arr, P, spec.derived(np.asarray(theta).reshape(1, -1))[0])
    u_vec = None
    if spec.kernel == _lib.SSM_MODEL_GENERIC:  # input rows per sub-step start, then the (unused) obs row
        nu = max(spec.n_input, 1)
        rows = [_input_row(inputs, t_k, spec.n_input, nu) for t_k, _ in subs] + [np.zeros(nu)]
        u_vec = np.concatenate(rows)
    xout, _, st = _run_pw(spec, theta, x, arr, noise, None, dtype, exact, check_finite, device, u_vec=u_vec)
    nf = int(st["err_nonfinite"])
    if check_finite and nf != _lib.INT32_MAX:
        t_k, d = subs[nf % 64]
        raise NonFiniteStateError(f"non-finite state after transition sub-step ending at t={t_k + d:g}",
                                  time=t_k + d)
    return xout.t().to(torch.float64).cpu().numpy()


def observe_logpdf(ir, theta, x, inputs, y, mask, *, dtype="float64", exact=True, device=None):
    """Sum of the present slots' observation log-densities, (P,) float64."""
    spec = resolve_model(ir)
    if hasattr(inputs, "at"):
        raise TypeError("observe_logpdf needs input values at the observation time, not a provider")
    mask = np.asarray(mask, dtype=bool)
    P = np.atleast_2d(x).shape[0]
    if not mask.any():
        return np.zeros(P)
    y = np.asarray(y, dtype=float)
    bits, yy = 0, np.zeros(8)
    for n in range(spec.n_obs):
        if mask[n]:
            bits |= 1 << n
            if n < 8:
                yy[n] = y[n]
    u_obs = float(np.asarray(inputs, dtype=float).reshape(-1)[0]) if spec.n_input else 0.0
    y_vec = u_vec = None
    if spec.kernel == _lib.SSM_MODEL_GENERIC:
        y_vec = np.where(mask[: spec.n_obs], y[: spec.n_obs], 0.0)
        u_vec = _input_row(inputs, None, spec.n_input, max(spec.n_input, 1))
    _, a_out, _ = _run_pw(spec, theta, x, np.zeros(0, _lib.SUBSTEP_DTYPE), None, (bits, yy, u_obs), dtype,
                          exact, False, device, y_vec=y_vec, u_vec=u_vec)
    return a_out.to(torch.float64).cpu().numpy()

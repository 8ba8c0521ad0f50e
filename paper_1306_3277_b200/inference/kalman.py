"""Kalman filter on the device for linear-Gaussian models --
the reference's inference/kalman.py API (KalmanRun, kalman_filter) and the
`filter_kind="kalman"` route of FilterRunner (mcmc.py:79-88).

The forward recursions of B systems run in one `ssm_kalman_filter` launch
(csrc/ssm_kalman.cu, one thread per system); the filtered and predicted
moments of every grid step stay on the device.  Backward smoothing draws
(kalman.py:98-114) run on the device too (`ssm_kalman_sample`, one thread per
run) from the reference's standard normals, drawn on the host from each
run's stream in its order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
from scipy.linalg import solve_triangular

from .. import _lib
from ..errors import CholeskyError, UnsupportedModelError
from ..lineargauss import LinearGaussianSystems
from .types import FilterOutcome

PIVOT_RTOL = 1e-12  # pivot tolerance relative to the largest diagonal entry (linalg.py:17-18)


@dataclass
class GaussianState:
    """Mean and upper-triangular square root of the covariance (linalg.py:100-110)."""

    mean: np.ndarray
    sqrt_cov: np.ndarray

    @property
    def dim(self):
        return self.mean.shape[0]

    def cov(self):
        return self.sqrt_cov.T @ self.sqrt_cov


def psd_cholesky_upper(S):
    """Upper U with U^T U = S for symmetric positive SEMI-definite S: a pivot
    within tolerance of zero leaves its row zero (the row must vanish), one
    below -tol raises CholeskyError (the rule of linalg.py:21-50)."""
    S = np.asarray(S, dtype=float)
    n = S.shape[0]
    tol = PIVOT_RTOL * max(1.0, float(np.max(np.abs(np.diag(S)))) if n else 1.0)
    U = np.zeros((n, n))
    for i in range(n):
        pivot = S[i, i] - U[:i, i] @ U[:i, i]
        if pivot < -tol:
            raise CholeskyError(f"matrix is not positive semi-definite at pivot {i}", index=i)
        if pivot <= tol:
            rest = S[i, i + 1 :] - U[:i, i] @ U[:i, i + 1 :]
            if np.any(np.abs(rest) > np.sqrt(tol) * max(1.0, np.max(np.abs(S)))):
                raise CholeskyError(f"matrix is not positive semi-definite at pivot {i}", index=i)
            continue
        U[i, i] = np.sqrt(pivot)
        U[i, i + 1 :] = (S[i, i + 1 :] - U[:i, i] @ U[:i, i + 1 :]) / U[i, i]
    return U


def _psd_chol_batch(S):
    """psd_cholesky_upper over a stack (B, n, n) (same pivot rule, per matrix)."""
    S = np.asarray(S, dtype=float)
    B, n, _ = S.shape
    tol = PIVOT_RTOL * np.maximum(1.0, np.max(np.abs(np.diagonal(S, axis1=1, axis2=2)), axis=1))
    big = np.sqrt(tol) * np.maximum(1.0, np.max(np.abs(S), axis=(1, 2)))
    U = np.zeros_like(S)
    for i in range(n):
        pivot = S[:, i, i] - np.einsum("bk,bk->b", U[:, :i, i], U[:, :i, i])
        rest = S[:, i, i + 1 :] - np.einsum("bk,bkj->bj", U[:, :i, i], U[:, :i, i + 1 :])
        neg = pivot < -tol
        zero = (~neg) & (pivot <= tol)
        if np.any(neg) or np.any(zero[:, None] & (np.abs(rest) > big[:, None])):
            raise CholeskyError(f"matrix is not positive semi-definite at pivot {i}", index=i)
        d = np.where(zero, 0.0, np.sqrt(np.where(zero, 1.0, pivot)))
        U[:, i, i] = d
        U[:, i, i + 1 :] = np.where(zero[:, None], 0.0, rest / np.where(zero, 1.0, d)[:, None])
    return U


def _solve_upper_t_batch(U, v):
    """U^-T v over a stack; v (B, n) or (B, n, m).  Zero pivots: pseudo-inverse."""
    Ut = U.transpose(0, 2, 1)
    vv = v[..., None] if v.ndim == 2 else v
    if np.all(np.diagonal(U, axis1=1, axis2=2) != 0):
        out = np.linalg.solve(Ut, vv)
    else:
        out = np.linalg.pinv(Ut) @ vv
    return out[..., 0] if v.ndim == 2 else out


def sample_kalman_trajectories(runs, rngs):
    """KalmanRun.sample_trajectory for many runs (kalman.py:98-114): per run the
    reference's draws in its order (step s first, then s-1 .. 0), drawn on the
    host from each run's stream; the backward recursion runs on the device
    (ssm_kalman_sample, one thread per run) over the forward pass's records."""
    out = [None] * len(runs)
    groups = {}
    for k, r in enumerate(runs):
        groups.setdefault((id(r._batch), r.pos), []).append(k)
    L = _lib.lib()
    for (_, s), ks in groups.items():
        b = runs[ks[0]]._batch
        nx = b.nx
        z = np.stack([np.asarray(rngs[k].standard_normal((s + 1) * nx), dtype=float).reshape(s + 1, nx)
                      for k in ks])  # row q = the draw for step s - q
        rows = torch.as_tensor([runs[k]._row for k in ks], dtype=torch.int32, device=b.device)
        zt = torch.as_tensor(z, dtype=torch.float64, device=b.device)
        res = torch.empty((len(ks), s + 1, nx), dtype=torch.float64, device=b.device)
        err = torch.zeros(len(ks), dtype=torch.int32, device=b.device)
        a = _lib.KalmanSampleArgs()
        a.G, a.nx, a.S, a.s = len(ks), nx, b.S, s
        a.rows, a.A, a.mu, a.P = rows.data_ptr(), b.A.data_ptr(), b.mu.data_ptr(), b.P.data_ptr()
        a.mu_p, a.P_p, a.z, a.out, a.err = b.mu_p.data_ptr(), b.P_p.data_ptr(), zt.data_ptr(), res.data_ptr(), err.data_ptr()
        with torch.cuda.device(b.device):
            _lib.check(L.ssm_kalman_sample(a, _lib.stream_ptr()), "ssm_kalman_sample")
        tr, e = res.cpu().numpy(), err.cpu().numpy()
        if e.any():
            i = int(e[e != 0][0]) - 1
            raise CholeskyError(f"matrix is not positive semi-definite at grid index {i}", index=i)
        for q, k in enumerate(ks):
            out[k] = tr[q]
    return out


def _sample_kalman_trajectories_host(runs, rngs):
    """Host (numpy) restatement of the backward recursion, vectorised over runs;
    kept to cross-check the device sampler (tests/test_gpu_kalman.py)."""
    out = [None] * len(runs)
    groups = {}
    for k, r in enumerate(runs):
        groups.setdefault((id(r._batch), r.pos), []).append(k)
    for (_, s), ks in groups.items():
        b = runs[ks[0]]._batch
        rows = torch.as_tensor([runs[k]._row for k in ks], device=b.device)
        mu = b.mu.index_select(0, rows)[:, : s + 1].cpu().numpy()
        P = b.P.index_select(0, rows)[:, : s + 1].cpu().numpy()
        mu_p = b.mu_p.index_select(0, rows)[:, : s + 1].cpu().numpy()
        P_p = b.P_p.index_select(0, rows)[:, : s + 1].cpu().numpy()
        A = b.A.index_select(0, rows)[:, :s].cpu().numpy()
        G, nx = len(ks), b.nx
        z = np.stack([np.asarray(rngs[k].standard_normal((s + 1) * nx), dtype=float).reshape(s + 1, nx)
                      for k in ks])  # row q = the draw for step s - q
        tr = np.empty((G, s + 1, nx))
        tr[:, s] = mu[:, s] + np.einsum("bji,bj->bi", _psd_chol_batch(P[:, s]), z[:, 0])
        for i in range(s - 1, -1, -1):
            Uh = _psd_chol_batch(P_p[:, i + 1])
            C = P[:, i] @ A[:, i].transpose(0, 2, 1)
            K = _solve_upper_t_batch(Uh, C.transpose(0, 2, 1)).transpose(0, 2, 1)  # C Uh^-1
            omega = mu[:, i] + np.einsum("bij,bj->bi", K, _solve_upper_t_batch(Uh, tr[:, i + 1] - mu_p[:, i + 1]))
            W = _psd_chol_batch(P[:, i] - K @ K.transpose(0, 2, 1))
            tr[:, i] = omega + np.einsum("bji,bj->bi", W, z[:, s - i])
        for q, k in enumerate(ks):
            out[k] = tr[q]
    return out


def _solve_upper_t(U, v):
    """U^-T v with zero pivots treated as absent directions."""
    d = np.diag(U)
    if np.all(d != 0):
        return solve_triangular(U, v, trans="T")
    return np.linalg.pinv(U.T) @ v


class _KalmanBatch:
    """Device tables and records of B systems along one grid."""

    def __init__(self, sys_: LinearGaussianSystems, grid, device=None):
        _lib.require_cuda()
        B, S, ny, nx = sys_.H.shape
        mx = _lib.lib().ssm_kalman_max_dim()
        if nx > mx or ny > mx:
            raise UnsupportedModelError(f"device Kalman filter: n_state, n_obs <= {mx}")
        if S != grid.last:
            raise ValueError("system and grid time axes differ")
        self.device = torch.device(device if device is not None else "cuda")
        f64 = dict(dtype=torch.float64, device=self.device)
        self.B, self.S, self.nx, self.ny = B, S, nx, ny
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=float), **f64)  # noqa: E731
        self.A, self.b, self.Q = t(sys_.A), t(sys_.b), t(sys_.Q)
        self.H, self.c, self.r = t(sys_.H), t(sys_.c), t(sys_.r_sd)
        y = np.zeros((S, max(ny, 1)))
        m = np.zeros((S, max(ny, 1)), dtype=np.uint8)
        for i in range(1, S + 1):
            obs = grid.obs_at(i)
            if obs is not None:
                y[i - 1, :ny] = np.asarray(obs[0], dtype=float)[:ny]
                m[i - 1, :ny] = np.asarray(obs[1], dtype=bool)[:ny]
        self.y = torch.as_tensor(y, **f64)
        self.mask = torch.as_tensor(m, device=self.device)
        self.mu = torch.zeros(B, S + 1, nx, **f64)
        self.P = torch.zeros(B, S + 1, nx, nx, **f64)
        self.mu[:, 0] = t(sys_.mu0)
        self.P[:, 0] = t(sys_.P0)
        self.mu_p = torch.zeros_like(self.mu)
        self.P_p = torch.zeros_like(self.P)
        self.loglik = torch.zeros(B, **f64)
        self.err = torch.zeros(B, dtype=torch.int32, device=self.device)

    def launch(self, rows, s0, s1):
        """Advance `rows` (a contiguous range lo..hi) from s0 to s1."""
        lo, hi = rows
        a = _lib.KalmanArgs()
        a.B, a.nx, a.ny, a.S, a.s0, a.s1 = hi - lo, self.nx, self.ny, self.S, s0, s1
        off = lambda t: t[lo:hi].data_ptr()  # noqa: E731
        a.A, a.b, a.Q, a.H, a.c, a.r_sd = (off(x) for x in (self.A, self.b, self.Q, self.H, self.c, self.r))
        a.y, a.mask = self.y.data_ptr(), self.mask.data_ptr()
        a.mu, a.P, a.mu_p, a.P_p = (off(x) for x in (self.mu, self.P, self.mu_p, self.P_p))
        a.loglik, a.err = off(self.loglik), off(self.err)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().ssm_kalman_filter(a, _lib.stream_ptr()), "ssm_kalman_filter")


class KalmanRun:
    """Resumable Kalman filter along a FilterGrid (kalman.py:26-114); one row of
    a device batch."""

    def __init__(self, system, grid, device=None, _batch=None, _row=0):
        self.grid = grid
        self._system = system
        self._batch = _batch if _batch is not None else _KalmanBatch(system, grid, device)
        self._row = _row
        self.loglik = 0.0
        self.pos = 0

    @property
    def system(self):
        """This run's LinearGaussianSystems row (materialised on first use)."""
        if isinstance(self._system, tuple):
            systems, k = self._system
            self._system = systems.row(k)
        return self._system

    def clone(self):
        b = self._batch
        r = self._row
        nb = _KalmanBatch.__new__(_KalmanBatch)
        nb.__dict__.update(b.__dict__)
        for f in ("A", "b", "Q", "H", "c", "r", "mu", "P", "mu_p", "P_p", "loglik", "err"):
            setattr(nb, f, getattr(b, f)[r : r + 1].clone())
        nb.B = 1
        other = KalmanRun(self._system, self.grid, _batch=nb, _row=0)
        other.loglik, other.pos = self.loglik, self.pos
        return other

    def advance_to(self, upto, rng=None):
        """Prediction/correction through grid index `upto`; returns the
        log-likelihood increment (kalman.py:53-59)."""
        return advance_kalman_runs([self], upto)[0]

    def _records(self):
        b, r = self._batch, self._row
        return (b.mu[r].cpu().numpy(), b.P[r].cpu().numpy(), b.mu_p[r].cpu().numpy(), b.P_p[r].cpu().numpy())

    def filtered(self, i):
        b, r = self._batch, self._row
        return GaussianState(b.mu[r, i].cpu().numpy(), psd_cholesky_upper(b.P[r, i].cpu().numpy()))

    def sample_trajectory(self, rng):
        """Backward smoothing sample x(t_{0:pos}) (kalman.py:98-114): the same
        draws in the same order, covariance-form algebra."""
        return sample_kalman_trajectories([self], [rng])[0]

    def _sample_trajectory_serial(self, rng):
        s = self.pos
        mu, P, mu_p, P_p = self._records()
        A = self._batch.A[self._row].cpu().numpy()
        nx = mu.shape[1]
        out = np.empty((s + 1, nx))
        out[s] = mu[s] + psd_cholesky_upper(P[s]).T @ rng.standard_normal(nx)
        for i in range(s - 1, -1, -1):
            Uh = psd_cholesky_upper(P_p[i + 1])
            C = P[i] @ A[i].T  # Cov(x_i, x_{i+1} | y_{1:i})
            K = _solve_upper_t(Uh, C.T).T  # C Uh^-1
            omega = mu[i] + K @ _solve_upper_t(Uh, out[i + 1] - mu_p[i + 1])
            W = psd_cholesky_upper(P[i] - K @ K.T)
            out[i] = omega + W.T @ rng.standard_normal(nx)
        return out


def advance_kalman_runs(runs, upto):
    """Advance many runs through `upto`: one launch per batch (runs of one batch
    at the same position), else one launch per run.  Returns the increments."""
    groups = {}
    for k, r in enumerate(runs):
        groups.setdefault((id(r._batch), r.pos), []).append(k)
    before = [r.loglik for r in runs]
    for (_, pos), ks in groups.items():
        if upto <= pos:
            continue
        b = runs[ks[0]]._batch
        rows = sorted(runs[k]._row for k in ks)
        if rows == list(range(rows[0], rows[0] + len(rows))):
            b.launch((rows[0], rows[-1] + 1), pos, upto)
        else:
            for k in ks:
                b.launch((runs[k]._row, runs[k]._row + 1), pos, upto)
    seen = {}
    for r in runs:
        if id(r._batch) not in seen:
            seen[id(r._batch)] = (r._batch.loglik.cpu().numpy(), r._batch.err.cpu().numpy())
    out = []
    for r, ll0 in zip(runs, before):
        ll, err = seen[id(r._batch)]
        if err[r._row]:
            t = float(r.grid.times[err[r._row]])
            raise CholeskyError(f"innovation covariance not positive definite at t={t:g}", index=int(err[r._row]))
        r.loglik = float(ll[r._row])
        r.pos = max(r.pos, upto)
        out.append(r.loglik - ll0)
    return out


def kalman_runs(systems: LinearGaussianSystems, grid, device=None):
    """B fresh runs sharing one device batch."""
    batch = _KalmanBatch(systems, grid, device)
    return [KalmanRun((systems, k), grid, _batch=batch, _row=k) for k in range(systems.B)]


def kalman_filter(system, grid, rng, upto=None, device=None):
    """Filter through `upto` (default: the whole grid) and draw one smoothing
    trajectory (kalman.py:117-122)."""
    run = KalmanRun(system, grid, device)
    run.advance_to(grid.last if upto is None else upto)
    trajectory = run.sample_trajectory(rng)
    summaries = [run.filtered(i) for i in range(run.pos + 1)]
    return FilterOutcome(loglik=run.loglik, trajectory=trajectory, summaries=summaries, run=run)

"""Bootstrap particle filter on the B200 (drop-in for the reference's
inference/particle.py:28-185).

`ParticleRun` implements the reference's run protocol -- init(rng),
advance_to(upto, rng) -> loglik increment, sample_trajectory(rng), clone(),
ess(), attributes pos / loglik / x / logw / n_particles / history -- with all
per-particle work in libssm_b200.so:

    per grid step i (particle.py:107-135)
      [K4 ssm_weights_scan]    cumsum(w / sum w)             resampling.py:26-27
      [K5 ssm_resample_search] searchsorted(cum, u, 'right') resampling.py:28-36
      [K1/K2 ssm_propagate_weight]  x[anc] -> step_transition -> observe_logpdf
                               -> logw + g -> LSE -> loglik, ESS gate (fused)

Several filters with the same grid, model and particle count advance in one
launch (`advance_runs`), which the PMMH and SMC^2 drivers use.  The host
loop only enqueues kernels; the device state machine (weights_uniform,
resample decision, errors) lives in `ssm_filter_state` and is read once per
advance_to call.

Noise modes
  "device": Philox4x32-10 normals/uniforms drawn on the device (fast path).
  "host":   the reference's own draws (numpy Philox via RngStream, same keys
            and order, rng.py / simulate.py:50-60 / resampling.py:28-33) are
            generated on the host and injected, so a float64 run reproduces
            the reference filter (parity mode).
Arithmetic: `exact` (default: True with host noise, False with device noise)
selects the reference's float64 op order without FMA contraction (bitwise)
over the FMA-contracted fast kernels (1e-12 of the reference per step).
"""

from __future__ import annotations

import ctypes as C
import math
import operator

import numpy as np
import torch

from .. import _lib, profiling
from ..errors import DegenerateEnsembleError, DistributionParameterError, NonFiniteStateError, UnsupportedModelError
from ..models import LOG_SQRT_2PI, ModelSpec, resolve_model
from ..rng import device_keys, first_uniforms
from .timegrid import as_filter_grid
from .types import FilterOutcome

import os

_NO_HINTS = bool(os.environ.get("SSM_NO_HINTS"))  # A/B switch for the specialised kernels
_NO_COOP = bool(os.environ.get("SSM_NO_COOP"))  # A/B switch: per-step kernels instead of the persistent driver
# the persistent cooperative driver (ssm_advance_coop) runs advances of at most this many
# particles per launch (B x P).  Off by default: measured on B200 it is slower than the
# per-step PDL chain at every size tried (config 3: 5.98 vs 4.27 ms per MH step; L96
# 2^16 / 2^18 / 2^20: 1.44 / 4.77 / 8.84e9 vs 1.69 / 5.79 / 12.4e9 particle-updates/s;
# profiles/r2_coop_ab.txt) -- grid-wide barriers cost more than the launches they replace.
COOP_MAX_PARTICLES = int(os.environ.get("SSM_COOP_MAX", "0"))
_RESAMPLE_KEY = 0  # particle.py:24
_PROPAGATE_KEY = 1  # particle.py:25
SCHEMES = ("multinomial", "stratified", "systematic")
_DT = {"float64": (torch.float64, _lib.SSM_F64), "float32": (torch.float32, _lib.SSM_F32)}


def _dtype_info(dtype):
    key = {torch.float64: "float64", torch.float32: "float32", np.float64: "float64",
           np.float32: "float32"}.get(dtype, dtype)
    if key not in _DT:
        raise ValueError(f"unsupported dtype {dtype!r}")
    return key, _DT[key][0], _DT[key][1]


# ---------------------------------------------------------------------------
# per-(grid, model, inputs) host schedule and its device table
# ---------------------------------------------------------------------------


def substep_schedule(t, dt, delta):
    """simulate.py:28-38."""
    if delta is None:
        return [(t, dt)]
    n_sub = max(1, int(np.ceil(dt / delta - 1e-9)))
    t_end = t + dt
    return [(t + k * delta, min(delta, t_end - (t + k * delta))) for k in range(n_sub)]


def _input_vector(inputs, t, n_input, width):
    """Input values at t (InputProvider.at, timeseries.py:205-210), zero-padded to width."""
    out = np.zeros(width)
    if inputs is not None and n_input:
        v = np.asarray(inputs.at(t) if hasattr(inputs, "at") else inputs, dtype=float).reshape(-1)
        out[:n_input] = v[:n_input]
    return out


def _input_value(inputs, t):
    if inputs is None:
        return 0.0
    if hasattr(inputs, "at"):
        return float(np.asarray(inputs.at(t), dtype=float).reshape(-1)[0])
    return float(np.asarray(inputs, dtype=float).reshape(-1)[0])


class Schedule:
    """Per-step sub-step records, observation data and error time lookup."""

    def __init__(self, grid, spec: ModelSpec, inputs, device):
        times = grid.times
        S = len(times) - 1
        recs, self.offsets, self.n_sub, self.sub_end = [], [0] * (S + 1), [0] * (S + 1), [None] * (S + 1)
        self.sub_start = [None] * (S + 1)
        self.host_subs = [None] * (S + 1)
        self.obs = [None] * (S + 1)
        self.single = [False] * (S + 1)
        for i in range(1, S + 1):
            t0, t1 = times[i - 1], times[i]
            dt = t1 - t0
            if dt <= 0:
                raise ValueError("step_transition requires dt > 0")
            subs = substep_schedule(t0, dt, spec.delta)
            arr = np.zeros(len(subs), dtype=_lib.SUBSTEP_DTYPE)
            ends = []
            for k, (t_k, d) in enumerate(subs):
                arr[k]["d"] = d
                arr[k]["sd"] = math.sqrt(d)
                arr[k]["u_in"] = _input_value(inputs, t_k) if spec.n_input else 0.0
                if spec.has_ode:
                    n_ode = max(1, int(np.ceil(d / spec.h - 1e-9)))  # simulate.py:85
                    if n_ode > 4:
                        raise UnsupportedModelError("more than 4 RK4 steps per sub-step")
                    for m in range(n_ode):
                        arr[k]["s"][m] = min(spec.h, d - m * spec.h)  # simulate.py:87
                    arr[k]["n_ode"] = n_ode
                ends.append(t_k + d)
            self.offsets[i] = len(recs)
            self.n_sub[i] = len(subs)
            self.single[i] = len(subs) == 1 and (not spec.has_ode or int(arr[0]["n_ode"]) == 1)
            if spec.kernel == _lib.SSM_MODEL_GENERIC:  # every ode statement: one RK4 step (codegen, simulate.py:85)
                self.single[i] = len(subs) == 1 and all(max(1, int(np.ceil(subs[0][1] / h - 1e-9))) == 1
                                                        for h in spec.ode_h)
            self.sub_end[i] = ends
            self.sub_start[i] = [t_k for t_k, _ in subs]
            self.host_subs[i] = arr
            recs.extend(arr)
            o = grid.obs_at(i)
            if o is not None:
                y, mask = o
                y = np.asarray(y, dtype=float)
                mask = np.asarray(mask, dtype=bool)
                bits = 0
                yy = np.zeros(8)
                for n in range(min(spec.n_obs, 8)):
                    if mask[n]:
                        bits |= 1 << n
                        yy[n] = y[n]
                u_obs = _input_value(inputs, t1) if spec.n_input else 0.0
                self.obs[i] = (bits, yy, u_obs)
        # generic models: per-step observation vectors and input rows in device tables
        # (ssm_pw_args.y_vec / u_vec; the fixed y[8] / u_in fields cover the hand-written kernels)
        self.y_off = [-1] * (S + 1)
        self.u_off = [-1] * (S + 1)
        ytab, utab = [], []
        if spec.kernel == _lib.SSM_MODEL_GENERIC:
            nu = max(spec.n_input, 1)
            for i in range(1, S + 1):
                rows = [_input_vector(inputs, t_k, spec.n_input, nu) for t_k in self.sub_start[i]]
                o = grid.obs_at(i)
                rows.append(_input_vector(inputs, times[i], spec.n_input, nu) if o is not None else np.zeros(nu))
                self.u_off[i] = len(utab)
                utab.extend(np.concatenate(rows))
                if o is not None:
                    self.y_off[i] = len(ytab)
                    yv = np.zeros(max(spec.n_obs, 1))
                    yv[: spec.n_obs] = np.where(np.asarray(o[1], dtype=bool), np.asarray(o[0], dtype=float), 0.0)
                    ytab.extend(yv)
                    bits = 0
                    for n in range(spec.n_obs):
                        if o[1][n]:
                            bits |= 1 << n
                    self.obs[i] = (bits, self.obs[i][1], self.obs[i][2])
        self.y_table = torch.tensor(ytab if ytab else [0.0], dtype=torch.float64, device=device)
        self.u_table = torch.tensor(utab if utab else [0.0], dtype=torch.float64, device=device)
        # native-driver step descriptors (ssm_step_desc), one per grid index
        self.desc = np.zeros(S + 1, dtype=_lib.STEP_DESC_DTYPE)
        for i in range(1, S + 1):
            d = self.desc[i]
            d["step"], d["n_sub"], d["subs_offset"] = i, self.n_sub[i], self.offsets[i]
            d["hints"] = _lib.SSM_HINT_SINGLE_SUBSTEP if self.single[i] else 0
            d["y_off"], d["u_off"] = self.y_off[i], self.u_off[i]
            if self.obs[i] is not None:
                d["has_obs"], d["obs_mask"] = 1, self.obs[i][0]
                d["y"] = self.obs[i][1]
                d["u_obs"] = self.obs[i][2]
        self.desc_dev = torch.from_numpy(self.desc.view(np.uint8).copy()).to(device)
        table = np.array(recs, dtype=_lib.SUBSTEP_DTYPE) if recs else np.zeros(1, _lib.SUBSTEP_DTYPE)
        self.table = torch.from_numpy(table.view(np.uint8).copy()).to(device)
        self.times = times

    def y_ptr(self, i):
        return None if self.y_off[i] < 0 else self.y_table.data_ptr() + 8 * self.y_off[i]

    def u_ptr(self, i):
        return None if self.u_off[i] < 0 else self.u_table.data_ptr() + 8 * self.u_off[i]

    def subs_ptr(self, i):
        return self.table.data_ptr() + self.offsets[i] * _lib.SUBSTEP_DTYPE.itemsize


def _schedule(grid, spec, inputs, device):
    key = (getattr(spec, "digest", spec.name), id(inputs), str(device))
    cache = grid._device_cache
    hit = cache.get(key)
    if hit is None or hit[0] is not inputs:
        hit = (inputs, Schedule(grid, spec, inputs, device))
        cache[key] = hit
    return hit[1]


_zero_cache: dict = {}


def _zeros_logw(P, tdtype, device):
    k = (P, tdtype, str(device))
    z = _zero_cache.get(k)
    if z is None:
        z = torch.zeros((1, P), dtype=tdtype, device=device)
        _zero_cache[k] = z
    return z


def _fs_init(B, device):
    fs = np.zeros(B, dtype=_lib.FILTER_STATE_DTYPE)
    fs["uniform"] = 1
    fs["err_nonfinite"] = _lib.INT32_MAX
    fs["err_degenerate"] = _lib.INT32_MAX
    fs["err_param"] = _lib.INT32_MAX
    return _lib.h2d(fs.view(np.uint8).reshape(B, 64), device)


def _stack_rows(tensors):
    """Batch per-filter views; zero-copy when they are consecutive rows of one
    base tensor (the common case: a run batch advanced together)."""
    t0 = tensors[0]
    if len(tensors) == 1:
        return t0.unsqueeze(0)
    base = t0._base if t0._base is not None else None
    if base is not None and base.is_contiguous() and base.dim() == t0.dim() + 1:
        stride = t0.numel()
        start = (t0.data_ptr() - base.data_ptr()) // t0.element_size()
        ok = start % stride == 0 and all(
            t._base is base and t.data_ptr() == t0.data_ptr() + k * stride * t0.element_size()
            for k, t in enumerate(tensors)
        )
        if ok:
            r0 = start // stride
            return base[r0 : r0 + len(tensors)]
    return torch.stack(tensors)


# ---------------------------------------------------------------------------
# history segments
# ---------------------------------------------------------------------------


class _Seg:
    """The history one init / advance call wrote for a batch of runs: grid
    indices i0 .. i0 + n - 1 of every run b in the batch.  x [n, B, nx, P]
    (None: history-free), anc [n, B, P] with used[k] (False: identity).  A
    run keeps (segment, b) pairs (which own the memory and give the history
    views) plus flat per-grid-index pointer arrays for the trace / replay
    kernels, extended once per call with numpy -- O(B) host work per call,
    not O(B x steps)."""

    __slots__ = ("x", "anc", "used", "n")

    def __init__(self, x, anc, used, n):
        self.x, self.anc, self.used, self.n = x, anc, used, n

    def views(self, b):
        for k in range(self.n):
            yield (self.x[k][b] if self.x is not None else None,
                   self.anc[k][b] if (self.anc is not None and self.used[k]) else None)


class _RowRef:
    """Descriptor for a run's per-filter device state (positions, log-weights,
    tile CDF / records, filter state): held as (batch tensor, row) and turned
    into a view only when read, so an advance over B runs sets B x 5
    references instead of slicing B x 5 tensors; `_rows` takes a batch back in
    one slice when the runs are consecutive rows of one batch."""

    def __init__(self, name):
        self.key = "_rb" + name

    def __get__(self, obj, cls=None):
        if obj is None:
            return self
        ref = obj.__dict__.get(self.key)
        if ref is None:
            return None
        t, b = ref
        return t if b is None else t[b]

    def __set__(self, obj, value):
        obj.__dict__[self.key] = None if value is None else (value, None)


class _NpRow:
    """Descriptor for a run's host pointer / key arrays (per grid index), held as
    (2-D batch array, row) after a batched advance so B runs share one block;
    `_np_rows` gives a batch back without re-stacking when possible."""

    def __init__(self, name):
        self.key = "_nb" + name

    def __get__(self, obj, cls=None):
        if obj is None:
            return self
        a, b = obj.__dict__[self.key]
        return a if b is None else a[b]

    def __set__(self, obj, value):
        obj.__dict__[self.key] = (value, None)


def _np_rows(runs, name):
    """[B, ...] array of the runs' `name` arrays: a slice / one fancy index of the shared
    block when every run holds a row of it, else np.stack."""
    key = "_nb" + name
    refs = [r.__dict__[key] for r in runs]
    a0, b0 = refs[0]
    if b0 is not None and all(a is a0 for a, _ in refs):
        rows = [b for _, b in refs]
        if rows == list(range(b0, b0 + len(rows))):
            return a0[b0 : b0 + len(rows)]
        return a0[rows]
    return np.stack([a if b is None else a[b] for a, b in refs])


def _set_row(run, name, batch, b):
    run.__dict__["_rb" + name] = None if batch is None else (batch, b)


def _has_row(run, name):
    return run.__dict__.get("_rb" + name) is not None


def _rows(runs, name):
    """[B, ...] tensor of the runs' `name` rows: one slice of the shared batch when
    they are its consecutive rows, else a stack of the views."""
    key = "_rb" + name
    refs = [r.__dict__.get(key) for r in runs]
    t0, b0 = refs[0]
    if b0 is not None and all(t is t0 for t, _ in refs):
        rows = [b for _, b in refs]
        if rows == list(range(b0, b0 + len(rows))):
            return t0 if (b0 == 0 and len(rows) == t0.shape[0]) else t0[b0 : b0 + len(rows)]
        # rows of one batch in another order (a theta-resampled SMC^2 ensemble): one gather
        return t0.index_select(0, _lib.h2d(np.asarray(rows, dtype=np.int64), t0.device))
    groups = {}
    for k, (t, b) in enumerate(refs):
        if b is None:
            break
        g = groups.setdefault(id(t), (t, [], []))
        g[1].append(k)
        g[2].append(b)
    else:
        if len(groups) <= 8:  # rows of a few batches (SMC^2 after a rejuvenation): one gather per batch
            out = torch.empty((len(refs),) + tuple(t0.shape[1:]), dtype=t0.dtype, device=t0.device)
            for t, pos, rows in groups.values():
                idx = _lib.h2d(np.array([pos, rows], dtype=np.int64), t0.device)
                out.index_copy_(0, idx[0], t.index_select(0, idx[1]))
            return out
    return torch.stack([t if b is None else t[b] for t, b in refs])


def _rows_many(runs, names):
    """{name: _rows(runs, name)} for names whose references share one row layout
    (every run's rows come from the same batches): the grouping and the index
    upload are done once for all names."""
    refs0 = [r.__dict__.get("_rb" + names[0]) for r in runs]
    if any(ref is None or ref[1] is None for ref in refs0):
        return {n: _rows(runs, n) for n in names}
    t0, b0 = refs0[0]
    rows = [b for _, b in refs0]
    if all(t is t0 for t, _ in refs0) and rows == list(range(b0, b0 + len(rows))):
        return {n: _rows(runs, n) for n in names}  # slices: nothing to share
    order = {}  # batch (identified by the first name's tensor) -> positions
    for k, (t, _) in enumerate(refs0):
        order.setdefault(id(t), []).append(k)
    if len(order) > 8:
        return {n: _rows(runs, n) for n in names}
    groups = list(order.values())
    flat = np.concatenate([np.array([pos, [rows[k] for k in pos]], dtype=np.int64) for pos in groups], axis=1)
    idx = _lib.h2d(flat, t0.device)  # [2, B]: positions, rows (group after group)
    out = {}
    for n in names:
        refs = [r.__dict__.get("_rb" + n) for r in runs]
        bases = []
        ok = True
        for pos in groups:
            tb = refs[pos[0]][0]
            if any(refs[k] is None or refs[k][0] is not tb or refs[k][1] != rows[k] for k in pos):
                ok = False
                break
            bases.append(tb)
        if not ok:
            out[n] = _rows(runs, n)
            continue
        tn = bases[0]
        res = torch.empty((len(runs),) + tuple(tn.shape[1:]), dtype=tn.dtype, device=tn.device)
        off = 0
        for pos, tb in zip(groups, bases):
            m = len(pos)
            res.index_copy_(0, idx[0, off : off + m], tb.index_select(0, idx[1, off : off + m]))
            off += m
        out[n] = res
    return out


_EMPTY_I64 = np.zeros(0, dtype=np.int64)
_EMPTY_KEYS = np.zeros((0, 2), dtype=np.uint32)


# ---------------------------------------------------------------------------
# the run object
# ---------------------------------------------------------------------------


class ParticleRun:
    """Resumable bootstrap particle filter along a FilterGrid, on the GPU."""

    _x = _RowRef("_x")  # (nx, P) positions at grid index pos
    _a = _RowRef("_a")  # (P,) unnormalised log-weights of the last weighted step
    _cdf = _RowRef("_cdf")  # (P,) tile-local fixed-point CDF of the last weighted step
    _trec = _RowRef("_trec")  # (ceil(P/32), 2) warp-tile records {max, Q} of the last weighted step
    _fs = _RowRef("_fs")  # (64,) uint8 view of an ssm_filter_state
    _hx = _NpRow("_hx")  # device pointers of history[i][0] (trace-kernel pointer table), per grid index
    _ha = _NpRow("_ha")  # device pointers of history[i][1] (0 = identity)
    _kk = _NpRow("_kk")  # history-free runs: Philox key (2 x uint32) used at each grid index

    def __init__(self, ir, theta, grid, inputs=None, n_particles=1024, resampler="multinomial",
                 ess_rel=None, initial_state=None, check_finite=True, *, dtype="float64",
                 exact=None, noise="device", device=None, keep_history=True):
        if n_particles < 2:
            raise ValueError("particle filter needs n_particles >= 2")
        if resampler not in SCHEMES:
            raise ValueError(f"unknown resampling scheme {resampler!r}")
        if noise not in ("device", "host"):
            raise ValueError(f"unknown noise mode {noise!r}")
        _lib.require_cuda()
        self.spec = resolve_model(ir)
        self.ir = ir
        self.theta = np.asarray(theta, dtype=float).reshape(1, -1)
        self.grid = as_filter_grid(grid)
        self.inputs = inputs
        self.n_particles = int(n_particles)
        self.resampler = resampler
        self.ess_rel = ess_rel
        self.initial_state = initial_state
        self.check_finite = check_finite
        self.dtype_name, self.tdtype, self.dtype_id = _dtype_info(dtype)
        # exact: float64 in the reference's op order without FMA contraction, which
        # with noise="host" is bitwise the reference; default on for host noise and
        # off (FMA, 1e-12 of the reference per step) for device noise
        self.exact = (noise == "host") if exact is None else bool(exact)
        self.noise = noise
        # keep_history=False (device noise): only the ancestors are stored per grid
        # step; sample_trajectory replays the chosen ancestral line (ssm_replay_path),
        # bitwise the same trajectory at ~1/17 of the f64 L96 history memory
        if not keep_history and noise != "device":
            raise ValueError("keep_history=False needs device noise (host draws cannot be replayed)")
        self.keep_history = bool(keep_history)
        if self.spec.kernel == _lib.SSM_MODEL_GENERIC:
            if not self.keep_history:
                raise UnsupportedModelError(f"{self.spec.name}: history-free runs need a hand-written model kernel")
            if noise == "host":
                self.spec.check_host_noise()
        self._kk = _EMPTY_KEYS  # history-free runs: Philox key (2 x uint32) used at each grid index
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.loglik = 0.0
        self.pos = 0
        self.weights_uniform = True
        self._segs = []  # (_Seg, row b) per init / advance call, in grid-index order
        self._x = None
        self._a = None  # unnormalised log-weights of the last weighted step
        self._fs = None  # (64,) uint8 view of an ssm_filter_state
        self._cdf = None  # (P,) tile-local fixed-point CDF of the last weighted step
        self._trec = None  # (ceil(P/32), 2) warp-tile records {max, Q} of the last weighted step
        self._hx = _EMPTY_I64  # device pointers of history[i][0] (trace-kernel pointer table), per grid index
        self._ha = _EMPTY_I64  # device pointers of history[i][1] (0 = identity)
        self._maybe_nonuniform = False
        self._derived = None

    # -- protocol -------------------------------------------------------------
    def init(self, rng):
        init_runs([self], [rng])
        return self

    def clone(self):
        # the pointer arrays are never modified in place (every advance makes new
        # ones), so a clone shares them; the segment list is copied
        other = ParticleRun.__new__(ParticleRun)
        other.__dict__ = dict(self.__dict__)
        other._segs = list(self._segs)
        return other

    @property
    def initialized(self):
        return self._x is not None

    @property
    def history(self):
        """[(x_i [nx, P], anc_i [P] | None)] per grid index (particle.py:59, 135); views made on access."""
        if not self.keep_history:
            raise ValueError("this run keeps no position history (keep_history=False); "
                             "sample_trajectory replays the ancestral line instead")
        return [v for seg, b in self._segs for v in seg.views(b)]

    def _set_history(self, xs, ancs, keys=None):
        """Install a history (a migrated SMC^2 theta-particle): xs [pos+1, nx, P] or None
        (history-free, keys [pos+1, 2]), ancs [pos, P] ancestors (identity rows included)."""
        n = ancs.shape[0] + 1
        self._segs = [(_Seg(xs[:1].unsqueeze(1) if xs is not None else None, None, np.zeros(1, bool), 1), 0)]
        if n > 1:
            self._segs.append((_Seg(xs[1:].unsqueeze(1) if xs is not None else None, ancs.unsqueeze(1),
                                    np.ones(n - 1, bool), n - 1), 0))
        if xs is not None:
            self._hx = xs.data_ptr() + (xs[0].numel() * xs.element_size()) * np.arange(n, dtype=np.int64)
        else:
            self._hx = np.zeros(n, dtype=np.int64)
        astep = ancs[0].numel() * ancs.element_size() if n > 1 else 0
        self._ha = np.concatenate([np.zeros(1, np.int64), ancs.data_ptr() + astep * np.arange(n - 1, dtype=np.int64)])
        self._kk = np.asarray(keys, dtype=np.uint32).reshape(n, 2) if keys is not None else _EMPTY_KEYS

    def advance_to(self, upto, rng):
        return float(advance_runs([self], upto, [rng])[0])

    def sample_trajectory(self, rng):
        return sample_trajectories([self], [rng])[0]

    def ess(self):
        a = self._a if not self.weights_uniform else _zeros_logw(self.n_particles, self.tdtype, self.device)[0]
        L = _lib.lib()
        ws = torch.empty(L.ssm_lse_workspace_bytes(1, self.n_particles), dtype=torch.uint8, device=self.device)
        out = torch.empty(2, dtype=torch.float64, device=self.device)
        _lib.check(L.ssm_logsumexp(self.dtype_id, 1, self.n_particles, _lib.ptr(a), _lib.ptr(out),
                                   C_ptr(out, 1), _lib.ptr(ws), _lib.stream_ptr()), "ssm_logsumexp")
        return float(out[1].item())

    @property
    def x(self):
        """(P, nx) float64 host copy (SoA -> AoS transpose on read)."""
        if self._x is None:
            return None
        return self._x.t().to(torch.float64).cpu().numpy()

    @property
    def logw(self):
        """(P,) normalised log-weights on the host (particle.py:58)."""
        if self._x is None:
            return None
        P = self.n_particles
        if self.weights_uniform:
            return np.full(P, -np.log(P))
        incr = _fs_view(self._fs)["incr"][0]
        return self._a.to(torch.float64).cpu().numpy() - incr

    def weighted_mean(self):
        lw = self.logw
        w = np.exp(lw - np.max(lw))
        w /= w.sum()
        return w @ self.x

    def x_device(self):
        """(nx, P) device tensor of the current positions (no copy)."""
        return self._x


def C_ptr(t, offset_elems):
    import ctypes

    return ctypes.c_void_p(t.data_ptr() + offset_elems * t.element_size())


def _fs_view(fs_tensor):
    return fs_tensor.detach().cpu().numpy().reshape(-1).view(_lib.FILTER_STATE_DTYPE)


_SETTINGS = operator.attrgetter("spec", "grid", "n_particles", "dtype_id", "resampler", "ess_rel", "check_finite",
                                "exact", "noise", "keep_history", "pos", "device", "inputs")


def _common(runs):
    r0 = runs[0]
    k0 = _SETTINGS(r0)
    for r in runs[1:]:
        k = _SETTINGS(r)
        # element-wise: identity for the shared objects (spec, grid, inputs), equality for the rest
        if k != k0 or k[0] is not k0[0] or k[1] is not k0[1] or k[12] is not k0[12]:
            raise ValueError("runs advanced together must share model, grid, settings and position")
    return r0


def _derived_tensor(runs):
    todo = [r for r in runs if r._derived is None]
    if todo:  # one vectorised call for the runs without cached constants
        d = todo[0].spec.derived(np.concatenate([r.theta for r in todo]))
        for r, row in zip(todo, d):
            r._derived = row
    return _lib.h2d(np.stack([r._derived for r in runs]), runs[0].device)


def init_runs(runs, rngs):
    """ParticleRun.init for a batch (particle.py:61-71)."""
    r0 = _common(runs)
    B, P, spec = len(runs), r0.n_particles, r0.spec
    dev = r0.device
    x = torch.empty((B, spec.nx, P), dtype=r0.tdtype, device=dev)
    need_draw = [b for b, r in enumerate(runs) if r.initial_state is None]
    fixed = [b for b, r in enumerate(runs) if r.initial_state is not None]
    if fixed:  # np.tile(initial_state, (P, 1)) (particle.py:63-65): one H2D + one broadcast copy
        x0 = torch.from_numpy(np.stack([np.asarray(runs[b].initial_state, dtype=float) for b in fixed]))
        x0 = _lib.h2d(x0, dev).to(r0.tdtype).view(len(fixed), spec.nx, 1).expand(len(fixed), spec.nx, P)
        if len(fixed) == B:
            x.copy_(x0)
        else:
            x[_lib.h2d(np.asarray(fixed, dtype=np.int64), dev)] = x0
    if need_draw:
        if r0.noise == "host":
            for b in need_draw:
                x0b = spec.host_initial(rngs[b], P, runs[b].theta)
                x[b].copy_(torch.from_numpy(x0b.T.copy()).to(r0.tdtype))
        else:
            keys = device_keys([rngs[b] for b in need_draw])
            kt = _lib.h2d(keys.view(np.int32), dev)
            if spec.kernel == _lib.SSM_MODEL_GENERIC:  # the model's initial block, NVRTC-compiled
                th = _lib.h2d(spec.derived(np.concatenate([runs[b].theta for b in need_draw])), dev)
                tmp = torch.empty((len(need_draw), spec.nx, P), dtype=r0.tdtype, device=dev)
                fs_init = _fs_init(len(need_draw), dev)
                _lib.check(_lib.lib().ssm_gen_init_particles(
                    C.c_void_p(spec.handle(dev)), r0.dtype_id, len(need_draw), P, 0, _lib.ptr(kt), _lib.ptr(th),
                    spec.theta_stride, _lib.ptr(tmp), _lib.ptr(fs_init), _lib.stream_ptr()), "ssm_gen_init_particles")
                if int(_fs_view(fs_init)["err_param"].min()) != _lib.INT32_MAX:
                    raise DistributionParameterError(f"{spec.name}: invalid initial-block distribution argument")
                for j, b in enumerate(need_draw):
                    x[b].copy_(tmp[j])
            elif len(need_draw) == B:
                _lib.check(_lib.lib().ssm_init_particles(spec.kernel, r0.dtype_id, B, P, 0, _lib.ptr(kt),
                                                         _lib.ptr(x), _lib.stream_ptr()), "ssm_init_particles")
            else:
                tmp = torch.empty((len(need_draw), spec.nx, P), dtype=r0.tdtype, device=dev)
                _lib.check(_lib.lib().ssm_init_particles(spec.kernel, r0.dtype_id, len(need_draw), P, 0,
                                                         _lib.ptr(kt), _lib.ptr(tmp), _lib.stream_ptr()),
                           "ssm_init_particles")
                for j, b in enumerate(need_draw):
                    x[b].copy_(tmp[j])
    fs = _fs_init(B, dev)
    if not r0.keep_history:  # what the trajectory replay needs to regenerate x_0
        init_keys = np.zeros((B, 2), dtype=np.uint32)
        if need_draw and r0.noise != "host":
            init_keys[need_draw] = keys
    seg = _Seg(x.unsqueeze(0) if r0.keep_history else None, None, np.zeros(1, bool), 1)
    xrow = x[0].numel() * x.element_size()
    hx0 = (x.data_ptr() + xrow * np.arange(B, dtype=np.int64)[:, None] if r0.keep_history
           else np.zeros((B, 1), dtype=np.int64))
    ha0 = np.zeros((B, 1), dtype=np.int64)
    kk0 = init_keys[:, None, :].copy() if not r0.keep_history else None
    for b, r in enumerate(runs):
        d = r.__dict__
        d["_nb_kk"] = (kk0, b) if kk0 is not None else (_EMPTY_KEYS, None)
        _set_row(r, "_x", x, b)
        r._a = None
        r._cdf = None
        r._trec = None
        _set_row(r, "_fs", fs, b)
        r.loglik = 0.0
        r.pos = 0
        r.weights_uniform = True
        r._maybe_nonuniform = False
        r._segs = [(seg, b)]
        d["_nb_hx"] = (hx0, b)
        d["_nb_ha"] = (ha0, b)
    return runs


# kernels per resample: tiles = tile scale (+ block prefix in its last block),
# offspring, long runs (sorted multinomial: tile scale, spacing sums, spacing
# prefix, merge); logw multinomial = scan, search; logw sorted multinomial = scan,
# spacing sums, spacing prefix, merge; logw systematic/stratified = tile sums,
# tile prefix, offspring, expand
_RS_LAUNCHES = {("tiles", 1): 3, ("tiles", 2): 3, ("tiles", 3): 4,
                ("logw", 0): 2, ("logw", 1): 4, ("logw", 2): 4, ("logw", 3): 4}


def _resample_bytes(esz):
    """Algorithmic bytes per particle of a resample (B_R without the
    gather, which the fused kernel performs): read the weight (r) + write the
    ancestor (4).  The CDF (cdf_local / tile records / spacing prefixes) is an
    implementation intermediate and is not counted."""
    return esz + 4


def _pw_bytes(nx, esz, resampled, weighted):
    """Algorithmic bytes per particle of one fused step (SURVEY 8d B_P plus the
    gather's ancestor read): x in + x out (2 nx r), the ancestor (4) when the step
    resampled, the log-weight (r) when it weighted.  cdf_local and a_out are
    implementation intermediates (not counted)."""
    return 2 * nx * esz + (4 if resampled else 0) + (esz if weighted else 0)


def _advance_native(L, r0, B, P, spec, sched, start, upto, args, x_prev, a_last, maybe, x_arena, a_arena,
                    cdf_local, tile_rec, rs_ws, tiles_ok, scheme, esz, new_hist, stream):
    """One ssm_advance call for all steps (device noise).  Returns (x_prev,
    a_last, maybe_nonuniform) and appends (x_out, anc | None) per step."""
    import ctypes as C

    n = upto - start
    desc = np.ascontiguousarray(sched.desc[start + 1 : upto + 1])
    if _NO_HINTS:
        desc["hints"] = 0
    anc_arena = torch.empty((n, B, P), dtype=torch.int32, device=args_device(x_arena)) if (maybe or any(
        desc["has_obs"][:-1])) else None
    anc_used = np.zeros(n, dtype=np.int32)
    A = _lib.AdvanceArgs()
    A.pw = args
    A.subs_table = sched.table.data_ptr()
    A.steps = desc.ctypes.data
    A.n_steps = n
    A.scheme = scheme
    A.tiles = 1 if tiles_ok else 0
    A.maybe_nonuniform = 1 if maybe else 0
    A.ess_gate = 1 if r0.ess_rel is not None else 0
    A.x_ring = 0 if r0.keep_history else x_arena.shape[0]
    A.a_ring = a_arena.shape[0] if a_arena is not None else 0
    A.x_in = x_prev.data_ptr()
    A.x_arena = x_arena.data_ptr()
    A.anc_arena = anc_arena.data_ptr() if anc_arena is not None else None
    A.a_prev = a_last.data_ptr() if a_last is not None else None
    A.a_arena = a_arena.data_ptr() if a_arena is not None else None
    A.cdf_local = cdf_local.data_ptr() if cdf_local is not None else None
    A.tile_rec = tile_rec.data_ptr() if tile_rec is not None else None
    A.resample_ws = rs_ws.data_ptr()
    A.anc_used = anc_used.ctypes.data
    A.y_table, A.u_table = sched.y_table.data_ptr(), sched.u_table.data_ptr()
    timer = profiling.active()
    evs = None
    coop = (tiles_ok and not _NO_COOP and not _NO_HINTS and scheme in (_lib.SCHEME_IDS["systematic"],
                                                                         _lib.SCHEME_IDS["stratified"])
            and spec.kernel != _lib.SSM_MODEL_GENERIC and B * P <= COOP_MAX_PARTICLES)
    if coop:  # the whole grid loop in one persistent cooperative launch
        steps_dev = C.c_void_p(sched.desc_dev.data_ptr() + (start + 1) * _lib.STEP_DESC_DTYPE.itemsize)
        with profiling.maybe("advance_coop", 0):
            st = L.ssm_advance_coop(A, steps_dev, stream)
        if st == _lib.SSM_ERR_UNSUPPORTED:
            coop = False
        else:
            _lib.check(st, "ssm_advance_coop")
    if not coop:
        if timer is not None:  # events around the sampled steps only (each one splits a PDL pair)
            evs = [profiling.NativeEvent() if timer.samples(start + 1 + k) else None for k in range(n) for _ in range(4)]
            ev_arr = (C.c_void_p * (4 * n))(*[e.h if e is not None else None for e in evs])
            A.events = C.cast(ev_arr, C.c_void_p)
        _lib.check(L.ssm_advance(A, stream), "ssm_advance")
        kind = "tiles" if tiles_ok else "logw"
        rs_n = _RS_LAUNCHES[(kind, scheme)]
        profiling.count_launch(n + rs_n * int(anc_used.sum()))
    ring = x_arena.shape[0]
    if evs is not None:
        for k in range(n):
            if evs[4 * k] is None:
                continue
            has_obs = bool(desc["has_obs"][k])
            if anc_used[k]:
                timer.add("resample", evs[4 * k], evs[4 * k + 1], int(B * P * _resample_bytes(esz)))
            nbytes = B * P * _pw_bytes(spec.nx, esz, bool(anc_used[k]), has_obs)
            timer.add("propagate_weight", evs[4 * k + 2], evs[4 * k + 3], nbytes)
    a_new = a_arena[A.a_last_index] if A.a_last_index >= 0 else a_last
    new_hist.update(anc=anc_arena, used=anc_used.astype(bool))
    return x_arena[(n - 1) % ring], a_new, bool(A.maybe_nonuniform)


_SMALL_MAX = None
_NO_SMALL = bool(os.environ.get("SSM_NO_SMALL"))  # A/B switch: force the multi-kernel path


def _small_max():
    global _SMALL_MAX
    if _SMALL_MAX is None:
        _SMALL_MAX = int(_lib.lib().ssm_small_max_particles())
    return _SMALL_MAX


def _advance_small(L, r0, B, P, spec, sched, start, upto, args, x_prev, a_last, maybe, x_arena, new_hist, stream):
    """All steps of all B filters in ONE persistent launch (P <= ssm_small_max_particles())."""
    n = upto - start
    dev = x_arena.device
    anc_arena = torch.empty((n, B, P), dtype=torch.int32, device=dev)
    any_obs = any(sched.obs[i] is not None for i in range(start + 1, upto + 1))
    a_out = torch.empty((B, P), dtype=r0.tdtype, device=dev) if (any_obs or a_last is not None) else None
    S = _lib.SmallArgs()
    S.model, S.dtype, S.B, S.P = spec.kernel, r0.dtype_id, B, P
    S.scheme = _lib.SCHEME_IDS[r0.resampler]
    S.exact, S.check_finite, S.n_steps = int(r0.exact), int(r0.check_finite), n
    S.log_w0, S.obs_log_sd, S.log_sqrt_2pi, S.ess_rel = args.log_w0, args.obs_log_sd, args.log_sqrt_2pi, args.ess_rel
    S.theta, S.keys, S.fs = args.theta, args.keys, args.fs
    S.subs = sched.table.data_ptr()
    S.steps = sched.desc_dev.data_ptr() + (start + 1) * _lib.STEP_DESC_DTYPE.itemsize
    S.x_in, S.x_arena, S.anc_arena = x_prev.data_ptr(), x_arena.data_ptr(), anc_arena.data_ptr()
    S.a_prev = a_last.data_ptr() if a_last is not None else None
    S.a_out = a_out.data_ptr() if a_out is not None else None
    with profiling.maybe("small_filter", 0):
        _lib.check(L.ssm_advance_small(S, stream), "ssm_advance_small")
    new_hist.update(anc=anc_arena, used=np.ones(n, dtype=bool))
    for k in range(n):
        i = start + 1 + k
        if sched.obs[i] is not None:
            maybe = True
        elif maybe and r0.ess_rel is None:
            maybe = False
    return x_arena[n - 1], (a_out if a_out is not None else a_last), maybe


def args_device(t):
    return t.device


def advance_runs(runs, upto, rngs):
    """Advance a batch of runs (same model, grid, P, settings, position)
    through grid index `upto`; returns the per-run loglik increments
    (particle.py:87-94).  Raises the reference's exceptions on failure."""
    r0 = _common(runs)
    start = r0.pos
    if upto <= start:
        for r in runs:
            r.pos = max(r.pos, upto)
        return np.zeros(len(runs))
    L = _lib.lib()
    B, P, spec = len(runs), r0.n_particles, r0.spec
    dev, tdt = r0.device, r0.tdtype
    sched = _schedule(r0.grid, spec, r0.inputs, dev)
    stream = _lib.stream_ptr()
    # the runs' rows of every per-filter tensor, gathered with one shared index upload
    names = ["_x", "_fs"] + (["_a"] if _has_row(r0, "_a") else [])
    if all(_has_row(r, "_cdf") for r in runs):
        names += ["_cdf", "_trec"]
    got = _rows_many(runs, names)
    x_prev = got["_x"]
    a_last = got.get("_a")
    fs = got["_fs"].clone()  # fresh copy: clones stay untouched
    theta = _derived_tensor(runs)
    maybe_nonuniform = r0._maybe_nonuniform
    host_noise = r0.noise == "host"
    keys_t = None
    if not host_noise:
        keys = device_keys(rngs)
        keys_t = _lib.h2d(keys.view(np.int32), dev)
    scheme = _lib.SCHEME_IDS[r0.resampler]
    if scheme == 0 and not host_noise:
        # device multinomial as sorted order statistics (exponential spacings):
        # the same law, ancestors ascending so the next gather streams
        scheme = _lib.SSM_MULTINOMIAL_SORTED
    pw_ws = torch.empty(L.ssm_pw_workspace_bytes(B, P), dtype=torch.uint8, device=dev)
    rs_ws = torch.empty(L.ssm_resample_workspace_bytes(B, P), dtype=torch.uint8, device=dev)
    # systematic / stratified resample from the pw kernel's tile-local CDF (no second pass over logw)
    small = (not host_noise and P <= _small_max() and not _NO_SMALL and r0.keep_history
             and spec.kernel != _lib.SSM_MODEL_GENERIC)
    # resample from the pw kernel's tile CDF (multi-kernel path; multinomial with device draws only)
    tiles_ok = (r0.resampler in ("systematic", "stratified") or scheme == _lib.SSM_MULTINOMIAL_SORTED) and not small
    ntile = (P + 31) // 32  # one tile record per warp tile
    cdf_local = tile_rec = None
    if tiles_ok:
        have = [_has_row(r, "_cdf") for r in runs]
        if all(have):  # resume: fresh copies, clones sharing the views stay intact
            cdf_local = got["_cdf"].clone()
            tile_rec = got["_trec"].clone()
        else:
            cdf_local = torch.empty((B, P), dtype=torch.int64, device=dev)
            tile_rec = torch.empty((B, ntile, 2), dtype=torch.float64, device=dev)
            for b, r in enumerate(runs):
                if have[b]:  # mixed batch: keep every carried CDF
                    cdf_local[b].copy_(r._cdf)
                    tile_rec[b].copy_(r._trec)
                elif not r.weights_uniform:
                    # the next step resamples from this run's tile CDF: it must travel with the run
                    raise RuntimeError("weighted run without its tile CDF (cdf_local / tile_rec) cannot resume")
    ess_rel = -1.0 if r0.ess_rel is None else float(r0.ess_rel)
    log_w0 = float(-np.log(P))
    obs_log_sd = float(np.log(spec.obs_sd))
    new_hist = {}  # the call's ancestor arena [n, B, P] and which steps resampled (used[k])
    esz = 8 if r0.dtype_id == _lib.SSM_F64 else 4
    theta_host = theta.cpu().numpy() if host_noise else None

    args = _lib.PwArgs()
    args.model = spec.kernel
    args.dtype = r0.dtype_id
    args.B, args.P = B, P
    args.exact = 1 if r0.exact else 0
    args.check_finite = 1 if r0.check_finite else 0
    args.log_w0 = log_w0
    args.obs_log_sd = obs_log_sd
    args.log_sqrt_2pi = float(LOG_SQRT_2PI)
    args.ess_rel = ess_rel
    args.theta = theta.data_ptr()
    if spec.kernel == _lib.SSM_MODEL_GENERIC:
        args.gen = spec.handle(dev)
        args.theta_stride = spec.theta_stride
    args.keys = keys_t.data_ptr() if keys_t is not None else None
    args.fs = fs.data_ptr()
    args.workspace = pw_ws.data_ptr()

    # one allocation per advance call for the history it produces (the caching
    # allocator would otherwise churn cudaMalloc on every step)
    n_steps = upto - start
    # history-free runs keep two position buffers (ring) instead of one per step
    x_slots = n_steps if r0.keep_history else min(n_steps, 2)
    x_arena = torch.empty((x_slots, B, spec.nx, P), dtype=tdt, device=dev)
    n_res = sum(1 for i in range(start + 1, upto + 1) if sched.obs[i] is not None)
    # log-weights: the native driver keeps a ring of two (the step reads the previous
    # weighted step's, later only the last one is used); host-noise loop: one per step
    a_slots = min(n_res, 2) if not host_noise else n_res
    a_arena = torch.empty((max(a_slots, 1), B, P), dtype=tdt, device=dev) if n_res else None
    anc_arena = None
    host_used = None
    a_slot = 0
    if small:  # the persistent kernel keeps its CDF in shared memory
        x_prev, a_last, maybe_nonuniform = _advance_small(
            L, r0, B, P, spec, sched, start, upto, args, x_prev, a_last, maybe_nonuniform, x_arena, new_hist, stream)
    elif not host_noise:
        x_prev, a_last, maybe_nonuniform = _advance_native(
            L, r0, B, P, spec, sched, start, upto, args, x_prev, a_last, maybe_nonuniform, x_arena, a_arena,
            cdf_local, tile_rec, rs_ws, tiles_ok, scheme, esz, new_hist, stream)
    for i in (range(start + 1, upto + 1) if host_noise else ()):
        step_rngs = [g.child(i) for g in rngs] if host_noise else None
        anc = None
        if maybe_nonuniform:
            if anc_arena is None:
                anc_arena = torch.empty((upto - start, B, P), dtype=torch.int32, device=dev)
                host_used = np.zeros(upto - start, dtype=bool)
            anc = anc_arena[i - start - 1]
            host_used[i - start - 1] = True
            u_t = None
            if host_noise:
                rr = [s.child(_RESAMPLE_KEY) for s in step_rngs]
                if r0.resampler == "systematic":
                    u = np.array([[g.uniform()] for g in rr])
                else:
                    u = np.stack([g.uniform(size=P) for g in rr])
                u_t = torch.from_numpy(u).to(dev)
            if tiles_ok:
                with profiling.maybe("resample", int(B * P * _resample_bytes(esz))):
                    _lib.check(L.ssm_resample_from_tiles(B, P, scheme, _lib.ptr(cdf_local), _lib.ptr(tile_rec),
                                                         _lib.ptr(fs), _lib.ptr(u_t), _lib.ptr(keys_t), i,
                                                         _lib.ptr(anc), _lib.ptr(rs_ws), stream),
                               "ssm_resample_from_tiles")
            else:
                with profiling.maybe("resample", int(B * P * _resample_bytes(esz))):
                    _lib.check(L.ssm_resample_from_logw(B, P, r0.dtype_id, scheme, _lib.ptr(a_last), None,
                                                        _lib.ptr(fs), _lib.ptr(u_t), _lib.ptr(keys_t), i,
                                                        _lib.ptr(anc), _lib.ptr(rs_ws), stream),
                               "ssm_resample_from_logw")
        n_sub = sched.n_sub[i]
        x_out = x_arena[i - start - 1]
        noise_t = None
        if host_noise:
            noise = np.stack([spec.host_noise(s.child(_PROPAGATE_KEY), sched.host_subs[i], P, theta_row)
                              for s, theta_row in zip(step_rngs, theta_host)])
            noise_t = torch.from_numpy(noise).to(dev, tdt)
        obs = sched.obs[i]
        a_out = None
        if obs is not None:
            a_out = a_arena[a_slot]
            a_slot += 1
        args.step = i
        args.n_sub = n_sub
        args.hints = _lib.SSM_HINT_SINGLE_SUBSTEP if (sched.single[i] and not _NO_HINTS) else 0
        args.subs = sched.subs_ptr(i)
        args.y_vec, args.u_vec = sched.y_ptr(i), sched.u_ptr(i)
        args.x_in = x_prev.data_ptr()
        args.x_out = x_out.data_ptr()
        args.anc = anc.data_ptr() if anc is not None else None
        args.a_prev = a_last.data_ptr() if a_last is not None else None
        args.a_out = a_out.data_ptr() if a_out is not None else None
        args.noise = noise_t.data_ptr() if noise_t is not None else None
        args.cdf_local = cdf_local.data_ptr() if (tiles_ok and obs is not None) else None
        args.tile_rec = tile_rec.data_ptr() if (tiles_ok and obs is not None) else None
        if obs is not None:
            args.has_obs = 1
            args.obs_mask = obs[0]
            for n in range(8):
                args.y[n] = float(obs[1][n])
            args.u_obs = obs[2]
        else:
            args.has_obs = 0
            args.obs_mask = 0
        nbytes = B * P * _pw_bytes(spec.nx, esz, anc is not None, obs is not None)
        with profiling.maybe("propagate_weight", nbytes):
            _lib.check(L.ssm_propagate_weight(args, stream), "ssm_propagate_weight")
        x_prev = x_out
        if obs is not None:
            a_last = a_out
            maybe_nonuniform = True
        elif maybe_nonuniform and r0.ess_rel is None:
            maybe_nonuniform = False

    xstride = spec.nx * P * esz
    astride = P * 4
    fs_host = _fs_view(fs)  # one synchronisation per advance
    if ((fs_host["err_nonfinite"] != _lib.INT32_MAX).any() or (fs_host["err_degenerate"] != _lib.INT32_MAX).any()
            or (fs_host["err_param"] != _lib.INT32_MAX).any()):
        for b, r in enumerate(runs):
            _raise_if_failed(fs_host[b], sched, r.check_finite)
    ll = fs_host["loglik"].astype(float)
    unif = fs_host["uniform"].astype(bool)
    incr = ll - np.array([r.loglik for r in runs])
    # the call's history segment; per-step base pointers once, each run's rows at a fixed stride
    if host_noise:
        new_hist.update(anc=anc_arena, used=host_used if host_used is not None else np.zeros(n_steps, bool))
    anc_t, used = new_hist.get("anc"), new_hist.get("used")
    seg = _Seg(x_arena if r0.keep_history else None, anc_t, used, n_steps)
    ks = np.arange(n_steps, dtype=np.int64)
    x_ptrs = x_arena.data_ptr() + ks * (B * xstride) if r0.keep_history else np.zeros(n_steps, np.int64)
    a_ptrs = np.where(used, anc_t.data_ptr() + ks * (B * astride), 0) if anc_t is not None else np.zeros(n_steps, np.int64)
    a_has = a_ptrs != 0
    has_a = a_last is not None
    keep_tiles = tiles_ok and has_a
    # the pointer arrays of all B runs in one [B, pos + 1 + n] block each (every run is
    # at the same position), each run keeping its row: O(1) numpy calls per advance
    rows_b = np.arange(B, dtype=np.int64)[:, None]
    new_hx = x_ptrs[None, :] + rows_b * xstride if r0.keep_history else np.broadcast_to(x_ptrs, (B, n_steps))
    new_ha = np.where(a_has[None, :], a_ptrs[None, :] + rows_b * astride, 0)
    all_hx = np.concatenate([_np_rows(runs, "_hx"), new_hx], axis=1)
    all_ha = np.concatenate([_np_rows(runs, "_ha"), new_ha], axis=1)
    all_kk = None
    if not r0.keep_history:  # ancestors only; positions are replayed by sample_trajectories
        new_kk = np.repeat(keys.astype(np.uint32)[:, None, :], n_steps, axis=1)
        all_kk = np.concatenate([_np_rows(runs, "_kk"), new_kk], axis=1)
    for b, r in enumerate(runs):
        d = r.__dict__
        d["loglik"] = float(ll[b])
        d["weights_uniform"] = bool(unif[b])
        d["_rb_x"] = (x_prev, b)
        d["_rb_a"] = (a_last, b) if has_a else None
        d["_rb_cdf"] = (cdf_local, b) if keep_tiles else None
        d["_rb_trec"] = (tile_rec, b) if keep_tiles else None
        d["_rb_fs"] = (fs, b)
        d["_maybe_nonuniform"] = maybe_nonuniform
        d["_segs"] = d["_segs"] + [(seg, b)]
        d["_nb_hx"] = (all_hx, b)
        d["_nb_ha"] = (all_ha, b)
        if all_kk is not None:
            d["_nb_kk"] = (all_kk, b)
        d["pos"] = upto
    return incr




def _raise_if_failed(st, sched, check_finite):
    nf = int(st["err_nonfinite"])
    dg = int(st["err_degenerate"])
    pe = int(st["err_param"])
    if pe != _lib.INT32_MAX and (nf == _lib.INT32_MAX or pe <= nf) and (dg == _lib.INT32_MAX or pe // 64 <= dg):
        step, sub = pe // 64, pe % 64
        where = "observation density" if sub == 63 else "transition"
        raise DistributionParameterError(f"invalid distribution argument in the {where} at grid index {step}")
    if nf == _lib.INT32_MAX and dg == _lib.INT32_MAX:
        return
    nf_step = nf // 64 if nf != _lib.INT32_MAX else None
    if nf_step is not None and (dg == _lib.INT32_MAX or nf_step <= dg) and check_finite:
        t = sched.sub_end[nf_step][nf % 64]
        raise NonFiniteStateError(f"non-finite state after transition sub-step ending at t={t:g}", time=t)
    if dg != _lib.INT32_MAX:
        t = float(sched.times[dg])
        raise DegenerateEnsembleError(f"all particle weights vanished at t={t:g}", time=t)


def sample_trajectories(runs, rngs):
    """ParticleRun.sample_trajectory for a batch (particle.py:137-149): one
    multinomial draw by final weight (host uniform, the reference's draw),
    device CDF + search, then a device ancestry trace."""
    r0 = runs[0]
    L = _lib.lib()
    B, P, nx = len(runs), r0.n_particles, r0.spec.nx
    dev = r0.device
    S = r0.pos
    stream = _lib.stream_ptr()
    if all(not r.weights_uniform and _has_row(r, "_cdf") and _has_row(r, "_trec") for r in runs):
        # final weights carry the fused kernel's tile records: one warp search per filter
        u = _lib.h2d(first_uniforms(rngs, 1)[:, 0].copy(), dev)
        j = torch.empty((B, 1), dtype=torch.int32, device=dev)
        ws = torch.empty(L.ssm_resample_workspace_bytes(B, P), dtype=torch.uint8, device=dev)
        cdf = _rows(runs, "_cdf").contiguous()
        trec = _rows(runs, "_trec").contiguous()
        fs_rows = _rows(runs, "_fs").contiguous()
        _lib.check(L.ssm_pick_from_tiles(B, P, _lib.ptr(cdf), _lib.ptr(trec), _lib.ptr(fs_rows), _lib.ptr(u),
                                         _lib.ptr(j), _lib.ptr(ws), stream), "ssm_pick_from_tiles")
        return _trajectories_from(L, runs, j, S, B, P, nx, dev, stream)
    # final log-weights (uniform -> zeros with shift log P, so the scan's
    # precondition sum(exp(a - shift)) = 1 holds: w_j = 1/P as the reference's
    # exp(logw) with logw = -log P, particle.py:139)
    a_rows, shifts = [], []
    for r in runs:
        if r.weights_uniform or r._a is None:
            a_rows.append(_zeros_logw(P, r0.tdtype, dev)[0])
            shifts.append(None)
        else:
            a_rows.append(r._a)
            shifts.append(r._fs)
    a = _stack_rows(a_rows)
    log_p = math.log(P)
    if all(f is None for f in shifts):
        shift = torch.full((B,), log_p, dtype=torch.float64, device=dev)
    else:  # ssm_filter_state.incr (bytes 8..16) of weighted runs, log P for uniform ones
        fs_rows = _rows(runs, "_fs").contiguous()
        incr = fs_rows.view(torch.float64)[:, 1]
        weighted = _lib.h2d(np.array([f is not None for f in shifts]), dev)
        shift = torch.where(weighted, incr, torch.full_like(incr, log_p))
    scan_ws = torch.empty(L.ssm_scan_workspace_bytes(B, P), dtype=torch.uint8, device=dev)
    cum = torch.empty((B, P), dtype=torch.int64, device=dev)
    flags = torch.zeros(B, dtype=torch.int32, device=dev)
    _lib.check(L.ssm_weights_scan(B, P, r0.dtype_id, _lib.ptr(a), 1, _lib.ptr(shift), None, _lib.ptr(cum),
                                  _lib.ptr(flags), _lib.ptr(scan_ws), stream), "ssm_weights_scan")
    u = _lib.h2d(first_uniforms(rngs, 1), dev)  # each stream's uniform(size=1)
    j = torch.empty((B, 1), dtype=torch.int32, device=dev)
    _lib.check(L.ssm_resample_search(B, P, 1, _lib.SCHEME_IDS["multinomial"], 1, _lib.ptr(cum), _lib.ptr(u),
                                     None, 0, None, _lib.ptr(j), None, stream), "ssm_resample_search")
    out = _trajectories_from(L, runs, j, S, B, P, nx, dev, stream)
    if int(flags.max().item()) & _lib.SSM_FLAG_UNNORMALISED:  # after the read-back: no extra sync
        raise ValueError("final weights violate the CDF normalisation precondition (ssm_weights_scan)")
    return out


def _trajectories_from(L, runs, j, S, B, P, nx, dev, stream):
    if runs[0].keep_history:
        return _trace_runs(L, runs, j, S, B, P, nx, dev, stream)
    return _replay_runs(L, runs, j, S, B, P, nx, dev, stream)


def _replay_runs(L, runs, j, S, B, P, nx, dev, stream):
    """History-free runs: regenerate the chosen ancestral line (ssm_replay_path)."""
    r0 = runs[0]
    for r in runs:
        if len(r._kk) != S + 1 or len(r._ha) != S + 1:
            raise ValueError("history length does not match the run position")
    sched = _schedule(r0.grid, r0.spec, r0.inputs, dev)
    desc = np.ascontiguousarray(sched.desc[: S + 1]).copy()
    if _NO_HINTS:
        desc["hints"] = 0
    desc_t = _lib.h2d(desc.view(np.uint8), dev)
    keys_t = _lib.h2d(np.ascontiguousarray(_np_rows(runs, "_kk").astype(np.uint32)).view(np.int32), dev)
    ancs_t = _lib.h2d(np.ascontiguousarray(_np_rows(runs, "_ha")), dev)
    theta = _derived_tensor(runs)
    fixed = [r.initial_state is not None for r in runs]
    x0_t = flag_t = None
    if any(fixed):
        x0 = np.zeros((B, nx))
        for b, r in enumerate(runs):
            if fixed[b]:
                x0[b] = np.asarray(r.initial_state, dtype=float)
        x0_t = _lib.h2d(x0, dev)
        flag_t = _lib.h2d(np.asarray(fixed, dtype=np.int32), dev)
    out = torch.empty((B, S + 1, nx), dtype=torch.float64, device=dev)
    R = _lib.ReplayArgs()
    R.model, R.dtype, R.B, R.P, R.S, R.exact = r0.spec.kernel, r0.dtype_id, B, P, S, int(r0.exact)
    R.theta, R.subs, R.steps = theta.data_ptr(), sched.table.data_ptr(), desc_t.data_ptr()
    R.keys, R.ancs, R.j_final, R.out = keys_t.data_ptr(), ancs_t.data_ptr(), j.data_ptr(), out.data_ptr()
    R.x0 = x0_t.data_ptr() if x0_t is not None else None
    R.x0_flag = flag_t.data_ptr() if flag_t is not None else None
    _lib.check(L.ssm_replay_path(R, stream), "ssm_replay_path")
    return list(out.cpu().numpy())


def _trace_runs(L, runs, j, S, B, P, nx, dev, stream):
    """Ancestry walk from the picked final particles j (device) -> trajectories."""
    r0 = runs[0]
    xs = _np_rows(runs, "_hx")
    ancs = _np_rows(runs, "_ha")
    if xs.shape[1] != S + 1:
        raise ValueError("history length does not match the run position")
    xs_t = _lib.h2d(xs, dev)
    ancs_t = _lib.h2d(ancs, dev)
    out = torch.empty((B, S + 1, nx), dtype=torch.float64, device=dev)
    _lib.check(L.ssm_trace(r0.dtype_id, B, S, nx, P, _lib.ptr(xs_t), _lib.ptr(ancs_t), _lib.ptr(j),
                           _lib.ptr(out), stream), "ssm_trace")
    return list(out.cpu().numpy())


def particle_filter(ir, theta, grid, rng, inputs=None, n_particles=1024, resampler="multinomial",
                    ess_rel=None, initial_state=None, check_finite=True, upto=None, **device_opts):
    """particle.py:156-185 on the GPU: init(child 0) -> advance(child 1) ->
    sample_trajectory(child 2).  device_opts: dtype, exact, noise, device."""
    run = ParticleRun(ir, theta, grid, inputs=inputs, n_particles=n_particles, resampler=resampler,
                      ess_rel=ess_rel, initial_state=initial_state, check_finite=check_finite,
                      **device_opts)
    run.init(rng.child(0))
    run.advance_to(run.grid.last if upto is None else upto, rng.child(1))
    trajectory = run.sample_trajectory(rng.child(2))
    return FilterOutcome(loglik=run.loglik, trajectory=trajectory, summaries=[], run=run)

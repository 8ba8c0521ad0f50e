"""One bootstrap particle filter sharded across GPUs (BASELINE config 5,
SURVEY 8e): rank r holds particles [r*P_loc, (r+1)*P_loc) of a P_global
filter; propagation and weighting are rank-local.  Per weighted step:

  C1  all-gather of the per-rank LSE/ESS partials (4 doubles) -> every rank
      runs the same combine kernel (global increment, loglik, ESS gate);
  C1' all-gather of the per-rank fixed-point CDF totals -> global offsets;
      global offspring bounds of the local particles (systematic /
      stratified on global query indices);
  C3  all-gather of (first owned output, count) and point-to-point transfer of
      the ancestor states whose output slot lives on another rank (only the
      load imbalance moves; sorted ancestors make it neighbour traffic).

All draws use global particle indices, so the filter is the same for any
rank count (up to the association of the LSE partials).  The ancestry of
the trajectory sample crosses ranks; it is walked with one broadcast per
grid step.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from .. import _lib, profiling
from ..distributed import Shard, exchange
from ..errors import DegenerateEnsembleError, NonFiniteStateError
from ..models import LOG_SQRT_2PI, resolve_model
from ..rng import device_key
from .particle import _dtype_info, _fs_init, _fs_view, _schedule
from .timegrid import as_filter_grid


def _allgather_tensor(t, shard):
    """All-gather a small device tensor (rank order); host-staged for gloo."""
    if shard.world == 1:
        return t.unsqueeze(0)
    if shard.backend == "nccl":
        out = [torch.empty_like(t) for _ in range(shard.world)]
        dist.all_gather(out, t.contiguous(), group=shard.group)
        return torch.stack(out)
    out = [torch.empty_like(t, device="cpu") for _ in range(shard.world)]
    dist.all_gather(out, t.detach().cpu().contiguous(), group=shard.group)
    return torch.stack(out).to(t.device)


class ShardedParticleFilter:
    def __init__(self, ir, theta, grid, n_particles, resampler="systematic", inputs=None, ess_rel=None,
                 check_finite=True, *, dtype="float64", exact=False, shard=None, device=None):
        if resampler not in ("systematic", "stratified"):
            raise ValueError("the sharded filter supports systematic and stratified resampling")
        if ess_rel is not None:
            raise ValueError("the sharded filter resamples every weighted step (ess_rel must be None)")
        _lib.require_cuda()
        self.shard = shard or Shard.current()
        W = self.shard.world
        if n_particles % W:
            raise ValueError("n_particles must be divisible by the number of ranks")
        self.spec = resolve_model(ir)
        self.theta = np.asarray(theta, dtype=float).reshape(1, -1)
        self.grid = as_filter_grid(grid)
        self.inputs = inputs
        self.P = int(n_particles)
        self.P_loc = self.P // W
        self.resampler = resampler
        self.ess_rel = ess_rel
        self.check_finite = check_finite
        self.dtype_name, self.tdtype, self.dtype_id = _dtype_info(dtype)
        self.exact = bool(exact)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.loglik = 0.0
        self.spill_cap = 0 if self.shard.world == 1 else max(1024, self.P_loc // 8)

    def run(self, rng, upto=None):
        """particle_filter(...) semantics: init(child 0), advance(child 1),
        trajectory(child 2).  Returns (loglik, trajectory) on every rank."""
        L = _lib.lib()
        sh, W, r = self.shard, self.shard.world, self.shard.rank
        spec, P, Pl, dev, tdt = self.spec, self.P, self.P_loc, self.device, self.tdtype
        upto = self.grid.last if upto is None else upto
        sched = _schedule(self.grid, spec, self.inputs, dev)
        stream = _lib.stream_ptr()
        off = r * Pl
        keys0 = torch.from_numpy(device_key(rng.child(0)).astype(np.uint32).reshape(1, 2).view(np.int32)).to(dev)
        keys1 = torch.from_numpy(device_key(rng.child(1)).astype(np.uint32).reshape(1, 2).view(np.int32)).to(dev)
        # every position buffer has `cap` spare columns: ancestor states received
        # from other ranks land there, so resampling never copies the local state
        cap = self.spill_cap
        xbuf = torch.empty((spec.nx, Pl + cap), dtype=tdt, device=dev)
        x0 = torch.empty((spec.nx, Pl), dtype=tdt, device=dev)
        theta = torch.from_numpy(spec.derived(self.theta)).to(dev)
        generic = spec.kernel == _lib.SSM_MODEL_GENERIC
        if generic:  # the model's initial block, global particle indices (the draws match one process)
            _lib.check(L.ssm_gen_init_particles(C.c_void_p(spec.handle(dev)), self.dtype_id, 1, Pl, off,
                                                _lib.ptr(keys0), _lib.ptr(theta), spec.theta_stride, _lib.ptr(x0),
                                                None, stream), "ssm_gen_init_particles")
        else:
            _lib.check(L.ssm_init_particles(spec.kernel, self.dtype_id, 1, Pl, off, _lib.ptr(keys0), _lib.ptr(x0),
                                            stream), "ssm_init_particles")
        xbuf[:, :Pl] = x0
        x = xbuf[:, :Pl]
        fs = _fs_init(1, dev)
        pw_ws = torch.empty(L.ssm_pw_workspace_bytes(1, Pl), dtype=torch.uint8, device=dev)
        sw = torch.empty(L.ssm_sharded_workspace_bytes(1, Pl, P), dtype=torch.uint8, device=dev)
        cdf = torch.empty(Pl, dtype=torch.int64, device=dev)
        trec = torch.empty(((Pl + 31) // 32, 2), dtype=torch.float64, device=dev)
        lse_part = torch.empty(4, dtype=torch.float64, device=dev)
        tot = torch.empty(1, dtype=torch.int64, device=dev)
        shift = torch.empty(1, dtype=torch.int32, device=dev)
        c_last = torch.empty(1, dtype=torch.int32, device=dev)
        scheme = _lib.SCHEME_IDS[self.resampler]
        ess_rel = -1.0 if self.ess_rel is None else float(self.ess_rel)

        A = _lib.PwArgs()
        A.model, A.dtype, A.B, A.P = spec.kernel, self.dtype_id, 1, Pl
        A.exact, A.check_finite = int(self.exact), int(self.check_finite)
        A.log_w0 = float(-np.log(P))
        A.obs_log_sd = float(np.log(spec.obs_sd))
        A.log_sqrt_2pi = float(LOG_SQRT_2PI)
        A.ess_rel = ess_rel
        A.theta, A.keys, A.fs, A.workspace = theta.data_ptr(), keys1.data_ptr(), fs.data_ptr(), pw_ws.data_ptr()
        A.p_offset = off
        if generic:
            A.gen, A.theta_stride = spec.handle(dev), spec.theta_stride

        hist = [(x, None)]  # (x_i [nx, Pl], global ancestor index [Pl] int64 | None)
        a_last = None
        maybe = False
        x_prev, xbuf_prev = x, xbuf
        for i in range(1, upto + 1):
            anc = gidx = None
            x_in, stride = x_prev, 0
            if maybe:
                with profiling.maybe("resample", Pl * (8 + 4 + 4 + 4)):
                    x_in, stride, anc, gidx = self._resample(L, i, x_prev, xbuf_prev, a_last, fs, cdf, trec, tot,
                                                             shift, c_last, sw, keys1, scheme, stream)
            obs = sched.obs[i]
            xbuf_out = torch.empty((spec.nx, Pl + cap), dtype=tdt, device=dev)
            x_out = xbuf_out[:, :Pl]
            a_out = torch.empty(Pl, dtype=tdt, device=dev) if obs is not None else None
            A.step, A.n_sub = i, sched.n_sub[i]
            A.hints = _lib.SSM_HINT_SINGLE_SUBSTEP if sched.single[i] else 0
            A.subs = sched.subs_ptr(i)
            A.y_vec, A.u_vec = sched.y_ptr(i), sched.u_ptr(i)
            A.x_in, A.x_in_stride = x_in.data_ptr(), (stride if stride else Pl + cap)
            A.x_out, A.x_out_stride = x_out.data_ptr(), Pl + cap
            A.anc = anc.data_ptr() if anc is not None else None
            A.a_prev = a_last.data_ptr() if a_last is not None else None
            A.a_out = a_out.data_ptr() if a_out is not None else None
            A.cdf_local = cdf.data_ptr() if obs is not None else None
            A.tile_rec = trec.data_ptr() if obs is not None else None
            A.lse_out = lse_part.data_ptr() if obs is not None else None
            if obs is not None:
                A.has_obs, A.obs_mask, A.u_obs = 1, obs[0], obs[2]
                for n in range(8):
                    A.y[n] = float(obs[1][n])
            else:
                A.has_obs, A.obs_mask = 0, 0
            esz = 8 if self.dtype_id == _lib.SSM_F64 else 4
            nbytes = Pl * (2 * spec.nx * esz + (4 if anc is not None else 0) + ((esz + 8) if obs is not None else 0))
            with profiling.maybe("propagate_weight", nbytes):
                _lib.check(L.ssm_propagate_weight(A, stream), "ssm_propagate_weight")
            if obs is not None:
                parts = _allgather_tensor(lse_part, sh)  # C1
                _lib.check(L.ssm_lse_combine(W, 1, _lib.ptr(parts), _lib.ptr(fs), ess_rel, float(P), i, stream),
                           "ssm_lse_combine")
                a_last = a_out
                maybe = True
            elif maybe and self.ess_rel is None:
                maybe = False
            hist.append((x_out, gidx))
            x_prev, xbuf_prev = x_out, xbuf_out
        st = _fs_view(fs)[0]
        nf, dg = int(st["err_nonfinite"]), int(st["err_degenerate"])
        if self.check_finite and nf != _lib.INT32_MAX and (dg == _lib.INT32_MAX or nf // 64 <= dg):
            t = sched.sub_end[nf // 64][nf % 64]
            raise NonFiniteStateError(f"non-finite state after transition sub-step ending at t={t:g}", time=t)
        if dg != _lib.INT32_MAX:
            t = float(sched.times[dg])
            raise DegenerateEnsembleError(f"all particle weights vanished at t={t:g}", time=t)
        self.loglik = float(st["loglik"])
        traj = self._trajectory(L, rng.child(2), hist, a_last, fs, stream)
        return self.loglik, traj

    # -- resampling across ranks ------------------------------------------------
    def _resample(self, L, i, x_prev, xbuf, a_last, fs, cdf, trec, tot, shift, c_last, sw, keys, scheme, stream):
        sh, W, r = self.shard, self.shard.world, self.shard.rank
        P, Pl, dev, nx = self.P, self.P_loc, self.device, self.spec.nx
        _lib.check(L.ssm_tiles_total(1, Pl, _lib.ptr(trec), _lib.ptr(fs), _lib.ptr(tot), _lib.ptr(sw), stream),
                   "ssm_tiles_total")
        tots = _allgather_tensor(tot, sh).reshape(W)  # C1': per-rank fixed-point totals
        csum = torch.cumsum(tots, 0)
        g_off = (csum[r] - tots[r]).reshape(1).contiguous()
        g_tot = csum[W - 1].reshape(1).contiguous()
        _lib.check(L.ssm_offspring_global(1, Pl, P, scheme, _lib.ptr(cdf), _lib.ptr(g_off), _lib.ptr(g_tot), None,
                                          _lib.ptr(keys), i, _lib.ptr(fs), _lib.ptr(shift), _lib.ptr(c_last),
                                          _lib.ptr(sw), stream), "ssm_offspring_global")
        mine = torch.stack([shift.to(torch.int64), c_last.to(torch.int64)]).reshape(2)
        owned = _allgather_tensor(mine, sh).cpu().numpy().reshape(W, 2)  # (first output, count) per rank
        A0, n_own = int(owned[r, 0]), int(owned[r, 1])
        anc_own = torch.empty(max(n_own, 1), dtype=torch.int32, device=dev)
        _lib.check(L.ssm_expand_own(1, Pl, P, n_own, _lib.ptr(fs), _lib.ptr(anc_own), _lib.ptr(sw), stream),
                   "ssm_expand_own")
        # plan: my outputs [A0, A0 + n_own) -> slots of rank d = [d*Pl, (d+1)*Pl)
        anc_final = torch.empty(Pl, dtype=torch.int32, device=dev)
        gidx = torch.empty(Pl, dtype=torch.int64, device=dev)
        sends, specs, recv_slots = {}, {}, []
        for d in range(W):
            lo, hi = max(A0, d * Pl), min(A0 + n_own, (d + 1) * Pl)
            if lo >= hi:
                continue
            seg = anc_own[lo - A0: hi - A0]
            if d == r:
                anc_final[lo - d * Pl: hi - d * Pl] = seg
                gidx[lo - d * Pl: hi - d * Pl] = seg.to(torch.int64) + r * Pl
            else:
                xs = torch.empty((nx, hi - lo), dtype=x_prev.dtype, device=dev)
                _lib.check(L.ssm_gather_cols(self.dtype_id, nx, hi - lo, xbuf.shape[1], _lib.ptr(xbuf), _lib.ptr(seg),
                                             _lib.ptr(xs), stream), "ssm_gather_cols")
                sends[d] = [xs, seg.to(torch.int64) + r * Pl]
        for s_ in range(W):
            if s_ == r:
                continue
            A_s, n_s = int(owned[s_, 0]), int(owned[s_, 1])
            lo, hi = max(A_s, r * Pl), min(A_s + n_s, (r + 1) * Pl)
            if lo < hi:
                specs[s_] = [((nx, hi - lo), x_prev.dtype), ((hi - lo,), torch.int64)]
                recv_slots.append((s_, lo - r * Pl, hi - lo))
        got = exchange(sends, specs, sh)  # C3
        if not recv_slots:
            return xbuf, xbuf.shape[1], anc_final, gidx
        R = sum(n for _, _, n in recv_slots)
        if R <= xbuf.shape[1] - Pl:
            x_ext = xbuf  # received states go to the spare columns: no copy of the local state
        else:  # spill larger than the capacity (degenerate weights): extend once
            x_ext = torch.empty((nx, Pl + R), dtype=x_prev.dtype, device=dev)
            x_ext[:, :Pl] = x_prev
        pos = Pl
        for s_, slot0, n in recv_slots:
            xs, gi = got[s_]
            x_ext[:, pos:pos + n] = xs.to(dev)
            anc_final[slot0:slot0 + n] = torch.arange(pos, pos + n, dtype=torch.int32, device=dev)
            gidx[slot0:slot0 + n] = gi.to(dev)
            pos += n
        return x_ext, x_ext.shape[1], anc_final, gidx

    # -- trajectory across ranks ------------------------------------------------
    def _trajectory(self, L, rng, hist, a_last, fs, stream):
        """sample_trajectory (particle.py:137-149): one multinomial draw on the
        global final weights (rank chosen by rank totals of exp(a - incr)),
        then the ancestry walk, one broadcast per grid step."""
        sh, W, r = self.shard, self.shard.world, self.shard.rank
        Pl, dev, nx = self.P_loc, self.device, self.spec.nx
        u = float(np.asarray(rng.uniform(size=1))[0])
        if a_last is None:
            jglob = min(int(u * self.P), self.P - 1)
        else:
            incr = float(_fs_view(fs)[0]["incr"])
            w = torch.exp(a_last.to(torch.float64) - incr)
            tots = _allgather_tensor(w.sum().reshape(1), sh).reshape(W).cpu().numpy()
            cum_r = np.cumsum(tots)
            target = u * cum_r[-1]
            owner = int(min(np.searchsorted(cum_r, target, side="right"), W - 1))
            jloc = 0
            if owner == r:
                cw = torch.cumsum(w, 0)
                t_loc = target - (cum_r[owner - 1] if owner > 0 else 0.0)
                jloc = int(min(torch.searchsorted(cw, torch.tensor([t_loc], dtype=torch.float64, device=dev),
                                                  right=True).item(), Pl - 1))
            jglob = int(self._bcast(np.array([float(owner * Pl + jloc)]), owner)[0])
        S = len(hist) - 1
        out = np.empty((S + 1, nx))
        j = jglob
        for i in range(S, -1, -1):
            owner = j // Pl
            vals = np.zeros(nx + 1)
            if owner == r:
                xi, gi = hist[i]
                jl = j - r * Pl
                vals[:nx] = xi[:, jl].to(torch.float64).cpu().numpy()
                vals[nx] = float(gi[jl].item()) if (i > 0 and gi is not None) else float(j)
            vals = self._bcast(vals, owner)
            out[i] = vals[:nx]
            j = int(vals[nx])
        return out

    def _bcast(self, vals, src):
        if self.shard.world == 1:
            return vals
        dev = torch.device("cuda", torch.cuda.current_device()) if self.shard.backend == "nccl" else torch.device("cpu")
        t = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64)).to(dev)
        dist.broadcast(t, src=src, group=self.shard.group)
        return t.cpu().numpy()


def particle_filter_sharded(ir, theta, grid, rng, n_particles, resampler="systematic", shard=None, **kw):
    """particle_filter over the ranks of `shard` (default torch.distributed)."""
    f = ShardedParticleFilter(ir, theta, grid, n_particles, resampler=resampler, shard=shard, **kw)
    return f.run(rng)

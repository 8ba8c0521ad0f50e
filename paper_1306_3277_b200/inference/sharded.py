"""One bootstrap particle filter sharded across GPUs (BASELINE config 5,
SURVEY 8e): rank r holds the particles [r*P_loc, (r+1)*P_loc) of a P_global
filter and owns the output slots of the same range.

Every rank maps every other rank's position and ancestor arenas into its own
address space once per run (CUDA IPC over NVLink peer memory,
`ssm_ipc_open`), so no particle state goes through the host and nothing
synchronises inside the grid loop.  Per weighted step:

  pw   the fused kernel gathers each ancestor from the rank that holds it
       (P2P loads, only at the rank boundaries: systematic / stratified
       ancestors are sorted) and writes the rank's LSE/ESS partial;
  C1   all-gather of the partials (4 doubles per rank) -> ssm_lse_combine:
       the same global increment, loglik and ESS gate on every rank;
  C1'  all-gather of the rank fixed-point weight totals -> global offsets;
  push ssm_offspring_push: global offspring counts of the local particles on
       global query indices, each ancestor stored straight into the array of
       the rank that owns the output slot (P2P stores at the boundaries);
  C2   rank barrier (the next gather reads ancestors other ranks wrote).

All draws use global particle indices, so the filter is the same for any
rank count (up to the association of the LSE partials); one rank is bitwise
`particle_filter`.  The trajectory is one multinomial pick on the global
weights (the owner rank's index, max over ranks) and one ancestry walk through
the peer-mapped arenas, identical on every rank.  With NCCL every collective
is stream-ordered on the device; with gloo (CPU tests, several processes on
one GPU) they are staged through the host.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from .. import _lib, profiling
from ..distributed import Shard
from ..errors import DegenerateEnsembleError, NonFiniteStateError, UnsupportedModelError
from ..models import LOG_SQRT_2PI, resolve_model
from ..rng import device_key
from .particle import _dtype_info, _fs_init, _fs_view, _pw_bytes, _resample_bytes, _schedule
from .timegrid import as_filter_grid


def _nccl(shard):
    return shard.world > 1 and shard.backend == "nccl"


def _allgather_tensor(t, shard):
    """All-gather a small device tensor in rank order -> [W, *t.shape] on t's device.
    NCCL: stream-ordered on the device (no host synchronisation); gloo: host-staged."""
    if shard.world == 1:
        return t.unsqueeze(0)
    if _nccl(shard):
        out = torch.empty((shard.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=shard.group)
        return out
    out = [torch.empty_like(t, device="cpu") for _ in range(shard.world)]
    dist.all_gather(out, t.detach().cpu().contiguous(), group=shard.group)
    return torch.stack(out).to(t.device)


def _barrier(shard, dev):
    """C2: every rank's peer stores are complete before any rank reads them."""
    if shard.world == 1:
        return
    if _nccl(shard):
        dist.all_reduce(torch.zeros(1, dtype=torch.int32, device=dev), group=shard.group)
    else:  # gloo orders host calls only: drain this rank's stream first
        torch.cuda.synchronize(dev)
        dist.barrier(group=shard.group)


def _allreduce_max_i32(t, shard):
    if shard.world == 1:
        return t
    if _nccl(shard):
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=shard.group)
        return t
    h = t.cpu()
    dist.all_reduce(h, op=dist.ReduceOp.MAX, group=shard.group)
    return h.to(t.device)


class PeerArena:
    """A device buffer shared with every rank: `ptrs[d]` is rank d's copy as
    mapped into this process (CUDA IPC handles exchanged once through
    torch.distributed; the local rank's own pointer for d == rank)."""

    def __init__(self, t: torch.Tensor, shard: Shard):
        self.tensor = t
        self.shard = shard
        self._opened = []
        local = t.data_ptr()
        if shard.world == 1:
            self.ptrs = [local]
            return
        st = t.untyped_storage()
        info = st._share_cuda_()  # (device, handle, size, offset of the storage in its base allocation, ...)
        handle, base_off = bytes(info[1]), int(info[3])
        # torch >= 2.5 prefixes the cudaIpcMemHandle_t (64 bytes) with a format version and a
        # type byte ('c': a cudaMalloc segment); expandable segments are not IPC-mappable here
        if len(handle) == 66:
            handle = handle[2:]
        elif len(handle) != 64:
            raise UnsupportedModelError("peer arenas need cudaMalloc-backed allocations "
                                        "(PYTORCH_CUDA_ALLOC_CONF without expandable_segments)")
        mine = (handle, base_off + t.storage_offset() * t.element_size())
        allinfo = [None] * shard.world
        dist.all_gather_object(allinfo, mine, group=shard.group)
        L = _lib.lib()
        self.ptrs = []
        for d, (h, off) in enumerate(allinfo):
            if d == shard.rank:
                self.ptrs.append(local)
                continue
            p = C.c_void_p()
            _lib.check(L.ssm_ipc_open(C.c_char_p(h), C.byref(p)), "ssm_ipc_open")
            self._opened.append(p.value)
            self.ptrs.append(p.value + off)

    def table(self, dev, stride_bytes=0, rows=1):
        """Device int64 table [rows][W]: rank d's pointer + row * stride_bytes."""
        base = np.array(self.ptrs, dtype=np.int64)
        tab = base[None, :] + stride_bytes * np.arange(rows, dtype=np.int64)[:, None]
        return torch.from_numpy(np.ascontiguousarray(tab)).to(dev)

    def close(self):
        L = _lib.lib()
        for p in self._opened:
            L.ssm_ipc_close(C.c_void_p(p))
        self._opened = []


class ShardedParticleFilter:
    def __init__(self, ir, theta, grid, n_particles, resampler="systematic", inputs=None, ess_rel=None,
                 check_finite=True, *, dtype="float64", exact=False, shard=None, device=None):
        if resampler not in ("systematic", "stratified"):
            raise ValueError("the sharded filter supports systematic and stratified resampling")
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
        if self.P_loc % 32:
            raise ValueError("particles per rank must be a multiple of 32 (warp tiles)")
        self.resampler = resampler
        self.ess_rel = ess_rel
        self.check_finite = check_finite
        self.dtype_name, self.tdtype, self.dtype_id = _dtype_info(dtype)
        self.exact = bool(exact)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.loglik = 0.0

    def run(self, rng, upto=None):
        """particle_filter(...) semantics: init(child 0), advance(child 1),
        trajectory(child 2).  Returns (loglik, trajectory) on every rank."""
        L = _lib.lib()
        sh, W, r = self.shard, self.shard.world, self.shard.rank
        spec, P, Pl, dev, tdt = self.spec, self.P, self.P_loc, self.device, self.tdtype
        nx, esz = spec.nx, (8 if self.dtype_id == _lib.SSM_F64 else 4)
        S = self.grid.last if upto is None else upto
        sched = _schedule(self.grid, spec, self.inputs, dev)
        stream = _lib.stream_ptr()
        off = r * Pl
        keys0 = torch.from_numpy(device_key(rng.child(0)).astype(np.uint32).reshape(1, 2).view(np.int32)).to(dev)
        keys1 = torch.from_numpy(device_key(rng.child(1)).astype(np.uint32).reshape(1, 2).view(np.int32)).to(dev)
        # arenas, allocated once and mapped by every rank: positions [S+1][nx][Pl],
        # ancestors (global indices) [S][Pl]
        X = torch.empty((S + 1, nx, Pl), dtype=tdt, device=dev)
        ANC = torch.empty((max(S, 1), Pl), dtype=torch.int32, device=dev)
        xa, aa = PeerArena(X, sh), PeerArena(ANC, sh)
        try:
            return self._run(L, rng, S, sched, stream, off, keys0, keys1, X, ANC, xa, aa)
        finally:
            _barrier(sh, dev)  # no rank unmaps / frees an arena another rank may still read
            xa.close()
            aa.close()

    def _run(self, L, rng, S, sched, stream, off, keys0, keys1, X, ANC, xa, aa):
        sh, W, r = self.shard, self.shard.world, self.shard.rank
        spec, P, Pl, dev = self.spec, self.P, self.P_loc, self.device
        nx, esz = spec.nx, (8 if self.dtype_id == _lib.SSM_F64 else 4)
        xtab = xa.table(dev, nx * Pl * esz, S + 1)  # [i][d]: rank d's x_i
        atab = aa.table(dev, Pl * 4, max(S, 1))  # [i-1][d]: rank d's ancestors used at step i
        theta = torch.from_numpy(spec.derived(self.theta)).to(dev)
        if spec.kernel == _lib.SSM_MODEL_GENERIC:  # the model's initial block, global particle indices
            _lib.check(L.ssm_gen_init_particles(C.c_void_p(spec.handle(dev)), self.dtype_id, 1, Pl, off,
                                                _lib.ptr(keys0), _lib.ptr(theta), spec.theta_stride, _lib.ptr(X[0]),
                                                None, stream), "ssm_gen_init_particles")
        else:
            _lib.check(L.ssm_init_particles(spec.kernel, self.dtype_id, 1, Pl, off, _lib.ptr(keys0), _lib.ptr(X[0]),
                                            stream), "ssm_init_particles")
        fs = _fs_init(1, dev)
        pw_ws = torch.empty(L.ssm_pw_workspace_bytes(1, Pl), dtype=torch.uint8, device=dev)
        sw = torch.empty(L.ssm_sharded_workspace_bytes(1, Pl, P), dtype=torch.uint8, device=dev)
        cdf = torch.empty(Pl, dtype=torch.int64, device=dev)
        trec = torch.empty(((Pl + 31) // 32, 2), dtype=torch.float64, device=dev)
        lse_part = torch.empty(4, dtype=torch.float64, device=dev)
        tot = torch.empty(1, dtype=torch.int64, device=dev)
        a_ring = torch.empty((2, Pl), dtype=self.tdtype, device=dev)
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
        A.x_in_stride = A.x_out_stride = Pl
        A.peer_n = Pl
        if spec.kernel == _lib.SSM_MODEL_GENERIC:
            A.gen, A.theta_stride = spec.handle(dev), spec.theta_stride

        has_anc = np.zeros(S + 1, dtype=np.int32)
        a_last = None
        slot = 0
        n_res = 0
        maybe = False
        # per-step pointers by arithmetic on the arena bases (no tensor views in the loop)
        x_base, x_step = X.data_ptr(), nx * Pl * esz
        anc_base, atab_base, xtab_base = ANC.data_ptr(), atab.data_ptr(), xtab.data_ptr()
        a_ptrs = [a_ring[0].data_ptr(), a_ring[1].data_ptr()]
        for i in range(1, S + 1):
            anc = None
            if maybe:  # resample at the start of step i (particle.py:96-105), across ranks
                anc_ptr = anc_base + (i - 1) * Pl * 4
                with profiling.maybe("resample", int(Pl * _resample_bytes(esz))):
                    if W == 1:  # one rank: the single filter's resample (same bits, PDL-chained)
                        _lib.check(L.ssm_resample_tiles_step(1, Pl, scheme, _lib.ptr(cdf), _lib.ptr(trec), _lib.ptr(fs),
                                                             None, _lib.ptr(keys1), i, C.c_void_p(anc_ptr),
                                                             _lib.ptr(sw), n_res & 1, int(n_res == 0), stream),
                                   "ssm_resample_tiles_step")
                    else:
                        _lib.check(L.ssm_tiles_total(1, Pl, _lib.ptr(trec), _lib.ptr(fs), _lib.ptr(tot),
                                                     _lib.ptr(sw), stream), "ssm_tiles_total")
                        tots = _allgather_tensor(tot, sh).reshape(W)  # C1'
                        _lib.check(L.ssm_offspring_push(Pl, P, W, r, scheme, _lib.ptr(cdf), _lib.ptr(tots), None,
                                                        _lib.ptr(keys1), i, _lib.ptr(fs),
                                                        C.c_void_p(atab_base + (i - 1) * W * 8), _lib.ptr(sw),
                                                        stream), "ssm_offspring_push")
                        _barrier(sh, dev)  # C2
                n_res += 1
                anc = anc_ptr
                has_anc[i] = 1
            obs = sched.obs[i]
            a_out = a_ptrs[slot % 2] if obs is not None else None
            A.step, A.n_sub = i, sched.n_sub[i]
            A.hints = _lib.SSM_HINT_SINGLE_SUBSTEP if sched.single[i] else 0
            A.subs = sched.subs_ptr(i)
            A.y_vec, A.u_vec = sched.y_ptr(i), sched.u_ptr(i)
            A.x_in, A.x_out = x_base + (i - 1) * x_step, x_base + i * x_step
            A.x_peer = (xtab_base + (i - 1) * W * 8) if W > 1 else None  # one rank: the plain gather
            A.anc = anc
            A.a_prev = a_last
            A.a_out = a_out
            A.cdf_local = cdf.data_ptr() if obs is not None else None
            A.tile_rec = trec.data_ptr() if obs is not None else None
            A.lse_out = lse_part.data_ptr() if obs is not None else None
            if obs is not None:
                A.has_obs, A.obs_mask, A.u_obs = 1, obs[0], obs[2]
                for n in range(8):
                    A.y[n] = float(obs[1][n])
            else:
                A.has_obs, A.obs_mask = 0, 0
            with profiling.maybe("propagate_weight", Pl * _pw_bytes(nx, esz, anc is not None, obs is not None)):
                _lib.check(L.ssm_propagate_weight(A, stream), "ssm_propagate_weight")
            if obs is not None:
                parts = _allgather_tensor(lse_part, sh)  # C1
                _lib.check(L.ssm_lse_combine(W, 1, _lib.ptr(parts), _lib.ptr(fs), ess_rel, float(P), i, stream),
                           "ssm_lse_combine")
                a_last = a_out
                slot += 1
                maybe = True
            elif maybe and self.ess_rel is None:
                maybe = False
        st = _fs_view(fs)[0]  # the run's one synchronisation
        nf, dg = int(st["err_nonfinite"]), int(st["err_degenerate"])
        if self.check_finite and nf != _lib.INT32_MAX and (dg == _lib.INT32_MAX or nf // 64 <= dg):
            t = sched.sub_end[nf // 64][nf % 64]
            raise NonFiniteStateError(f"non-finite state after transition sub-step ending at t={t:g}", time=t)
        if dg != _lib.INT32_MAX:
            t = float(sched.times[dg])
            raise DegenerateEnsembleError(f"all particle weights vanished at t={t:g}", time=t)
        self.loglik = float(st["loglik"])
        traj = self._trajectory(L, rng.child(2), S, a_last, fs, cdf, trec, tot, sw, xa, aa, has_anc, stream)
        return self.loglik, traj

    def _trajectory(self, L, rng, S, a_last, fs, cdf, trec, tot, sw, xa, aa, has_anc, stream):
        """sample_trajectory (particle.py:137-149): one multinomial draw on the
        global final weights, then the ancestry walk through the peer arenas."""
        sh, W, r = self.shard, self.shard.world, self.shard.rank
        P, Pl, dev, nx = self.P, self.P_loc, self.device, self.spec.nx
        u = float(np.asarray(rng.uniform(size=1))[0])
        if a_last is None:  # uniform weights: cum_j = (j + 1) / P
            j = torch.tensor([min(int(u * P), P - 1)], dtype=torch.int32, device=dev)
        else:
            _lib.check(L.ssm_tiles_total(1, Pl, _lib.ptr(trec), _lib.ptr(fs), _lib.ptr(tot), _lib.ptr(sw), stream),
                       "ssm_tiles_total")
            tots = _allgather_tensor(tot, sh).reshape(W)
            ut = torch.tensor([u], dtype=torch.float64, device=dev)
            j = torch.empty(1, dtype=torch.int32, device=dev)
            _lib.check(L.ssm_pick_sharded(Pl, W, r, _lib.ptr(cdf), _lib.ptr(tots), _lib.ptr(ut), _lib.ptr(j),
                                          _lib.ptr(sw), stream), "ssm_pick_sharded")
            j = _allreduce_max_i32(j, sh)
        xt = xa.table(dev)
        at = aa.table(dev)
        ha = torch.from_numpy(has_anc).to(dev)
        out = torch.empty((S + 1, nx), dtype=torch.float64, device=dev)
        _lib.check(L.ssm_trace_peer(self.dtype_id, S, nx, Pl, _lib.ptr(xt), _lib.ptr(at), _lib.ptr(ha), _lib.ptr(j),
                                    _lib.ptr(out), stream), "ssm_trace_peer")
        return out.cpu().numpy()


def particle_filter_sharded(ir, theta, grid, rng, n_particles, resampler="systematic", shard=None, **kw):
    """particle_filter over the ranks of `shard` (default torch.distributed)."""
    f = ShardedParticleFilter(ir, theta, grid, n_particles, resampler=resampler, shard=shard, **kw)
    return f.run(rng)

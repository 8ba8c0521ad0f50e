"""Multinomial, stratified and systematic resampling on the device
(drop-in for the reference's inference/resampling.py:15-36).

`resample(weights, scheme, rng, size=None)` keeps the reference's signature,
validation order and exceptions.  The CDF is the exact fixed-point scan
(K4) and the search is K5; the uniforms are the reference's own draws from
`rng` (so given the same rng the ancestors are the reference's).
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _lib
from ..errors import DegenerateEnsembleError

SCHEMES = ("multinomial", "stratified", "systematic")


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def resample(weights, scheme, rng, size=None):
    """Draw ancestor indices proportional to `weights` (>= 0, sum > 0)."""
    w = np.asarray(weights, dtype=float)
    if w.ndim != 1 or w.size == 0:
        raise ValueError("weights must be a non-empty vector")
    if scheme not in SCHEMES:
        raise ValueError(f"unknown resampling scheme {scheme!r}")
    _lib.require_cuda()
    L = _lib.lib()
    dev = _device()
    P_in = w.size
    P = P_in if size is None else int(size)
    stream = _lib.stream_ptr()
    wt = torch.from_numpy(w).to(dev)
    ws = torch.empty(L.ssm_scan_workspace_bytes(1, P_in), dtype=torch.uint8, device=dev)
    cum = torch.empty(P_in, dtype=torch.int64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(L.ssm_weights_scan(1, P_in, _lib.SSM_F64, _lib.ptr(wt), 0, None, None, _lib.ptr(cum),
                                  _lib.ptr(flags), _lib.ptr(ws), stream), "ssm_weights_scan")
    f = int(flags.item())
    if f & _lib.SSM_FLAG_BAD_WEIGHT:
        raise ValueError("weights must be finite and non-negative")
    if f & _lib.SSM_FLAG_ZERO_TOTAL:
        raise DegenerateEnsembleError("all resampling weights are zero")
    if scheme == "systematic":
        u = np.array([float(rng.uniform())])
    else:
        u = np.asarray(rng.uniform(size=P), dtype=float)
    ut = torch.from_numpy(u).to(dev)
    anc = torch.empty(P, dtype=torch.int32, device=dev)
    sws = torch.empty(max(1, L.ssm_search_workspace_bytes(1, P_in, P)), dtype=torch.uint8, device=dev)
    _lib.check(L.ssm_resample_search(1, P_in, P, _lib.SCHEME_IDS[scheme], 1, _lib.ptr(cum), _lib.ptr(ut),
                                     None, 0, None, _lib.ptr(anc), _lib.ptr(sws), stream), "ssm_resample_search")
    return anc.cpu().numpy().astype(np.int64)


def search_cdf(cum, u, scheme, P_out=None, device=None):
    """Ancestors from an injected float64 CDF and injected uniforms (the
    exact-parity entry point: identical (cum, u) -> identical ancestors)."""
    _lib.require_cuda()
    L = _lib.lib()
    dev = device or _device()
    cum = torch.as_tensor(np.ascontiguousarray(cum, dtype=np.float64)).to(dev)
    P_in = cum.shape[-1]
    B = 1 if cum.dim() == 1 else cum.shape[0]
    P_out = P_in if P_out is None else P_out
    ut = torch.as_tensor(np.ascontiguousarray(u, dtype=np.float64)).to(dev)
    anc = torch.empty((B, P_out), dtype=torch.int32, device=dev)
    sws = torch.empty(max(1, L.ssm_search_workspace_bytes(B, P_in, P_out)), dtype=torch.uint8, device=dev)
    _lib.check(L.ssm_resample_search(B, P_in, P_out, _lib.SCHEME_IDS[scheme], 0, _lib.ptr(cum), _lib.ptr(ut),
                                     None, 0, None, _lib.ptr(anc), _lib.ptr(sws), _lib.stream_ptr()),
               "ssm_resample_search")
    out = anc.cpu().numpy().astype(np.int64)
    return out[0] if cum.dim() == 1 else out

"""Out-of-bounds reads past the end of an input array: every input is placed so
that it ends exactly at the end of a mapped 2 MB region whose next page is
reserved but unmapped (cuMemAddressReserve / cuMemCreate / cuMemMap), so a
kernel reading even one element past the array faults.  Covers the
resampling entry points at sizes that leave the last 2048-particle tile
partial (the search kernel read C_{j-1} for threads past P_in, which crashed
a 256-slot theta resample depending on where the allocator had put the
array).  Runs in a subprocess: a fault poisons the CUDA context.
Reference: inference/resampling.py:15-36 (the calls' semantics)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import sys
import numpy as np, torch
sys.path.insert(0, %r)
from cuda.bindings import driver as d
from paper_1306_3277_b200 import _lib

def ok(r):
    assert r[0] == d.CUresult.CUDA_SUCCESS, r
    return r[1] if len(r) > 1 else None

torch.zeros(1, device="cuda")  # primary context current
dev = torch.cuda.current_device()
prop = d.CUmemAllocationProp()
prop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
prop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
prop.location.id = dev
gran = ok(d.cuMemGetAllocationGranularity(prop, d.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))
va = int(ok(d.cuMemAddressReserve(4 * gran, 0, 0, 0)))
h = ok(d.cuMemCreate(gran, prop, 0))
ok(d.cuMemMap(va, gran, 0, h, 0))  # [va, va + gran) mapped; [va + gran, va + 4 gran) reserved only
acc = d.CUmemAccessDesc()
acc.location = prop.location
acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
ok(d.cuMemSetAccess(va, gran, [acc], 1))
END = va + gran

def at_end(arr):
    # copy a host array so that it ends exactly at the guard page; returns its device pointer
    a = np.ascontiguousarray(arr)
    p = END - a.nbytes
    ok(d.cuMemcpyHtoD(p, a.ctypes.data, a.nbytes))
    return p

L = _lib.lib()
st = _lib.stream_ptr()
dv = torch.device("cuda")
rs = np.random.default_rng(5)
n_calls = 0
for P in (1, 5, 256, 2047, 2049, 5000, 70001):
    w = rs.random(P) + 0.01
    ws = torch.empty(max(1, L.ssm_scan_workspace_bytes(1, P)), dtype=torch.uint8, device=dv)
    flags = torch.zeros(1, dtype=torch.int32, device=dv)
    cum = torch.empty(P, dtype=torch.int64, device=dv)
    _lib.check(L.ssm_weights_scan(1, P, _lib.SSM_F64, at_end(w), 0, None, None, _lib.ptr(cum), _lib.ptr(flags),
                                  _lib.ptr(ws), st), "weights_scan")
    torch.cuda.synchronize(); n_calls += 1
    cum_end = at_end(cum.cpu().numpy())
    for scheme in (0, 1, 2):  # multinomial, stratified, systematic
        u = torch.as_tensor(np.sort(rs.random(P)) if scheme == 0 else rs.random(P), device=dv)
        anc = torch.empty(P, dtype=torch.int32, device=dv)
        sws = torch.empty(max(1, L.ssm_search_workspace_bytes(1, P, P)), dtype=torch.uint8, device=dv)
        _lib.check(L.ssm_resample_search(1, P, P, scheme, 1, cum_end, _lib.ptr(u), None, 0, None, _lib.ptr(anc),
                                         _lib.ptr(sws), st), "resample_search")
        torch.cuda.synchronize(); n_calls += 1
        a = anc.cpu().numpy()
        assert a.min() >= 0 and a.max() < P and np.all(np.diff(a) >= 0), (P, scheme)
    # double-valued normalised CDF (cum_kind 0)
    cd = np.cumsum(w / w.sum()); cd[-1] = 1.0
    cd_end = at_end(cd)
    for scheme in (1, 2):
        u = torch.as_tensor(rs.random(P), device=dv)
        anc = torch.empty(P, dtype=torch.int32, device=dv)
        sws = torch.empty(max(1, L.ssm_search_workspace_bytes(1, P, P)), dtype=torch.uint8, device=dv)
        _lib.check(L.ssm_resample_search(1, P, P, scheme, 0, cd_end, _lib.ptr(u), None, 0, None, _lib.ptr(anc),
                                         _lib.ptr(sws), st), "resample_search (double cum)")
        torch.cuda.synchronize(); n_calls += 1
    # log-weights -> tile records -> tile-path resample; log-sum-exp
    lw = rs.normal(0.0, 1.0, size=P)
    lw_end = at_end(lw)
    shift = torch.as_tensor([float(np.log(np.sum(np.exp(lw))))], dtype=torch.float64, device=dv)
    keys = torch.tensor([[7, 11]], dtype=torch.int32, device=dv)
    rws = torch.empty(max(1, L.ssm_resample_workspace_bytes(1, P)), dtype=torch.uint8, device=dv)
    for scheme in (1, 2, 3):
        anc = torch.empty(P, dtype=torch.int32, device=dv)
        _lib.check(L.ssm_resample_from_logw(1, P, _lib.SSM_F64, scheme, lw_end, _lib.ptr(shift), None, None,
                                            _lib.ptr(keys), 2, _lib.ptr(anc), _lib.ptr(rws), st), "from_logw")
        torch.cuda.synchronize(); n_calls += 1
        a = anc.cpu().numpy()
        assert a.min() >= 0 and a.max() < P, (P, scheme)
    lse = torch.empty(1, dtype=torch.float64, device=dv)
    ess = torch.empty(1, dtype=torch.float64, device=dv)
    lws = torch.empty(max(1, L.ssm_lse_workspace_bytes(1, P)), dtype=torch.uint8, device=dv)
    _lib.check(L.ssm_logsumexp(_lib.SSM_F64, 1, P, lw_end, _lib.ptr(lse), _lib.ptr(ess), _lib.ptr(lws), st), "lse")
    torch.cuda.synchronize(); n_calls += 1
    assert abs(float(lse) - float(shift)) < 1e-9
    # ancestors at the guard page for the state gather
    if P * 8 * 3 <= gran:
        x = torch.as_tensor(rs.random((3, P)), device=dv)
        xo = torch.empty_like(x)
        idx = np.sort(rs.integers(0, P, size=P)).astype(np.int32)
        _lib.check(L.ssm_gather(_lib.SSM_F64, 1, 3, P, _lib.ptr(x), at_end(idx), _lib.ptr(xo), st), "gather")
        torch.cuda.synchronize(); n_calls += 1
        assert np.array_equal(xo.cpu().numpy(), x.cpu().numpy()[:, idx])
print("ok", n_calls)
""" % ROOT


def test_resampling_reads_stay_inside_their_arrays():
    r = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert r.stdout.split()[0] == "ok"


GUARD_SELFTEST = r"""
import os, sys
sys.path.insert(0, %r)
from tests.conftest import install_guard_allocator
install_guard_allocator()
import numpy as np, torch
from paper_1306_3277_b200 import _lib
L = _lib.lib()
P = 1000
x = torch.zeros((1, P), dtype=torch.float64, device="cuda")
xo = torch.empty_like(x)
idx = torch.tensor(np.arange(P, dtype=np.int32), device="cuda")
_lib.check(L.ssm_gather(_lib.SSM_F64, 1, 1, P, _lib.ptr(x), _lib.ptr(idx), _lib.ptr(xo), _lib.stream_ptr()), "g")
torch.cuda.synchronize()
print("in-bounds ok", flush=True)
idx[-1] = P + 64  # 512 bytes past the end of x
_lib.check(L.ssm_gather(_lib.SSM_F64, 1, 1, P, _lib.ptr(x), _lib.ptr(idx), _lib.ptr(xo), _lib.stream_ptr()), "g")
torch.cuda.synchronize()
print("OOB not detected", flush=True)
""" % ROOT


def test_guard_allocator_catches_an_out_of_bounds_read():
    """The allocator behind SSM_GUARD_ALLOC (tests/tools/guard_alloc.cpp) faults a
    gather that reads 512 bytes past its input."""
    r = subprocess.run([sys.executable, "-c", GUARD_SELFTEST], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "SSM_GUARD_ALIGN": "16"})
    assert "in-bounds ok" in r.stdout, r.stderr[-2000:]
    assert "OOB not detected" not in r.stdout
    assert r.returncode != 0


def test_parity_suite_under_guard_allocator():
    """tests/test_gpu_parity.py with every torch tensor ending at an unmapped guard
    page (16-byte slack): no kernel of the filter, resampling, trajectory,
    small-P or generic paths touches memory past a tensor's end.  (The whole
    GPU suite passes this way except the CUDA-IPC sharded tests, whose peer
    mappings need cudaMalloc memory.)"""
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-q", "-x",
                        "-p", "no:cacheprovider"], capture_output=True, text=True, timeout=1200, cwd=ROOT,
                       env={**os.environ, "SSM_GUARD_ALLOC": "1", "SSM_GUARD_ALIGN": "16"})
    assert r.returncode == 0, r.stdout[-3000:]

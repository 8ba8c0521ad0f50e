"""Split the r microbench (bench_outer configr) into its two calls: ssm_resample_from_logw
and ssm_gather at 2^24, f64, nx=8, sigma_w in {0, 1, 10}; CUDA events, 10 reps each.
usage: python profiles/gather_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1306_3277_b200 import _lib  # noqa: E402


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    L = _lib.lib()
    P = 1 << 24
    dev = torch.device("cuda")
    rs = np.random.default_rng(1234)
    x = torch.as_tensor(rs.uniform(-1.0, 3.0, size=(8, P)), device=dev)
    xo = torch.empty_like(x)
    anc = torch.empty(P, dtype=torch.int32, device=dev)
    ws = torch.empty(L.ssm_resample_workspace_bytes(1, P), dtype=torch.uint8, device=dev)
    keys = torch.tensor([[12345, 678]], dtype=torch.int32, device=dev)
    st = _lib.stream_ptr()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6536.4)
    for sw in (0.0, 1.0, 10.0):
        a = torch.as_tensor(rs.normal(0.0, sw, size=P) if sw > 0 else np.zeros(P), device=dev)
        shift = torch.logsumexp(a, 0).reshape(1)
        for name, scheme in (("systematic", 2), ("stratified", 1), ("multinomial_sorted", 3)):
            def rsmp():
                _lib.check(L.ssm_resample_from_logw(1, P, _lib.SSM_F64, scheme, _lib.ptr(a), _lib.ptr(shift), None,
                                                    None, _lib.ptr(keys), 1, _lib.ptr(anc), _lib.ptr(ws), st), "rs")

            def gath():
                _lib.check(L.ssm_gather(_lib.SSM_F64, 1, 8, P, _lib.ptr(x), _lib.ptr(anc), _lib.ptr(xo), st), "g")

            t_r = timed(rsmp)
            t_g = timed(gath)
            gb = 132.0 * P / (t_g / 1e3) / 1e9
            print(f"sigma_w={sw:g} {name:20s} resample {t_r * 1e3:7.1f} us  gather {t_g * 1e3:7.1f} us "
                  f"({gb:6.0f} GB/s = {gb / peak:.2f} of peak at 132 B)")


if __name__ == "__main__":
    main()

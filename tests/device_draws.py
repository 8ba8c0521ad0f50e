"""Test helper: the device noise of the fast path, restated or exported, so
the CPU oracle can be run on EXACTLY the draws the benchmark kernels consumed.

  * Philox4x32-10 words (ssm_common.cuh) are restated in numpy: the device
    uniforms (initial states, systematic / stratified queries, exponential
    spacings of the sorted multinomial) are reproduced bit for bit;
  * the float32 Box-Muller normals use MUFU approximations (lg2 / sincos) that
    numpy cannot reproduce, so they are exported from the device through the
    C ABI (ssm_device_normals) -- the same device functions the fused kernel
    calls.

`DeviceDrawStream` mimics the oracle's Stream (child / uniform / normal) for
one particle filter run: grid step i's child(i).child(0) yields the
resampling draws, child(i).child(1) the transition noise (slot-major, sub-step
by sub-step, as simulate.py:50-60 consumes them).
"""

from __future__ import annotations

import numpy as np
import torch

PURPOSE_NOISE, PURPOSE_RESAMPLE, PURPOSE_INIT, PURPOSE_SYSTEMATIC, PURPOSE_SPACING = 1, 2, 3, 4, 5


def philox4x32_10(ctr, k0, k1):
    """numpy restatement of the device Philox4x32-10 (ssm_common.cuh)."""
    M0, M1, W0, W1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57), 0x9E3779B9, 0xBB67AE85
    c = [np.asarray(x, dtype=np.uint64) & np.uint64(0xFFFFFFFF) for x in ctr]
    k0, k1 = int(k0), int(k1)
    for _ in range(10):
        p0, p1 = M0 * c[0], M1 * c[2]
        lo0, hi0 = p0 & np.uint64(0xFFFFFFFF), p0 >> np.uint64(32)
        lo1, hi1 = p1 & np.uint64(0xFFFFFFFF), p1 >> np.uint64(32)
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
        k0, k1 = (k0 + W0) & 0xFFFFFFFF, (k1 + W1) & 0xFFFFFFFF
    return c


def u53(hi, lo):
    return ((hi << np.uint64(32)) | lo) >> np.uint64(11)


def u53f(hi, lo):
    return u53(hi, lo).astype(np.float64) * 2.0**-53


def device_uniform(keys, k, step, purpose):
    """device_uniform(k0, k1, k, step, purpose) of ssm_resample.cu for an array of k."""
    k = np.atleast_1d(np.asarray(k, dtype=np.uint64))
    n = k.size
    r = philox4x32_10([k, np.full(n, step), np.zeros(n), np.full(n, purpose)], *keys)
    return u53f(r[0], r[1])


def device_init_l96(keys, P):
    """init_one<L96> (ssm_models.cuh): x[2g], x[2g+1] = -1 + 4 u53 of Philox block g."""
    p = np.arange(P, dtype=np.uint64)
    x = np.zeros((P, 8))
    for g in range(4):
        r = philox4x32_10([p, np.zeros(P), np.full(P, g), np.full(P, PURPOSE_INIT)], *keys)
        x[:, 2 * g] = -1.0 + 4.0 * u53f(r[0], r[1])
        x[:, 2 * g + 1] = -1.0 + 4.0 * u53f(r[2], r[3])
    return x


def sorted_multinomial_uniforms(keys, P, step):
    """U_(k) = S_k / S_{P+1} from the device's exponential spacings (spacing k:
    Philox block k // 2, words (x, y) even / (z, w) odd)."""
    k = np.arange(P + 1, dtype=np.uint64)
    r = philox4x32_10([k >> np.uint64(1), np.full(P + 1, step), np.zeros(P + 1), np.full(P + 1, PURPOSE_SPACING)],
                      *keys)
    odd = (k & np.uint64(1)).astype(bool)
    u = np.where(odd, u53(r[2], r[3]), u53(r[0], r[1]))
    E = -np.log(1.0 - u.astype(np.float64) * 2.0**-53)
    S = np.cumsum(E)
    return S[:P] / S[P]


def device_normals(model, keys, P, step, sub, p_offset=0):
    """The fused kernel's float32 standard normals (C ABI ssm_device_normals):
    L96 (8, P) slot-major, windkessel (P,)."""
    from paper_1306_3277_b200 import _lib

    L = _lib.lib()
    nx = 8 if model == _lib.SSM_MODEL_LORENZ96 else 1
    kt = torch.from_numpy(np.asarray(keys, dtype=np.uint32).reshape(1, 2).view(np.int32)).cuda()
    out = torch.empty((nx, P), dtype=torch.float32, device="cuda")
    _lib.check(L.ssm_device_normals(model, 1, P, p_offset, _lib.ptr(kt), step, sub, _lib.ptr(out),
                                    _lib.stream_ptr()), "ssm_device_normals")
    z = out.cpu().numpy().astype(np.float64)
    return z if nx > 1 else z[0]


class DeviceDrawStream:
    """Oracle-facing stream replaying one device-noise filter run's draws.

    keys_init / keys_adv: the Philox keys of the run's init and advance
    streams (rng.device_key of rng.child(0) / rng.child(1) for particle_filter);
    scheme: the resampler the device ran ("multinomial" = the sorted
    multinomial of the device filter path)."""

    def __init__(self, model, keys_init, keys_adv, P, scheme, path=()):
        self.model, self.keys_init, self.keys_adv = model, keys_init, keys_adv
        self.P, self.scheme, self.path = P, scheme, tuple(path)
        self._calls = 0

    def child(self, *key):
        return DeviceDrawStream(self.model, self.keys_init, self.keys_adv, self.P, self.scheme, self.path + key)

    def uniform(self, low=0.0, high=1.0, size=None):
        (i, purpose) = self.path
        assert purpose == 0, self.path
        P = self.P
        if self.scheme == "systematic":
            return float(device_uniform(self.keys_adv, 0, i, PURPOSE_SYSTEMATIC)[0])
        if self.scheme == "stratified":
            return device_uniform(self.keys_adv, np.arange(P), i, PURPOSE_RESAMPLE)
        return sorted_multinomial_uniforms(self.keys_adv, P, i)

    def normal(self, loc=0.0, scale=1.0, size=None):
        from paper_1306_3277_b200 import _lib

        (i, purpose) = self.path
        assert purpose == 1, self.path
        c = self._calls
        self._calls += 1
        if self.model == "lorenz96":
            sub, slot = divmod(c, 8)
            if slot == 0:
                self._z = device_normals(_lib.SSM_MODEL_LORENZ96, self.keys_adv, self.P, i, sub)
            z = self._z[slot]
        else:
            z = device_normals(_lib.SSM_MODEL_WINDKESSEL, self.keys_adv, self.P, i, c)
        return loc + np.asarray(scale) * z

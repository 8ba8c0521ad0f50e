"""Per-kernel CUDA-event timing and launch counting for the filter path.

`KernelTimer` records a (start, end) event pair on the launching stream
around every C-ABI kernel launch while active; nothing synchronises until
`summary()`.  `launch_count()` counts libssm_b200 kernel launches (a wrapper
in `_lib` increments it), which bench.py reports as `gpu_launches`.
"""

from __future__ import annotations

import contextlib
import gc
from collections import defaultdict

import torch

_ACTIVE = None
_LAUNCHES = 0


def count_launch(n=1):
    global _LAUNCHES
    _LAUNCHES += n


def launch_count():
    return _LAUNCHES


class NativeEvent:
    """cudaEvent_t owned by libssm_b200 (recorded inside native drivers)."""

    def __init__(self):
        import ctypes as C

        from . import _lib

        h = C.c_void_p()
        _lib.check(_lib.lib().ssm_event_create(C.byref(h)), "ssm_event_create")
        self.h = h.value

    def elapsed_time(self, end):
        import ctypes as C

        from . import _lib

        ms = C.c_float()
        _lib.check(_lib.lib().ssm_event_elapsed_ms(self.h, end.h, C.byref(ms)), "ssm_event_elapsed_ms")
        return float(ms.value)

    def __del__(self):
        try:
            from . import _lib

            _lib.lib().ssm_event_destroy(self.h)
        except Exception:
            pass


class KernelTimer:
    """`every` = k: inside the native grid-loop driver only grid steps i with
    i % k == k - 1 are bracketed by events (an event between two programmatic
    dependent launches serialises them, so timing every step would slow the
    run it measures); every=1 times every launch."""

    def __init__(self, every=1):
        self.events = defaultdict(list)  # name -> [(start, end, bytes)]
        self.every = max(int(every), 1)

    def samples(self, step):
        return self.every == 1 or step % self.every == self.every - 1

    def add(self, name, start, end, nbytes=0):
        self.events[name].append((start, end, nbytes))

    @contextlib.contextmanager
    def kernel(self, name, nbytes=0):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        try:
            yield
        finally:
            e.record()
            self.events[name].append((s, e, nbytes))

    def summary(self):
        torch.cuda.synchronize()
        out = {}
        for name, lst in self.events.items():
            ms = [s.elapsed_time(e) for s, e, _ in lst]
            nb = sum(b for _, _, b in lst)
            out[name] = {"launches": len(lst), "total_ms": float(sum(ms)),
                         "avg_ms": float(sum(ms) / len(ms)), "bytes": int(nb)}
        return out


def active():
    return _ACTIVE


@contextlib.contextmanager
def timing(timer: KernelTimer):
    global _ACTIVE
    prev, _ACTIVE = _ACTIVE, timer
    try:
        yield timer
    finally:
        _ACTIVE = prev


@contextlib.contextmanager
def maybe(name, nbytes=0):
    t = _ACTIVE
    if t is None:
        yield
    else:
        with t.kernel(name, nbytes):
            yield


@contextlib.contextmanager
def gc_paused():
    """Pause Python's cyclic garbage collector for a batched outer loop (PMMH,
    SMC^2): those loops allocate many small host objects per step, and the
    collector's periodic traversals of every live tensor / run object cost a
    third of an SMC^2 run's host time (profiles/r2_host_overhead.txt).  The loops
    create no reference cycles that must be reclaimed before they return."""
    was = gc.isenabled()
    gc.disable()
    try:
        yield
    finally:
        if was:
            gc.enable()

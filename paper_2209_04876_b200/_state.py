"""Per-thread state and the graph-capture gate.

The reference's contract (exercised by experiments.py:196-198 ``--parallel``) is that
independent solves may run concurrently on threads.  Everything a solve keeps between its own
calls -- the deferred validation flags, the captured-graph timeline, the events around the last
loop launch, the last step-norm history, the diagnostic phase marks -- is therefore per thread
(``TLSlot``) and the graph caches are keyed by thread and guarded by ``CACHE_LOCK``.

CUDA graph capture cannot overlap another thread's device-wide synchronisation (the eager paths
synchronise), so captures go through ``GATE``: every public entry point is ``gated`` (re-entrant,
counted per thread), and a thread captures only when it is the only one inside the API; new
entrants wait for the capture to finish.  When other solves are in flight the capture is skipped
and that call runs the eager pipeline (bit-identical results), to be captured on a later call."""

from __future__ import annotations

import contextlib
import functools
import threading


class TLSlot(threading.local):
    """One value per thread, read and written as ``slot[0]`` (the former module-level one-element
    lists keep their call sites)."""

    def __init__(self, value=None):
        self.value = value

    def __getitem__(self, i):
        return self.value

    def __setitem__(self, i, v):
        self.value = v


CACHE_LOCK = threading.RLock()
CAPTURE_MODE = "thread_local"


class Gate:
    def __init__(self):
        self._cv = threading.Condition()
        self._active = 0
        self._capturing = False
        self._tl = threading.local()

    def enter(self):
        depth = getattr(self._tl, "depth", 0)
        if depth == 0:
            with self._cv:
                while self._capturing:
                    self._cv.wait()
                self._active += 1
        self._tl.depth = depth + 1

    def exit(self):
        depth = self._tl.depth - 1
        self._tl.depth = depth
        if depth == 0:
            with self._cv:
                self._active -= 1
                self._cv.notify_all()

    @contextlib.contextmanager
    def capture(self):
        """Yields True when the calling thread may capture now (no other thread inside the API)."""
        inside = getattr(self._tl, "depth", 0) > 0
        with self._cv:
            ok = not self._capturing and self._active == (1 if inside else 0)
            if ok:
                self._capturing = True
        try:
            yield ok
        finally:
            if ok:
                with self._cv:
                    self._capturing = False
                    self._cv.notify_all()


GATE = Gate()


def gated(fn):
    """Public entry point: counted by GATE (re-entrant)."""
    if getattr(fn, "_ks_gated", False):
        return fn

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        GATE.enter()
        try:
            return fn(*args, **kwargs)
        finally:
            GATE.exit()

    wrapper._ks_gated = True
    return wrapper


def gate_names(namespace: dict, names):
    for n in names:
        namespace[n] = gated(namespace[n])


def thread_key() -> int:
    return threading.get_ident()


def cache_put(cache: dict, key, value, cap: int):
    """Insert under CACHE_LOCK, evicting the oldest entry beyond ``cap`` (a thread still replaying
    an evicted graph holds its own reference)."""
    with CACHE_LOCK:
        while len(cache) >= cap:
            cache.pop(next(iter(cache)))
        cache[key] = value
    return value


def cache_get(cache: dict, key):
    with CACHE_LOCK:
        return cache.get(key)


def cache_drop(cache: dict, key):
    with CACHE_LOCK:
        cache.pop(key, None)

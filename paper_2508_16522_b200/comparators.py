"""GPU comparators for the paper's claim direction (
PAPER.md:979-1003): the same DAG replayed as a CUDA Graph (one kernel node per
task) and by a generic event-driven per-task runtime (one launch + one event
per task on per-worker streams).  Library: libtdcmp.so."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .errors import DeviceError
from .flat import FlatGraph

_L = None


def _lib():
    global _L
    if _L is None:
        L = C.CDLL(N.CMP_LIB_PATH)
        vp = C.c_void_p
        L.td_cmp_last_error.restype = C.c_char_p
        L.td_cmp_graph_create.argtypes = [C.c_int64, vp, vp, vp, vp, vp, C.c_uint64, C.POINTER(vp)]
        L.td_cmp_graph_run.argtypes = [vp, C.POINTER(C.c_float)]
        L.td_cmp_tokens.argtypes = [vp, vp]
        L.td_cmp_destroy.argtypes = [vp]
        L.td_cmp_events.argtypes = [C.c_int64, vp, vp, vp, vp, vp, vp, C.c_int32, C.c_uint64,
                                    C.POINTER(C.c_float), vp]
        _L = L
    return _L


def _chk(rc):
    if rc:
        raise DeviceError(_lib().td_cmp_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _arrays(g: FlatGraph):
    order = np.argsort(g.topo_rank()).astype(np.int64)
    return (np.ascontiguousarray(g.pred.ptr, np.int64), np.ascontiguousarray(g.pred.iv, np.int32),
            np.ascontiguousarray(g.kind, np.uint8), np.ascontiguousarray(g.arg, np.uint32), order)


class CudaGraphReplay:
    """The DAG as one instantiated CUDA Graph."""

    def __init__(self, g: FlatGraph, seed: int = 0):
        self.n = g.n
        self._keep = _arrays(g)
        pp, piv, k, a, order = self._keep
        h = C.c_void_p()
        _chk(_lib().td_cmp_graph_create(g.n, _p(pp), _p(piv), _p(k), _p(a), _p(order), seed, C.byref(h)))
        self._h = h

    def run(self) -> float:
        ms = C.c_float()
        _chk(_lib().td_cmp_graph_run(self._h, C.byref(ms)))
        return float(ms.value)

    def tokens(self) -> np.ndarray:
        out = np.empty(self.n, np.uint64)
        _chk(_lib().td_cmp_tokens(self._h, _p(out)))
        return out

    def close(self):
        if self._h.value:
            _lib().td_cmp_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def event_runtime(g: FlatGraph, n_streams: int, seed: int = 0):
    """Generic runtime replay; returns (ms, tokens)."""
    pp, piv, k, a, order = _arrays(g)
    worker = np.ascontiguousarray(g.worker, np.int32)
    ms = C.c_float()
    out = np.empty(g.n, np.uint64)
    _chk(_lib().td_cmp_events(g.n, _p(pp), _p(piv), _p(k), _p(a), _p(order), _p(worker), n_streams, seed,
                              C.byref(ms), _p(out)))
    return float(ms.value), out

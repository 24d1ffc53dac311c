"""Sequential topological oracles over a flattened graph — TEST INFRASTRUCTURE.

* :func:`run_c`  — ctypes binding of seq_oracle.c (fast, full BASELINE sizes).
* :func:`run_py` — pure-Python restatement for small graphs (random DAGs).

Both restate SPEC.md:224/408 ("identical to a sequential topological
execution oracle") for the token definition of oracle/tokens.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import tokens as T

_DIR = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_DIR, "_build", "liboracle.so")
_lib = None


def build() -> str:
    src = os.path.join(_DIR, "seq_oracle.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_SO), exist_ok=True)
        subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", _SO, src], check=True)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        L.td_oracle_run.restype = C.c_int
        L.td_oracle_run.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]
        L.td_oracle_stencil2d.restype = C.c_int
        L.td_oracle_stencil2d.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p]
        L.td_oracle_compute_loop.restype = C.c_uint64
        L.td_oracle_compute_loop.argtypes = [C.c_uint64, C.c_uint32]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def run_c(n: int, pred_ptr: np.ndarray, pred_iv: np.ndarray, kind: np.ndarray | None,
          arg: np.ndarray | None, seed: int = 0, order: np.ndarray | None = None,
          literal_loop: bool = False, body_extra: np.ndarray | None = None) -> np.ndarray:
    """Token array via the C oracle.  `order` = node ids in a topological
    order (None = id order, valid for Task Bench graphs)."""
    pred_ptr = np.ascontiguousarray(pred_ptr, np.int64)
    pred_iv = np.ascontiguousarray(pred_iv, np.int32)
    kind = None if kind is None else np.ascontiguousarray(kind, np.uint8)
    arg = None if arg is None else np.ascontiguousarray(arg, np.uint32)
    order = None if order is None else np.ascontiguousarray(order, np.int64)
    extra = None if body_extra is None else np.ascontiguousarray(body_extra, np.uint64)
    out = np.zeros(n, dtype=np.uint64)
    rc = _load().td_oracle_run(n, _p(pred_ptr), _p(pred_iv), _p(kind), _p(arg), _p(order),
                               seed & T.M64, int(literal_loop), _p(extra), _p(out))
    if rc:
        raise ValueError(f"oracle: bad graph or order (rc={rc})")
    return out


def compute_loop(h: int, iters: int) -> int:
    return int(_load().td_oracle_compute_loop(h & T.M64, iters))


def run_py(n: int, preds: list[list[int]], kind=None, arg=None, seed: int = 0) -> list[int]:
    """Pure-Python sequential oracle: Kahn order, tokens per oracle/tokens.py."""
    succs = [[] for _ in range(n)]
    indeg = [0] * n
    for v in range(n):
        for u in preds[v]:
            succs[u].append(v)
            indeg[v] += 1
    ready = [v for v in range(n) if indeg[v] == 0]
    tok = [None] * n
    done = 0
    while ready:
        v = ready.pop()
        tok[v] = T.token_int(seed, v, [(u, tok[u]) for u in sorted(preds[v])],
                             0 if kind is None else int(kind[v]), 0 if arg is None else int(arg[v]))
        done += 1
        for s in succs[v]:
            indeg[s] -= 1
            if indeg[s] == 0:
                ready.append(s)
    if done != n:
        raise ValueError("cycle")
    return tok


def stencil2d_c(nx: int, ny: int, steps: int, seed: int = 0):
    """(per-task tile folds r[steps*ntiles], final grid) of the config-5 mini-app."""
    nt = (nx // 64) * (ny // 64)
    r = np.zeros(steps * nt, dtype=np.uint64)
    grid = np.zeros((ny, nx), dtype=np.uint32)
    rc = _load().td_oracle_stencil2d(nx, ny, steps, seed & T.M64, _p(r), _p(grid))
    if rc:
        raise ValueError(f"stencil2d oracle failed ({rc})")
    return r, grid


def stencil2d_tokens(g, seed: int = 0):
    """Full token array of a generate_stencil2d graph (C oracle)."""
    m = g.meta
    r, grid = stencil2d_c(m["nx"], m["ny"], m["steps"], seed)
    tok = run_c(g.n, g.pred.ptr, g.pred.iv, None, None, seed=seed, body_extra=r)
    return tok, grid

"""Host handle of one uploaded (compiled) graph on one GPU.

Thin owner of a ``td_graph*`` (include/tdexec.h).  The numpy arrays of the
FlatGraph are borrowed only for the upload call (tdexec.h "Ownership"); device
buffers are owned by the handle and freed by :meth:`close` / ``__del__``.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .flat import FlatGraph


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def device_info(device: int = 0, threads_per_block: int = 128) -> dict:
    info = N.TdDeviceInfo()
    N.check(N.lib().td_device_info_get(device, threads_per_block, C.byref(info)))
    return dict(sm_count=info.sm_count, l2_bytes=info.l2_bytes, max_workers=info.max_workers,
                max_workers_st2d=info.max_workers_st2d, cc=(info.cc_major, info.cc_minor),
                name=info.name.decode())


class DeviceGraph:
    """A FlatGraph resident on one GPU (counters, tokens, CSR in HBM)."""

    def __init__(self, g: FlatGraph, device: int = 0, *, n_ranks: int = 1, my_rank: int = 0,
                 node_rank: np.ndarray | None = None, work_ptr=None, work=None,
                 n_ext_pre: int = 0, n_ext_post: int = 0, ident: np.ndarray | None = None,
                 dynamic: bool = False):
        self.graph = g
        self.device = device
        self.n = g.n
        self.n_cols = g.n_cols
        self.n_ranks = n_ranks
        self.my_rank = my_rank
        if work_ptr is None:
            work_ptr, work = g.worker_lists()
        keep = dict(
            pred_ptr=np.ascontiguousarray(g.pred.ptr, np.int64),
            pred_iv=np.ascontiguousarray(g.pred.iv, np.int32),
            succ_ptr=np.ascontiguousarray(g.succ.ptr, np.int64),
            succ_iv=np.ascontiguousarray(g.succ.iv, np.int32),
            kind=np.ascontiguousarray(g.kind, np.uint8),
            arg=np.ascontiguousarray(g.arg, np.uint32),
            work_ptr=np.ascontiguousarray(work_ptr, np.int64),
            work=np.ascontiguousarray(work, np.int32),
            col=None if g.col is None else np.ascontiguousarray(g.col, np.int32),
            node_rank=None if node_rank is None else np.ascontiguousarray(node_rank, np.uint8),
            ident=None if ident is None else np.ascontiguousarray(ident, np.int32),
        )
        csr = N.TdCsr(
            n_nodes=g.n,
            pred_ptr=_ptr(keep["pred_ptr"]), pred_iv=_ptr(keep["pred_iv"]),
            succ_ptr=_ptr(keep["succ_ptr"]), succ_iv=_ptr(keep["succ_iv"]),
            kind=_ptr(keep["kind"]), arg=_ptr(keep["arg"]),
            n_workers=int(len(keep["work_ptr"]) - 1),
            work_ptr=_ptr(keep["work_ptr"]), work=_ptr(keep["work"]),
            n_cols=int(g.n_cols if g.col is not None else 0), col=_ptr(keep["col"]),
            n_ranks=n_ranks, my_rank=my_rank, node_rank=_ptr(keep["node_rank"]),
            n_ext_pre=n_ext_pre, n_ext_post=n_ext_post, ident=_ptr(keep["ident"]),
            options=N.TD_UPLOAD_DYNAMIC if dynamic else 0,
        )
        self.n_workers = csr.n_workers
        if g.col is None:
            self.n_cols = 0
        h = C.c_void_p()
        N.check(N.lib().td_graph_upload(C.byref(csr), device, C.byref(h)))
        self._h = h
        self.last_flags = 0

    # -- execution ----------------------------------------------------------
    def launch(self, seed: int = 0, *, flags: int = N.TD_F_CHECKSUM, threads_per_block: int = 0,
               spin_limit: int = 0, stream: int | None = None) -> None:
        p = N.TdLaunchParams(seed=seed & ((1 << 64) - 1), flags=flags,
                             threads_per_block=threads_per_block, spin_limit=spin_limit)
        N.check(N.lib().td_graph_launch(self._h, C.byref(p), stream))
        self.last_flags = flags

    def wait(self, timeout: float | None = None) -> None:
        N.check(N.lib().td_graph_wait(self._h, -1.0 if timeout is None else float(timeout)))

    def query(self) -> bool:
        d = C.c_int32()
        N.check(N.lib().td_graph_query(self._h, C.byref(d)))
        return bool(d.value)

    def run(self, seed: int = 0, **kw) -> "DeviceGraph":
        self.launch(seed, **kw)
        self.wait()
        return self

    def set_body_arg(self, arg: int) -> None:
        """Set the arg of every COMPUTE / BUSY_WAIT body (granularity sweeps)."""
        N.check(N.lib().td_graph_set_body_arg(self._h, int(arg)))

    def trigger_pre(self, index: int) -> None:
        N.check(N.lib().td_graph_trigger_pre(self._h, index))

    def post_fired(self, index: int) -> bool:
        d = C.c_int32()
        N.check(N.lib().td_graph_post_fired(self._h, index, C.byref(d)))
        return bool(d.value)

    # -- results ------------------------------------------------------------
    def tokens(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.uint64)
        N.check(N.lib().td_graph_tokens(self._h, _ptr(out), self.n))
        return out

    def checksums(self) -> np.ndarray:
        out = np.empty(self.n_cols, dtype=np.uint64)
        N.check(N.lib().td_graph_checksums(self._h, _ptr(out), self.n_cols))
        return out

    def tally(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.uint32)
        N.check(N.lib().td_graph_tally(self._h, _ptr(out), self.n))
        return out

    def stats(self) -> dict:
        s = N.TdStats()
        N.check(N.lib().td_graph_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in N.TdStats._fields_}

    def trace(self, words: int = 4) -> np.ndarray:
        """(n, 4) %globaltimer ns: wait start, deps observed, gathered, signalled.
        (A -DTD_CYCLE_PROBE diagnostic build records (n, 8) %clock64 points.)"""
        out = np.empty(words * self.n, dtype=np.uint64)
        N.check(N.lib().td_graph_trace(self._h, _ptr(out), words * self.n))
        return out.reshape(self.n, words)

    def info(self) -> dict:
        """How the graph was lowered: kernel variant (plain), nodes per warp
        pass (group: 0, 2 or 4), workers, descriptor size."""
        i = N.TdGraphInfo()
        N.check(N.lib().td_graph_info_get(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in N.TdGraphInfo._fields_}

    def last_ms(self) -> float:
        ms = C.c_float()
        N.check(N.lib().td_graph_last_ms(self._h, C.byref(ms)))
        return float(ms.value)

    # -- config-5 mini-app ---------------------------------------------------
    def attach_stencil2d(self, nx: int, ny: int) -> None:
        N.check(N.lib().td_graph_attach_stencil2d(self._h, nx, ny))
        self.st_shape = (ny, nx)

    def attach_scratch(self, words_per_worker: int) -> None:
        """Per-worker scratch for memory_bound (KIND_MEMORY) bodies."""
        N.check(N.lib().td_graph_attach_scratch(self._h, int(words_per_worker)))

    def stencil2d_grid(self, buf: int) -> np.ndarray:
        ny, nx = self.st_shape
        out = np.empty(nx * ny, dtype=np.uint32)
        N.check(N.lib().td_graph_stencil2d_grid(self._h, buf, _ptr(out), nx * ny))
        return out.reshape(ny, nx)

    # -- multi-GPU ----------------------------------------------------------
    def ipc_export(self) -> bytes:
        buf = C.create_string_buffer(1024)
        ln = C.c_size_t()
        N.check(N.lib().td_graph_ipc_export(self._h, buf, 1024, C.byref(ln)))
        return buf.raw[: ln.value]

    def ipc_attach(self, rank: int, handle: bytes) -> None:
        b = C.create_string_buffer(handle, len(handle))
        N.check(N.lib().td_graph_ipc_attach(self._h, rank, b, len(handle)))

    def attach_direct(self, rank: int, peer: "DeviceGraph") -> None:
        N.check(N.lib().td_graph_peer_attach_direct(self._h, rank, peer._h))

    # -- lifetime -----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            N.lib().td_graph_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

"""Alg. 1 on the GPU: ``compile`` / ``execute`` / ``message_stats``
(SPEC.md compiler 351-425; Alg. 1 632-693).

``compile(g)`` partitions the graph by resource (each resource becomes one
persistent worker warp, Alg. 1 ``RegisterActor(Worker(r,(V_w,E_w)), r)``),
orders each worker's nodes topologically, and uploads the flattened worker
programs + dependence counters to HBM through the C ABI
(``td_graph_upload``).  ``execute`` launches ONE persistent kernel
(``td_graph_launch``) — the INIT message to every worker — and returns the
``done`` event plus one event per external postcondition.

Differences from the CPU design, each documented in DESIGN.md:
* a node's counter is a mailbox word [count:16 | term sum:48] that its
  producers add to with one data-carrying atomic per edge; the consumer
  re-arms it to 0 after consuming it (SPEC.md:412's re-arm, done by the
  owner), so every replay starts from zeroed mailboxes.  Consumers with a
  shared large predecessor list poll shared mailbox replicas instead, banked
  by execution parity: each launch zeroes the bank the next one will use.
  An aborted or poisoned execution can leave partial sums behind: it marks
  the graph dirty and the next launch memsets the mailboxes first;
* executions are stream-ordered; a second ``execute`` before the previous
  one completed still raises ExecutionStateError.
"""
from __future__ import annotations

import threading
import time

import numpy as np

from . import _native as N
from .errors import CompileError, ExecutionStateError, WaitTimeout
from .executor import DeviceGraph, device_info
from .flat import FlatGraph
from .graph import AsyncNode, Copy, ExtPostcond, ExtPrecond, Task, TaskGraph, owners, to_flat
from .tasks import TaskRegistry, default_registry


MANUAL = object()  # execute(pre=[MANUAL, ...]): the caller triggers that precondition itself


class Event:
    """One-shot completion token backed by the device."""

    def __init__(self, poll, on_wait=None):
        self._poll = poll
        self._on_wait = on_wait
        self._done = False

    @staticmethod
    def triggered() -> "Event":
        e = Event(lambda: True)
        e._done = True
        return e

    def query(self) -> bool:
        if not self._done:
            self._done = bool(self._poll())
        return self._done

    @property
    def has_triggered(self) -> bool:
        return self.query()

    def wait(self, timeout: float | None = None) -> None:
        if self._on_wait is not None:
            self._on_wait(timeout)
            self._done = True
            return
        t0 = time.perf_counter()
        while not self.query():
            if timeout is not None and time.perf_counter() - t0 > timeout:
                raise WaitTimeout("event did not trigger in time")
            time.sleep(20e-6)


class CompiledGraph:
    """Per-resource worker programs resident on one GPU."""

    def __init__(self, flat: FlatGraph, resources: list, *, device: int = 0, source=None):
        self.flat = flat
        self.resources = resources
        self.source = source
        self.device = device
        info = device_info(device)
        if flat.n_workers > info["max_workers"]:
            raise CompileError(f"{flat.n_workers} workers exceed the {info['max_workers']} co-resident "
                               f"warps of {info['name']}; map resources onto fewer workers")
        self.n_ext_pre = int(flat.meta.get("n_ext_pre", 0))
        self.n_ext_post = int(flat.meta.get("n_ext_post", 0))
        self.dev = DeviceGraph(flat, device, n_ext_pre=self.n_ext_pre, n_ext_post=self.n_ext_post)
        self._outstanding = False
        self._lock = threading.RLock()
        self._last_flags = 0

    # -- Alg. 1 Execute ---------------------------------------------------
    def execute(self, pre=(), *, seed: int = 0, flags: int = N.TD_F_CHECKSUM | N.TD_F_STATS,
                spin_limit: int = 0):
        """Send INIT to every worker = one persistent-kernel launch.
        Returns (done, post) events."""
        pre = list(pre)
        if len(pre) != self.n_ext_pre:
            raise ExecutionStateError(f"expected {self.n_ext_pre} preconditions, got {len(pre)}")
        with self._lock:
            if self._outstanding and not self.dev.query():
                raise ExecutionStateError("an execution of this compiled graph is outstanding")
            if self._outstanding:
                self._finish(None)
            self.dev.launch(seed, flags=flags, spin_limit=spin_limit)
            self._outstanding = True
            self._last_flags = flags
        for i, ev in enumerate(pre):
            if ev is MANUAL:
                continue
            if ev is None or (hasattr(ev, "query") and ev.query()):
                self.dev.trigger_pre(i)
            else:
                threading.Thread(target=self._forward_pre, args=(i, ev), daemon=True).start()
        done = Event(self.dev.query, on_wait=self._finish)
        post = [Event(lambda j=j: self.dev.post_fired(j)) for j in range(self.n_ext_post)]
        return done, post

    def trigger_pre(self, i: int) -> None:
        """Trigger external precondition i of the outstanding execution."""
        self.dev.trigger_pre(i)

    def _forward_pre(self, i: int, ev) -> None:
        ev.wait()
        self.dev.trigger_pre(i)

    def _finish(self, timeout) -> None:
        with self._lock:
            if not self._outstanding:
                return
            try:
                self.dev.wait(timeout)
            finally:
                self._outstanding = False

    def wait(self, timeout: float | None = None) -> None:
        self._finish(timeout)

    # -- results --------------------------------------------------------------
    def message_stats(self) -> dict:
        """{cross_worker_messages, local_decrements, init_messages} of the last
        execution; requires the default TD_F_STATS flag."""
        s = self.dev.stats()
        return dict(cross_worker_messages=int(s["cross_worker_edges"]),
                    local_decrements=int(s["local_decrements"]),
                    init_messages=int(s["init_messages"]))

    def tokens(self) -> np.ndarray:
        return self.dev.tokens()

    def checksums(self) -> np.ndarray:
        return self.dev.checksums()

    def close(self) -> None:
        self.dev.close()


def compile(g, *, registry: TaskRegistry | None = None, device: int = 0) -> CompiledGraph:
    """Alg. 1 Compile.

    ``g`` is a validated :class:`TaskGraph` (tasks must be registered with a
    DeviceBody) or an already-flattened :class:`FlatGraph` (Task Bench)."""
    if isinstance(g, FlatGraph):
        return CompiledGraph(g, [("worker", w) for w in range(g.n_workers)], device=device)
    if not isinstance(g, TaskGraph):
        raise CompileError("compile() takes a TaskGraph or FlatGraph")
    reg = registry or default_registry()
    kind = np.zeros(g.n, np.uint8)
    arg = np.zeros(g.n, np.uint32)
    for v, x in enumerate(g.nodes):
        if isinstance(x, AsyncNode):
            raise CompileError("graph has async nodes: compile it with hybrid.HybridGraph")
        if isinstance(x, Task):
            if x.proc < 0:
                raise CompileError(f"node {v}: invalid processor {x.proc}")
            b = reg.device_body(x.tid)
            kind[v], arg[v] = b.kind, b.arg
        elif not isinstance(x, (Copy, ExtPrecond, ExtPostcond)):
            raise CompileError(f"node {v}: unknown kind")
    own, rs = owners(g)
    flat = to_flat(g, kind, arg, own, len(rs) if g.n else 0)
    return CompiledGraph(flat, rs, device=device, source=g)


def execute(cg: CompiledGraph, pre=(), **kw):
    return cg.execute(pre, **kw)


def message_stats(cg: CompiledGraph) -> dict:
    return cg.message_stats()

"""CPU reference executor: Alg. 1 on the reference's machine substrate —
TEST INFRASTRUCTURE / CPU BASELINE ONLY.

The reference artifact specifies but does not implement its compiler and
actor runtime.  This module restates them on the reference's
real, unmodified substrate ``taskdual.machine`` (machine.py:305-465) so the
GPU executor can be checked against, and timed beside, the reference design:

* actor runtime: ``register_actor(behavior, aid, proc)``
  pins an actor to a processor context; ``send_message`` is
  ``Machine.deliver`` (machine.py:364-371), whose handler runs on the target
  context's thread (``Context._run``, machine.py:111-120).  Handlers of one
  actor are serial because a context is one thread.
* compiler (Alg. 1 632-693):
  ``compile`` partitions nodes by resource, builds each
  worker's edge index with per-node counters initialised to in-degree; the
  interpreter handles INIT / COMPLETED_EDGE / EXECUTE_OP
  with SPEC.md's design decisions: counters re-armed at zero (412), one
  outstanding execution (413), local successors decremented directly and
  counted separately (414), EXECUTE_OP self-dispatch queued (424).
* message_stats.

Task bodies compute the token of oracle/tokens.py.  BUSY_WAIT bodies use the
reference's own ``precise_sleep`` (machine.py:45-62); COMPUTE bodies run the
literal 64-lane LCG loop in C through ctypes (which releases the GIL, so
bodies on different processors really run in parallel).
"""
from __future__ import annotations

import os
import threading
import time

import numpy as np

from . import seq, tokens as T
from .substrate import load as _load_substrate

INIT, COMPLETED_EDGE, EXECUTE_OP = 0, 1, 2


class ActorRuntime:
    """Minimal Fig. 3 actor runtime over taskdual.machine."""

    def __init__(self, machine, errors):
        self.machine = machine
        self.errors = errors
        self._actors = {}
        self.messages = 0
        self._lock = threading.Lock()

    def register_actor(self, behavior, aid: int, proc: int) -> None:
        if aid in self._actors:
            raise self.errors.RegistrationError(f"actor {aid} already registered")
        self._actors[aid] = (behavior, self.machine.processor(proc))

    def send_message(self, aid: int, mid: int, payload=None) -> None:
        behavior, ctx = self._actors[aid]
        self.machine.deliver(ctx, lambda: behavior.handle(mid, payload))

    def context_of(self, aid: int):
        return self._actors[aid][1]


class Worker:
    """Alg. 1 ``class Worker(r, (V, E))``."""

    def __init__(self, cg: "CompiledGraph", r: int, nodes: np.ndarray):
        self.cg = cg
        self.r = r
        self.nodes = nodes
        ind = cg.indeg
        self.indeg = {int(v): int(ind[v]) for v in nodes}
        # linearizable counters: a lock per worker
        self.ctr = dict(self.indeg)
        self.lock = threading.Lock()
        self.cross = 0
        self.local = 0

    def handle(self, mid: int, payload) -> None:
        if mid == INIT:
            for v in self.nodes:  # "Start all ready to execute work."
                if self.indeg[int(v)] == 0:
                    self.cg.rt.send_message(self.r, EXECUTE_OP, int(v))
        elif mid == COMPLETED_EDGE:
            self.decrement(payload[1])
        elif mid == EXECUTE_OP:
            self.execute(payload)

    def decrement(self, dst: int) -> None:
        with self.lock:
            c = self.ctr[dst] - 1
            if c < 0:
                raise RuntimeError(f"counter underflow at node {dst}")
            if c == 0:
                c = self.indeg[dst]  # re-arm
                fire = True
            else:
                fire = False
            self.ctr[dst] = c
        if fire:
            self.cg.rt.send_message(self.r, EXECUTE_OP, dst)  # queued self-dispatch

    def execute(self, v: int) -> None:
        cg = self.cg
        tok = cg.tokens
        preds = cg.preds[v]
        acc = 0
        for u in preds:
            acc += T.term_int(tok[u], u)
        h = T.mix64_int(T.mix64_int(cg.seed ^ T.mix64_int(v + T.G1)) ^ acc)
        kind = int(cg.kind[v])
        r = 0
        if kind == T.BODY_COMPUTE:
            r = seq.compute_loop(h, int(cg.arg[v]))
        elif kind == T.BODY_BUSY_WAIT:
            cg.precise_sleep(int(cg.arg[v]) * 1e-9)
        tok[v] = h ^ r
        for d in cg.succs[v]:
            o = int(cg.owner[d])
            if o == self.r:
                self.local += 1
                self.decrement(d)  # direct linearizable decrement
            else:
                self.cross += 1
                cg.rt.send_message(o, COMPLETED_EDGE, (v, d))
        cg.node_done()


class CompiledGraph:
    """SPEC.md CompiledGraph (360-363) on the CPU substrate."""

    def __init__(self, machine, errors, precise_sleep, n, preds, succs, owner, kind=None, arg=None):
        self.machine = machine
        self.errors = errors
        self.precise_sleep = precise_sleep
        self.n = n
        self.preds = preds
        self.succs = succs
        self.owner = np.asarray(owner)
        self.indeg = np.array([len(p) for p in preds], dtype=np.int64)
        self.kind = np.zeros(n, np.uint8) if kind is None else np.asarray(kind)
        self.arg = np.zeros(n, np.uint32) if arg is None else np.asarray(arg)
        self.rt = ActorRuntime(machine, errors)
        self.workers = {}
        for r in sorted(set(int(x) for x in self.owner)):  # resources used by G
            w = Worker(self, r, np.flatnonzero(self.owner == r))
            self.workers[r] = w
            self.rt.register_actor(w, r, r)  # RegisterActor(Worker(r,(V_w,E_w)), r)
        self.tokens = [0] * n
        self._done = threading.Event()
        self._count = 0
        self._count_lock = threading.Lock()
        self._outstanding = False
        self.seed = 0

    def node_done(self) -> None:
        with self._count_lock:
            self._count += 1
            if self._count == self.n:
                self._done.set()

    def execute(self, seed: int = 0) -> threading.Event:
        """Alg. 1 Execute: INIT to every worker."""
        if self._outstanding and not self._done.is_set():
            raise self.errors.ExecutionStateError("execution outstanding")
        self.seed = seed & T.M64
        self._done.clear()
        self._count = 0
        for w in self.workers.values():
            w.cross = w.local = 0
        self._outstanding = True
        if self.n == 0:
            self._done.set()
        for r in self.workers:
            self.rt.send_message(r, INIT)
        return self._done

    def wait(self, timeout: float | None = None) -> None:
        if not self._done.wait(timeout):
            raise self.errors.WaitTimeout("execution did not finish")
        errs = self.machine.context_errors()
        if errs:
            raise self.errors.ExecutionPoisoned(str(errs[0][1]))
        self._outstanding = False

    def message_stats(self) -> dict:
        return dict(cross_worker_messages=sum(w.cross for w in self.workers.values()),
                    local_decrements=sum(w.local for w in self.workers.values()),
                    init_messages=len(self.workers))


def compile_flat(machine, n, pred_rows, owner, kind=None, arg=None):
    m, e, _ = _load_substrate()
    succs = [[] for _ in range(n)]
    for v in range(n):
        for u in pred_rows[v]:
            succs[u].append(v)
    return CompiledGraph(machine, e, m.precise_sleep, n, pred_rows, succs, owner, kind, arg)


def run_flat(n, pred_rows, owner, kind=None, arg=None, seed=0, processors=None, reps=1,
             timeout=None):
    """Run Alg. 1 on a fresh taskdual Machine; returns (tokens, stats, [secs])."""
    m, e, _ = _load_substrate()
    P = int(max(owner) + 1) if processors is None else processors
    times = []
    with m.create_machine(m.MachineSpec(processor_count=max(1, P))) as mach:
        cg = compile_flat(mach, n, pred_rows, owner, kind, arg)
        for _ in range(reps):
            t0 = time.perf_counter()
            cg.execute(seed)
            cg.wait(timeout)
            times.append(time.perf_counter() - t0)
        return np.array(cg.tokens, dtype=np.uint64), cg.message_stats(), times


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def run_sweep(n, pred_rows, owner, kind, iterations, processors=None, warmups=1, reps=3, seed=0,
              plateau=4, tol=0.03, check=None):
    """Granularity sweep of the COMPUTE body on ONE compiled graph (the CPU
    reference's METG curve): for each iteration count, the
    median wall of `reps` executions after `warmups`.  Stops once `plateau`
    consecutive points' rates agree within `tol`.  `check(iters, tokens)`
    (optional) validates one execution's tokens per point.
    Returns [(iters, median_seconds, check_ok or None)]."""
    m, e, _ = _load_substrate()
    P = int(max(owner) + 1) if processors is None else processors
    out = []
    with m.create_machine(m.MachineSpec(processor_count=max(1, P))) as mach:
        cg = compile_flat(mach, n, pred_rows, owner, kind, np.zeros(n, np.uint32))
        is_compute = np.asarray(cg.kind) == T.BODY_COMPUTE
        for it in iterations:
            cg.arg = np.where(is_compute, it, 0).astype(np.uint32)
            ts = []
            for r in range(warmups + reps):
                t0 = time.perf_counter()
                cg.execute(seed)
                cg.wait()
                if r >= warmups:
                    ts.append(time.perf_counter() - t0)
            ok = None if check is None else bool(check(it, np.array(cg.tokens, dtype=np.uint64)))
            out.append((int(it), float(np.median(ts)), ok))
            if plateau and len(out) >= plateau:
                rates = [i * 64 / t for i, t, _ in out[-plateau:]]
                if max(rates) <= (1 + tol) * min(rates):
                    break
    return out


def compute_peak(processors: int, iters: int = 1 << 16, calls: int = 8, reps: int = 3) -> dict:
    """The CPU's peak for the compute_bound body's unit of work (lane-updates
    per second): `processors` threads each run the literal 64-lane LCG body
    (seq_oracle.c, called through ctypes, which releases the GIL) back to
    back, with no runtime around it.  The fixed METG denominator of the CPU
    reference's curve (efficiency vs the machine's peak)."""
    def work(k):
        for c in range(calls):
            seq.compute_loop(k * 7919 + c, iters)
    seq.compute_loop(1, 16)  # load the library before timing
    best = 0.0
    for _ in range(reps):
        th = [threading.Thread(target=work, args=(k,)) for k in range(processors)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        best = max(best, processors * calls * iters * 64 / (time.perf_counter() - t0))
    return {"lane_updates_per_s": best, "threads": processors, "reps": reps,
            "body": "seq_oracle.c td_oracle_compute_loop (64 lanes x iters u64 LCG), gcc -O2; best of reps"}

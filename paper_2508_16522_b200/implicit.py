"""Implicitly-parallel frontend with tracing (SPEC.md implicit 427-493;
PAPER.md §5 803-871).

* ``issue`` computes dependences from declared region accesses with the
  last-conflict rule: a reader depends on the last writer
  of the region; a writer depends on every reader since the last write, or on
  the last writer when there were none (edges transitively reduced per
  region, so A:w B:r C:r D:w gives {A->B, A->C, B->D, C->D}).  Untraced ops execute immediately through the per-task launch
  runtime (``td_rt_launch_task``: one kernel per task, the generic path).
* ``begin_trace``/``end_trace`` record the op sequence and its memoized
  edges.  Re-beginning a recorded trace id enters replay
  mode: the ops issued must match the recording (else TraceError,
  SPEC.md:482) and the trace is replayed at ``end_trace``.
* ``replay(tid, mode, plan)``: ``memoized`` re-issues the
  recorded ops with the stored edges through the per-task runtime (no
  re-analysis); ``compiled`` lowers the trace once to a CompiledGraph (the
  persistent kernel) and replays it with one launch.

Memory model on the GPU: each op produces a 64-bit token (oracle/tokens.py)
from its trace-local index and its in-trace predecessors; a region's value is
the token of its last writer.  The three execution modes therefore yield
identical region images.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import ResourceError, TraceError
from .flat import FlatGraph, IntervalCSR, transpose
from .shard import ShardingPlan, lowering_stats, node_shards
from .tasks import TaskRegistry, default_registry

READ, WRITE, READWRITE = "read", "write", "readwrite"


@dataclass(frozen=True)
class AccessDecl:
    region: int
    privilege: str = READ


@dataclass
class IssuedOp:
    seq: int
    tid: int
    proc: int
    args: bytes = b""
    accesses: tuple = ()

    def signature(self):
        return (self.tid, self.proc, self.args, self.accesses)


@dataclass
class Trace:
    tid: int
    ops: list = field(default_factory=list)
    edges: set = field(default_factory=set)    # (i, j) trace-local indices
    state: str = "recording"                    # recording | recorded
    compiled: object = None
    lowering: dict | None = None
    writes: dict = field(default_factory=dict)  # region -> last writer (local idx)
    readers: dict = field(default_factory=dict) # region -> readers since (local idx)
    slots: list = field(default_factory=list)   # token slot of each op (recording)
    rt_slots: list | None = None                # runtime slots standing for a compiled replay's outputs
    imported: bool = False                      # rt_slots hold the compiled replay's tokens


class _Rt:
    """ctypes owner of a td_rt (per-task launch runtime)."""

    def __init__(self, device: int, capacity: int):
        h = C.c_void_p()
        N.check(N.lib().td_rt_create(device, capacity, C.byref(h)))
        self._h = h
        self.capacity = capacity

    def launch(self, slot, key, kind, arg, seed, preds):
        arr = np.ascontiguousarray(preds, dtype=np.int64)
        N.check(N.lib().td_rt_launch_task(self._h, slot, key, kind, arg, seed,
                                          arr.ctypes.data_as(C.c_void_p), len(arr)))

    def sync(self):
        N.check(N.lib().td_rt_sync(self._h))

    def store(self, slots, keys, tokens):
        sl = np.ascontiguousarray(slots, dtype=np.int64)
        ky = np.ascontiguousarray(keys, dtype=np.uint64)
        tk = np.ascontiguousarray(tokens, dtype=np.uint64)
        N.check(N.lib().td_rt_store_tokens(self._h, sl.ctypes.data_as(C.c_void_p), ky.ctypes.data_as(C.c_void_p),
                                           tk.ctypes.data_as(C.c_void_p), len(sl)))

    def tokens(self, first, n):
        out = np.empty(n, dtype=np.uint64)
        N.check(N.lib().td_rt_tokens(self._h, first, n, out.ctypes.data_as(C.c_void_p)))
        return out

    def close(self):
        if self._h.value:
            N.lib().td_rt_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ImplicitRuntime:
    """Single host context drives issue/begin/end/replay."""

    def __init__(self, registry: TaskRegistry | None = None, device: int = 0, capacity: int = 1 << 20,
                 seed: int = 0):
        self.registry = registry or default_registry()
        self.device = device
        self.seed = seed
        self._rt = _Rt(device, capacity)
        self._n_regions = 0
        self._seq = 0
        # dynamic analysis state over slots of the untraced token store
        self._last_writer: dict[int, int] = {}
        self._readers: dict[int, list] = {}
        self._slot_of_seq: dict[int, int] = {}
        self._next_slot = 0
        self._traces: dict[int, Trace] = {}
        self._active: Trace | None = None
        self._replay_pos = None
        self.region_value: dict[int, tuple] = {}   # region -> (mode, slot or node)
        self._last_compiled = None
        # slots standing for outputs of a compiled replay whose tokens have not
        # been imported into the runtime yet: slot -> trace id
        self._pending: dict[int, int] = {}

    # -- regions --------------------------------------------------------------
    def region(self) -> int:
        self._n_regions += 1
        return self._n_regions - 1

    def _check_regions(self, accesses):
        out = []
        for a in accesses:
            a = a if isinstance(a, AccessDecl) else AccessDecl(*a)
            if not 0 <= a.region < self._n_regions:
                raise ResourceError(f"unknown region {a.region}")
            if a.privilege not in (READ, WRITE, READWRITE):
                raise ResourceError(f"bad privilege {a.privilege!r}")
            out.append(a)
        return tuple(out)

    # -- dependence analysis (last-conflict rule) -----------------------------
    @staticmethod
    def analyze(accesses, last_writer: dict, readers: dict, me: int) -> set:
        deps = set()
        for a in accesses:
            r = a.region
            lw = last_writer.get(r)
            if a.privilege == READ:
                if lw is not None:
                    deps.add(lw)
            else:
                # readers since the last write already depend on it, so the
                # writer->last-writer edge is implied (per-region transitive
                # reduction; KAT SPEC.md:456)
                rs = readers.get(r, [])
                if rs:
                    deps.update(rs)
                elif lw is not None:
                    deps.add(lw)
        for a in accesses:
            r = a.region
            if a.privilege == READ:
                readers.setdefault(r, []).append(me)
            else:
                last_writer[r] = me
                readers[r] = []
        deps.discard(me)
        return deps

    # -- issue ------------------------------------------------------------------
    def issue(self, tid: int, proc: int = 0, args: bytes = b"", accesses=()):
        body = self.registry.device_body(tid)
        acc = self._check_regions(accesses)
        op = IssuedOp(self._seq, tid, proc, args, acc)
        self._seq += 1
        tr = self._active
        if tr is not None and tr.state == "recorded":  # replay mode: validate only
            i = self._replay_pos
            if i >= len(tr.ops) or tr.ops[i].signature() != op.signature():
                raise TraceError(f"op {i} differs from the recorded trace {tr.tid}")
            self._replay_pos += 1
            return None
        # untraced execution (also the recording iteration)
        slot = self._alloc_slot()
        deps = self.analyze(acc, self._last_writer, self._readers, slot)
        if tr is not None:
            local = len(tr.ops)
            tr.ops.append(op)
            tdeps = self.analyze(acc, tr.writes, tr.readers, local)
            tr.edges.update((d, local) for d in tdeps)
            key, preds = local, [tr.slots[d] for d in sorted(tdeps)]
            tr.slots.append(slot)
        else:
            key, preds = op.seq, [s for s in sorted(deps)]
            self._materialize(preds)
        self._rt.launch(slot, key, body.kind, body.arg, self.seed, preds)
        for a in acc:
            if a.privilege != READ:
                self.region_value[a.region] = ("slot", slot)
        return slot

    def _after_replay(self, tr: Trace, slots) -> None:
        """A replay re-defines the regions its ops write: later untraced ops
        must depend on the replayed ops (slots), not on whatever last wrote
        those regions before the replay (last-conflict rule)."""
        for i, o in enumerate(tr.ops):
            self.analyze(o.accesses, self._last_writer, self._readers, slots[i])

    def _materialize(self, preds) -> None:
        """Import the tokens of compiled replays that untraced ops are about to
        read into their runtime slots (once per trace: a trace's tokens depend
        only on the seed and its own ops)."""
        tids = {self._pending[p] for p in preds if p in self._pending}
        for tid in tids:
            tr = self._traces[tid]
            cg = tr.compiled
            if hasattr(cg, "wait"):
                cg.wait()
            tok = cg.tokens()
            n = len(tr.ops)
            self._rt.store(tr.rt_slots, np.arange(n, dtype=np.uint64), tok[:n])
            tr.imported = True
            for sl in tr.rt_slots:
                self._pending.pop(sl, None)

    def _alloc_slot(self) -> int:
        if self._next_slot >= self._rt.capacity:
            raise ResourceError("token store exhausted")
        self._next_slot += 1
        return self._next_slot - 1

    # -- trace demarcation --------------------------------------------------------
    def begin_trace(self, tid: int) -> None:
        if self._active is not None:
            raise TraceError("nested traces are not allowed")
        tr = self._traces.get(tid)
        if tr is None:
            tr = Trace(tid)
            self._traces[tid] = tr
        else:
            self._replay_pos = 0
        self._active = tr

    def end_trace(self, tid: int):
        tr = self._active
        if tr is None or tr.tid != tid:
            raise TraceError("end_trace without a matching begin_trace")
        self._active = None
        if tr.state == "recording":
            tr.state = "recorded"
            return None
        if self._replay_pos != len(tr.ops):
            raise TraceError("replayed op sequence is shorter than the recording")
        self._replay_pos = None
        return self.replay(tid, "compiled")

    # -- replay ----------------------------------------------------------------------
    def trace_graph(self, tid: int, n_workers: int | None = None) -> FlatGraph:
        tr = self._require(tid)
        n = len(tr.ops)
        src = np.array([a for a, _ in sorted(tr.edges)], dtype=np.int64)
        dst = np.array([b for _, b in sorted(tr.edges)], dtype=np.int64)
        pred = IntervalCSR.from_edges(n, dst, src)
        procs = sorted({o.proc for o in tr.ops})
        pidx = {p: i for i, p in enumerate(procs)}
        kind = np.zeros(n, np.uint8)
        arg = np.zeros(n, np.uint32)
        for i, o in enumerate(tr.ops):
            b = self.registry.device_body(o.tid)
            kind[i], arg[i] = b.kind, b.arg
        return FlatGraph(n=n, pred=pred, succ=transpose(pred), kind=kind, arg=arg,
                         worker=np.array([pidx[o.proc] for o in tr.ops], np.int32),
                         n_workers=max(1, len(procs)), order=np.arange(n, dtype=np.int64),
                         meta=dict(procs=procs))

    def _require(self, tid) -> Trace:
        tr = self._traces.get(tid)
        if tr is None or tr.state != "recorded":
            raise TraceError(f"trace {tid} is not recorded")
        return tr

    def replay(self, tid: int, mode: str = "compiled", plan: ShardingPlan | None = None):
        """Returns the done Event (compiled) or None after the per-task launches
        were issued (memoized); region_value is updated either way."""
        tr = self._require(tid)
        if mode == "memoized":
            base = []
            for i, o in enumerate(tr.ops):
                slot = self._alloc_slot()
                base.append(slot)
            preds_of = {}
            for a, b in tr.edges:
                preds_of.setdefault(b, []).append(a)
            for i, o in enumerate(tr.ops):
                body = self.registry.device_body(o.tid)
                self._rt.launch(base[i], i, body.kind, body.arg, self.seed,
                                [base[d] for d in sorted(preds_of.get(i, []))])
                for a in o.accesses:
                    if a.privilege != READ:
                        self.region_value[a.region] = ("slot", base[i])
            self._after_replay(tr, base)
            return None
        if mode != "compiled":
            raise TraceError(f"unknown replay mode {mode!r}")
        if tr.compiled is None:
            from .compiler import compile as td_compile
            g = self.trace_graph(tid)
            if plan is not None:
                procs = g.meta["procs"]
                if len(plan.shard_of_worker) != len(procs):
                    raise ResourceError("plan references unknown processors")
                tr.lowering = lowering_stats(g, node_shards(g, plan))
            else:
                tr.lowering = dict(ext_pairs=0, nodes_per_shard=[g.n])
            if plan is not None and plan.devices and len(set(plan.devices)) > 1:
                # sharded lowering onto several GPUs of this process
                from .shard import InProcessShards
                tr.compiled = InProcessShards(g, plan, plan.devices)
            else:
                tr.compiled = td_compile(g, device=self.device)
        if hasattr(tr.compiled, "shards"):
            tr.compiled.run(self.seed)
            from .compiler import Event
            done = Event.triggered()
        else:
            done, _ = tr.compiled.execute(seed=self.seed, flags=0)
        for i, o in enumerate(tr.ops):
            for a in o.accesses:
                if a.privilege != READ:
                    self.region_value[a.region] = ("trace", tid, i)
        if tr.rt_slots is None:
            tr.rt_slots = [self._alloc_slot() for _ in tr.ops]
        if not tr.imported:
            for sl in tr.rt_slots:
                self._pending[sl] = tid
        self._after_replay(tr, tr.rt_slots)
        self._last_compiled = tr.compiled
        return done

    # -- state --------------------------------------------------------------------------
    def memory_image(self) -> dict:
        """region -> token of its last writer (machine.py:395-397 analogue)."""
        self._rt.sync()
        out = {}
        cache = {}
        for r, loc in self.region_value.items():
            if loc[0] == "slot":
                out[r] = int(self._rt.tokens(loc[1], 1)[0])
            else:
                _, tid, i = loc
                if tid not in cache:
                    cg = self._traces[tid].compiled
                    if hasattr(cg, "wait"):
                        cg.wait()
                    cache[tid] = cg.tokens()
                out[r] = int(cache[tid][i])
        return out

    def save_trace(self, tid: int, path: str) -> None:
        """Trace dump to the on-disk graph format: the
        recorded ops' flattened graph as .npz (bodies resolved to device kinds)."""
        from .flat import save_npz
        save_npz(self.trace_graph(tid), path)

    def ext_pairs(self, tid: int) -> int:
        tr = self._require(tid)
        return 0 if tr.lowering is None else tr.lowering["ext_pairs"]

    def close(self) -> None:
        for tr in self._traces.values():
            if tr.compiled is not None:
                tr.compiled.close()
        self._rt.close()

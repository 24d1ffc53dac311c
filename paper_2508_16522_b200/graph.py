"""Static task-graph IR with external conditions (SPEC.md graph module 285-349;
PAPER.md §4.1 564-584, draft Operation/SubgraphDefn 1604-1660).

Node kinds, ``build`` with its validation (cycle, ext-degree, dangling edge,
duplicate edge), lowering to the flat interval CSR the
executor uploads (:func:`to_flat`), and the graph passes of SURVEY §8(f):
serialization (``to_json``/``from_json``/``to_dot``), ``transitive_reduce``
and ``async_transform`` (host-side / device-side split, §4.3
776-801; executed by :mod:`.hybrid`).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Union

import numpy as np

from .errors import GraphError
from .flat import (FlatGraph, IntervalCSR, KIND_EMPTY, KIND_EXT_POST, KIND_EXT_PRE, topological_rank,
                   transpose)


@dataclass(frozen=True)
class Task:
    """Task{proc, tid, args}.  ``device_work``: the task's
    operation launches asynchronous device work."""
    proc: int
    tid: int
    args: bytes = b""
    device_work: bool = False


@dataclass(frozen=True)
class AsyncNode:
    """The asynchronous (device-side) work of node ``of``, added by
    :func:`async_transform` ("we add a new async node")."""
    of: int


@dataclass(frozen=True)
class Copy:
    """Copy{src, dst}: bound to the (src, dst) memory channel resource."""
    src_memory: int
    dst_memory: int
    size: int = 0


@dataclass(frozen=True)
class ExtPrecond:
    """External precondition i: in-degree 0."""
    index: int


@dataclass(frozen=True)
class ExtPostcond:
    """External postcondition j: out-degree 0."""
    index: int


NodeKind = Union[Task, Copy, ExtPrecond, ExtPostcond, AsyncNode]
EDGE_KINDS = ("host", "async", "sync", "launch")


@dataclass(frozen=True)
class TaskGraph:
    """Immutable validated DAG."""
    nodes: tuple
    edges: tuple            # sorted (src, dst) pairs
    n_ext_pre: int = 0
    n_ext_post: int = 0
    pred: IntervalCSR = field(default=None, compare=False, repr=False)
    succ: IntervalCSR = field(default=None, compare=False, repr=False)
    rank: np.ndarray = field(default=None, compare=False, repr=False)
    edge_kinds: tuple = ()  # aligned with edges; () = all "host"

    @property
    def n(self) -> int:
        return len(self.nodes)

    def edge_kind(self, i: int) -> str:
        return self.edge_kinds[i] if self.edge_kinds else "host"


def build(nodes, edges) -> TaskGraph:
    """build(nodes, edges) -> TaskGraph or GraphError.
    An edge is (src, dst) or (src, dst, kind), kind in EDGE_KINDS."""
    nodes = tuple(nodes)
    n = len(nodes)
    for x in nodes:
        if not isinstance(x, (Task, Copy, ExtPrecond, ExtPostcond, AsyncNode)):
            raise GraphError(f"unknown node kind {x!r}")
    ekind = {}
    e = []
    for ed in edges:
        a, b = int(ed[0]), int(ed[1])
        k = ed[2] if len(ed) > 2 else "host"
        if k not in EDGE_KINDS:
            raise GraphError(f"unknown edge kind {k!r}")
        e.append((a, b))
        ekind[(a, b)] = k
    for a, b in e:
        if not (0 <= a < n and 0 <= b < n):
            raise GraphError(f"dangling edge ({a}, {b})")
        if a == b:
            raise GraphError(f"self edge on node {a}: cycle detected")
    if len(set(e)) != len(e):
        raise GraphError("duplicate edge")
    src = np.array([a for a, _ in e], dtype=np.int64)
    dst = np.array([b for _, b in e], dtype=np.int64)
    indeg = np.bincount(dst, minlength=n) if n else np.zeros(0, np.int64)
    outdeg = np.bincount(src, minlength=n) if n else np.zeros(0, np.int64)
    pre_idx, post_idx = [], []
    for v, x in enumerate(nodes):
        if isinstance(x, ExtPrecond):
            if indeg[v]:
                raise GraphError(f"ExtPrecond node {v} has incoming edges")
            pre_idx.append(x.index)
        if isinstance(x, ExtPostcond):
            if outdeg[v]:
                raise GraphError(f"ExtPostcond node {v} has outgoing edges")
            post_idx.append(x.index)
    for name, idx in (("ExtPrecond", pre_idx), ("ExtPostcond", post_idx)):
        if sorted(idx) != list(range(len(idx))):
            raise GraphError(f"{name} indices must be dense 0..k-1, got {sorted(idx)}")
    for v, x in enumerate(nodes):
        if isinstance(x, AsyncNode) and not (0 <= x.of < n and isinstance(nodes[x.of], Task)):
            raise GraphError(f"async node {v} refers to {x.of}, which is not a task")
    pred = IntervalCSR.from_edges(n, dst, src)
    succ = transpose(pred)
    rank = topological_rank(pred, succ)  # raises GraphError on a cycle
    se = tuple(sorted(e))
    kinds = tuple(ekind[x] for x in se) if any(k != "host" for k in ekind.values()) else ()
    return TaskGraph(nodes, se, len(pre_idx), len(post_idx), pred, succ, rank, kinds)


def resources(g: TaskGraph) -> list:
    """'all processors and memory channels used in G' (Alg. 1 Compile,
    PAPER.md:650-651): ('proc', p) and ('chan', src, dst), sorted."""
    rs = set()
    for x in g.nodes:
        if isinstance(x, Task):
            rs.add(("proc", x.proc))
        elif isinstance(x, AsyncNode):
            rs.add(("proc", g.nodes[x.of].proc))
        elif isinstance(x, Copy):
            rs.add(("chan", x.src_memory, x.dst_memory))
    return sorted(rs)


def owners(g: TaskGraph) -> tuple[np.ndarray, list]:
    """Owner resource index per node.  Tasks/copies: their resource.
    ExtPostcond: owner of its last predecessor in topological order, ties by
    lowest resource id.  ExtPrecond: owner of its first
    successor (the worker that receives its COMPLETED_EDGE messages)."""
    rs = resources(g)
    index = {r: i for i, r in enumerate(rs)}
    own = np.full(g.n, -1, dtype=np.int32)
    for v, x in enumerate(g.nodes):
        if isinstance(x, Task):
            own[v] = index[("proc", x.proc)]
        elif isinstance(x, AsyncNode):
            own[v] = index[("proc", g.nodes[x.of].proc)]
        elif isinstance(x, Copy):
            own[v] = index[("chan", x.src_memory, x.dst_memory)]
    # ext nodes: resolve in topological order (posts) / reverse (pres)
    order = np.argsort(g.rank)
    for v in order:
        x = g.nodes[v]
        if isinstance(x, ExtPostcond):
            preds = g.pred.row(int(v))
            if preds:
                last = max(g.rank[u] for u in preds)
                cands = [int(own[u]) for u in preds if g.rank[u] == last and own[u] >= 0]
                own[v] = min(cands) if cands else 0
    for v in order[::-1]:
        x = g.nodes[v]
        if isinstance(x, ExtPrecond):
            succs = g.succ.row(int(v))
            own[v] = min(int(own[s]) for s in succs if own[s] >= 0) if succs and (own[succs] >= 0).any() else 0
    if len(rs) == 0 and g.n:
        rs = [("proc", 0)]
    own[own < 0] = 0
    return own, rs


def to_flat(g: TaskGraph, kind: np.ndarray, arg: np.ndarray, owner: np.ndarray,
            n_workers: int) -> FlatGraph:
    """Lower a validated TaskGraph to the executor's flat form."""
    k = np.array(kind, dtype=np.uint8)
    a = np.array(arg, dtype=np.uint32)
    for v, x in enumerate(g.nodes):
        if isinstance(x, ExtPrecond):
            k[v], a[v] = KIND_EXT_PRE, x.index
        elif isinstance(x, ExtPostcond):
            k[v], a[v] = KIND_EXT_POST, x.index
        elif isinstance(x, Copy):
            k[v], a[v] = KIND_EMPTY, 0
    return FlatGraph(n=g.n, pred=g.pred, succ=g.succ, kind=k, arg=a,
                     worker=np.asarray(owner, np.int32), n_workers=max(1, n_workers),
                     order=g.rank, meta=dict(n_ext_pre=g.n_ext_pre, n_ext_post=g.n_ext_post))


# ---------------------------------------------------------------------------
# Graph file format: version, nodes[] {id, kind,
# proc|channel, tid, args_hex, device_work}, edges[] {src, dst, kind},
# ext_preconds, ext_postconds.  Round-trip identity.
# ---------------------------------------------------------------------------
FORMAT_VERSION = 1


def to_json(g: TaskGraph) -> str:
    import json
    nodes = []
    for v, x in enumerate(g.nodes):
        if isinstance(x, Task):
            nodes.append({"id": v, "kind": "task", "proc": x.proc, "tid": x.tid, "args_hex": x.args.hex(),
                          "device_work": x.device_work})
        elif isinstance(x, AsyncNode):
            nodes.append({"id": v, "kind": "async", "of": x.of})
        elif isinstance(x, Copy):
            nodes.append({"id": v, "kind": "copy", "channel": [x.src_memory, x.dst_memory], "size": x.size})
        elif isinstance(x, ExtPrecond):
            nodes.append({"id": v, "kind": "ext_pre", "index": x.index})
        else:
            nodes.append({"id": v, "kind": "ext_post", "index": x.index})
    doc = {"version": FORMAT_VERSION, "nodes": nodes,
           "edges": [{"src": a, "dst": b, "kind": g.edge_kind(i)} for i, (a, b) in enumerate(g.edges)],
           "ext_preconds": g.n_ext_pre, "ext_postconds": g.n_ext_post}
    return json.dumps(doc, indent=1)


def from_json(text: str) -> TaskGraph:
    """Parse + validate; malformed text raises GraphParseError with line/column."""
    import json
    from .errors import GraphParseError
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise GraphParseError(f"malformed graph file: {e.msg}", e.lineno, e.colno) from None
    try:
        if doc.get("version") != FORMAT_VERSION:
            raise GraphParseError(f"unsupported graph format version {doc.get('version')!r}")
        raw = sorted(doc["nodes"], key=lambda d: d["id"])
        if [d["id"] for d in raw] != list(range(len(raw))):
            raise GraphParseError("node ids must be dense 0..n-1")
        nodes = []
        for d in raw:
            k = d["kind"]
            if k == "task":
                nodes.append(Task(int(d["proc"]), int(d["tid"]), bytes.fromhex(d.get("args_hex", "")),
                                  bool(d.get("device_work", False))))
            elif k == "async":
                nodes.append(AsyncNode(int(d["of"])))
            elif k == "copy":
                src, dst = d["channel"]
                nodes.append(Copy(int(src), int(dst), int(d.get("size", 0))))
            elif k == "ext_pre":
                nodes.append(ExtPrecond(int(d["index"])))
            elif k == "ext_post":
                nodes.append(ExtPostcond(int(d["index"])))
            else:
                raise GraphParseError(f"unknown node kind {k!r}")
        edges = [(int(e["src"]), int(e["dst"]), e.get("kind", "host")) for e in doc["edges"]]
    except (KeyError, TypeError, ValueError) as e:
        raise GraphParseError(f"malformed graph file: {e}") from None
    return build(nodes, edges)


def transitive_reduce(g: TaskGraph) -> TaskGraph:
    """Minimal edge set with the same reachability (PAPER.md
    §5 859-860).  Node set unchanged; runs in O(V*E/64) with bitset closures
    (intended for compile-time passes over traced graphs, not for the
    million-node Task Bench graphs, which are already reduced)."""
    n = g.n
    order = np.argsort(g.rank)              # topological order
    words = (n + 63) // 64
    reach = np.zeros((n, words), dtype=np.uint64)  # strict descendants
    succ = [g.succ.row(int(v)) for v in range(n)]
    keep = []
    for v in order[::-1]:
        v = int(v)
        # successors in topological order: an edge v->s is redundant if s is
        # reachable from another successor of v
        ss = sorted(succ[v], key=lambda x: g.rank[x])
        covered = np.zeros(words, dtype=np.uint64)
        for s in ss:
            bit = np.uint64(1) << np.uint64(s % 64)
            if not (covered[s // 64] & bit):
                keep.append((v, s))
            covered |= reach[s]
            covered[s // 64] |= bit
        reach[v] = covered
    kinds = {e: g.edge_kind(i) for i, e in enumerate(g.edges)}
    return build(g.nodes, [(a, b, kinds[(a, b)]) for a, b in sorted(keep)])


def reachability(g: TaskGraph) -> np.ndarray:
    """Boolean closure matrix (test helper for transitive_reduce)."""
    n = g.n
    R = np.zeros((n, n), dtype=bool)
    for v in np.argsort(g.rank)[::-1]:
        v = int(v)
        for s in g.succ.row(v):
            R[v, s] = True
            R[v] |= R[s]
    return R


def async_transform(g: TaskGraph) -> TaskGraph:
    """Decouple the host side of operations from their device work
    (§4.3 776-801, Fig. 9).

    For every task n with ``device_work`` an AsyncNode n_a is added.  For
    every original edge (n, d) leaving such a task: if d has d_a, an async
    edge (n_a, d_a) is added, else a sync edge (n_a, d).  Original host edges
    are retained.  Each n_a also gets a ``launch`` edge (n, n_a): the device
    work starts once its host side has issued it (the SPEC's examples list
    only the async/sync edges; the launch edge is this build's explicit
    rendering of "n launches n_a").  Nodes without device work pass through;
    the output is acyclic (every added edge leaves an async node or enters it
    from its own host node)."""
    n = g.n
    a_of = {}
    nodes = list(g.nodes)
    for v, x in enumerate(g.nodes):
        if isinstance(x, Task) and x.device_work:
            a_of[v] = len(nodes)
            nodes.append(AsyncNode(v))
    if not a_of:
        return g
    edges = [(a, b, g.edge_kind(i)) for i, (a, b) in enumerate(g.edges)]
    for v, av in a_of.items():
        edges.append((v, av, "launch"))
    for a, b in g.edges:
        if a in a_of:
            edges.append((a_of[a], a_of[b], "async") if b in a_of else (a_of[a], b, "sync"))
    del n
    return build(nodes, edges)


_DOT_SHAPE = {Task: "box", Copy: "ellipse", ExtPrecond: "invtriangle", ExtPostcond: "triangle",
              AsyncNode: "box"}
_DOT_EDGE = {"host": "solid", "async": "dashed", "sync": "dashed", "launch": "dotted"}


def to_dot(g: TaskGraph) -> str:
    """One dot node per graph node with a kind-specific shape; async nodes and
    async / sync edges dashed."""
    out = ["digraph taskgraph {"]
    for v, x in enumerate(g.nodes):
        if isinstance(x, Task):
            label = f"task {x.tid}@P{x.proc}" + (" (device)" if x.device_work else "")
        elif isinstance(x, Copy):
            label = f"copy {x.src_memory}->{x.dst_memory}"
        elif isinstance(x, ExtPrecond):
            label = f"pre {x.index}"
        elif isinstance(x, ExtPostcond):
            label = f"post {x.index}"
        else:
            label = f"async of {x.of}"
        style = ', style=dashed' if isinstance(x, AsyncNode) else ""
        out.append(f'  n{v} [shape={_DOT_SHAPE[type(x)]}, label="{label}"{style}];')
    for i, (a, b) in enumerate(g.edges):
        k = g.edge_kind(i)
        attrs = f"style={_DOT_EDGE[k]}" + (f', label="{k}"' if k != "host" else "")
        out.append(f"  n{a} -> n{b} [{attrs}];")
    out.append("}")
    return "\n".join(out) + "\n"

"""Flattened interval-CSR task graph: what the trace recorder emits and what the
C ABI uploads (include/tdexec.h ``td_csr``).

This replaces the reference's per-worker Python edge index (Alg. 1 "An edge
list pre-processed for O(1) lookup of edges"; SPEC.md
WorkerProgram 356-359) with flat arrays:

* node ids are dense ``int32``;
* predecessor and successor lists are stored as sorted, disjoint, inclusive
  id **intervals** ``(lo, hi)`` — Task Bench dependence sets are intervals, so
  all_to_all needs one interval per node instead of W ids;
* ``indeg`` counts every incoming edge (including ext-precondition edges,
  SPEC.md:357);
* ``kind``/``arg`` select the device body (tdexec.h ``TD_BODY_*``);
* ``worker`` is the static owner of each node (Alg. 1 ``V_w``),
  ``col`` the checksum column.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import GraphError

KIND_EMPTY = 0
KIND_BUSY_WAIT = 1
KIND_COMPUTE = 2
KIND_STENCIL2D = 3
KIND_EXT_PRE = 4   # waits for an external precondition flag, then completes
KIND_EXT_POST = 5  # completes, then raises an external postcondition flag
KIND_MEMORY = 6    # memory_bound: streams arg u64 words through the worker's scratch


@dataclass
class IntervalCSR:
    """Per-node lists of inclusive id intervals, ascending and disjoint."""

    ptr: np.ndarray  # int64[N+1]
    iv: np.ndarray   # int32[K, 2]  (lo, hi)

    @property
    def n(self) -> int:
        return len(self.ptr) - 1

    def degrees(self) -> np.ndarray:
        lens = (self.iv[:, 1].astype(np.int64) - self.iv[:, 0] + 1)
        out = np.zeros(self.n, dtype=np.int64)
        if len(lens):
            node = np.repeat(np.arange(self.n), np.diff(self.ptr))
            np.add.at(out, node, lens)
        return out

    def n_edges(self) -> int:
        return int((self.iv[:, 1].astype(np.int64) - self.iv[:, 0] + 1).sum()) if len(self.iv) else 0

    def row(self, v: int) -> list[int]:
        out: list[int] = []
        for k in range(self.ptr[v], self.ptr[v + 1]):
            lo, hi = self.iv[k]
            out.extend(range(int(lo), int(hi) + 1))
        return out

    def expand(self) -> tuple[np.ndarray, np.ndarray]:
        """Explicit (node, neighbour) arrays; only for graphs of modest size."""
        lens = (self.iv[:, 1].astype(np.int64) - self.iv[:, 0] + 1)
        total = int(lens.sum()) if len(lens) else 0
        node_of_iv = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.ptr))
        src = np.repeat(node_of_iv, lens)
        starts = np.repeat(self.iv[:, 0].astype(np.int64), lens)
        offs = np.arange(total, dtype=np.int64) - np.repeat(np.cumsum(lens) - lens, lens)
        return src, starts + offs

    @staticmethod
    def from_lists(n: int, rows: list[list[int]] | dict) -> "IntervalCSR":
        ptr = np.zeros(n + 1, dtype=np.int64)
        ivs: list[tuple[int, int]] = []
        for v in range(n):
            r = sorted(set(rows[v])) if (isinstance(rows, list) or v in rows) else []
            k0 = len(ivs)
            for x in r:
                if len(ivs) > k0 and ivs[-1][1] + 1 == x:
                    ivs[-1] = (ivs[-1][0], x)
                else:
                    ivs.append((x, x))
            ptr[v + 1] = len(ivs)
        iv = np.array(ivs, dtype=np.int32).reshape(-1, 2)
        return IntervalCSR(ptr, iv)

    @staticmethod
    def from_edges(n: int, node: np.ndarray, nbr: np.ndarray) -> "IntervalCSR":
        """Build from explicit (node, neighbour) pairs (duplicates rejected)."""
        node = np.asarray(node, dtype=np.int64)
        nbr = np.asarray(nbr, dtype=np.int64)
        if len(node) and max(int(node.max()), int(nbr.max())) < (1 << 31):
            key = np.sort((node << 31) | nbr)   # one int64 sort instead of a two-key lexsort
            node, nbr = key >> 31, key & ((1 << 31) - 1)
        else:
            order = np.lexsort((nbr, node))
            node, nbr = node[order], nbr[order]
        if len(node) > 1:
            dup = (node[1:] == node[:-1]) & (nbr[1:] == nbr[:-1])
            if dup.any():
                raise GraphError("duplicate edge")
        # a new interval starts where node changes or nbr is not previous+1
        start = np.ones(len(node), dtype=bool)
        if len(node) > 1:
            start[1:] = (node[1:] != node[:-1]) | (nbr[1:] != nbr[:-1] + 1)
        sidx = np.flatnonzero(start)
        eidx = np.append(sidx[1:], len(node)) - 1
        iv = np.stack([nbr[sidx], nbr[eidx]], axis=1).astype(np.int32) if len(sidx) else np.zeros((0, 2), np.int32)
        counts = np.bincount(node[sidx], minlength=n) if len(sidx) else np.zeros(n, np.int64)
        ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=ptr[1:])
        return IntervalCSR(ptr, iv)


def transpose(pred: IntervalCSR) -> IntervalCSR:
    """Successor intervals from predecessor intervals by explicit expansion."""
    dst, src = pred.expand()
    return IntervalCSR.from_edges(pred.n, src, dst)


@dataclass
class FlatGraph:
    n: int
    pred: IntervalCSR
    succ: IntervalCSR
    kind: np.ndarray            # uint8[N]
    arg: np.ndarray             # uint32[N]
    worker: np.ndarray          # int32[N] static owner (Alg. 1 V_w)
    n_workers: int
    col: np.ndarray | None = None   # int32[N] checksum column, -1 = none
    n_cols: int = 0
    order: np.ndarray | None = None  # int64[N] a global topological rank
    meta: dict = field(default_factory=dict)

    @property
    def indeg(self) -> np.ndarray:
        return self.pred.degrees()

    def n_edges(self) -> int:
        return self.pred.n_edges()

    def topo_rank(self) -> np.ndarray:
        if self.order is None:
            self.order = topological_rank(self.pred, self.succ)
        return self.order

    def worker_lists(self) -> tuple[np.ndarray, np.ndarray]:
        """(work_ptr int64[n_workers+1], work int32[N]): each worker's nodes in
        one global topological order — the order a worker scans its queue."""
        rank = self.topo_rank()
        order = np.lexsort((rank, self.worker))
        counts = np.bincount(self.worker, minlength=self.n_workers)
        ptr = np.zeros(self.n_workers + 1, dtype=np.int64)
        np.cumsum(counts, out=ptr[1:])
        return ptr, order.astype(np.int32)

    def cross_worker_edges(self) -> int:
        """|{(u,v) in E : owner(u) != owner(v)}| (SPEC.md:407 message minimality)."""
        v, u = self.pred.expand()
        return int((self.worker[u] != self.worker[v]).sum())


def topological_rank(pred: IntervalCSR, succ: IntervalCSR) -> np.ndarray:
    """Kahn levels (longest path from a source), tie-broken by id; raises
    GraphError on a cycle."""
    n = pred.n
    level = kahn_levels(pred, succ)
    # rank = position in (level, id) order
    order = np.lexsort((np.arange(n), level))
    rank = np.empty(n, dtype=np.int64)
    rank[order] = np.arange(n)
    return rank


def kahn_levels(pred: IntervalCSR, succ: IntervalCSR) -> np.ndarray:
    """Level of every node = length of the longest path from a source.
    Vectorised frontier sweep over explicit edges; GraphError on a cycle."""
    n = pred.n
    indeg = pred.degrees().copy()
    s_src, s_dst = succ.expand()
    order_idx = np.argsort(s_src, kind="stable")
    s_dst = s_dst[order_idx]
    s_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(s_src, minlength=n), out=s_ptr[1:])
    level = np.full(n, -1, dtype=np.int64)
    frontier = np.flatnonzero(indeg == 0)
    lv = 0
    seen = 0
    while len(frontier):
        level[frontier] = lv
        seen += len(frontier)
        lens = s_ptr[frontier + 1] - s_ptr[frontier]
        idx = np.repeat(s_ptr[frontier], lens) + (np.arange(lens.sum()) - np.repeat(np.cumsum(lens) - lens, lens))
        targets = s_dst[idx]
        np.subtract.at(indeg, targets, 1)
        cand = np.unique(targets)
        frontier = cand[indeg[cand] == 0]
        lv += 1
    if seen != n:
        raise GraphError("cycle detected")
    return level


def save_npz(g: FlatGraph, path: str) -> None:
    """Persist a flattened (recorded) graph for offline replay."""
    extra = {}
    if g.col is not None:
        extra["col"] = g.col
    if g.order is not None:
        extra["order"] = g.order
    np.savez_compressed(path, n=np.int64(g.n), pred_ptr=g.pred.ptr, pred_iv=g.pred.iv, succ_ptr=g.succ.ptr,
                        succ_iv=g.succ.iv, kind=g.kind, arg=g.arg, worker=g.worker,
                        n_workers=np.int64(g.n_workers), n_cols=np.int64(g.n_cols),
                        meta=np.frombuffer(repr({k: (v.tolist() if hasattr(v, "tolist") else v)
                                                 for k, v in g.meta.items()}).encode(), dtype=np.uint8),
                        **extra)


def load_npz(path: str) -> FlatGraph:
    import ast
    z = np.load(path, allow_pickle=False)
    meta = ast.literal_eval(bytes(z["meta"]).decode()) if "meta" in z else {}
    return FlatGraph(n=int(z["n"]), pred=IntervalCSR(z["pred_ptr"], z["pred_iv"]),
                     succ=IntervalCSR(z["succ_ptr"], z["succ_iv"]), kind=z["kind"], arg=z["arg"],
                     worker=z["worker"], n_workers=int(z["n_workers"]),
                     col=z["col"] if "col" in z else None, n_cols=int(z["n_cols"]),
                     order=z["order"] if "order" in z else None, meta=meta)

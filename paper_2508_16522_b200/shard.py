"""Sharded lowering across GPUs (SPEC.md implicit.replay 465-473, ShardingPlan
444-447; §5 825-853, Fig. 12).

The reference realises each inter-shard edge u->v as an ExtPostcond (on u's
shard) -> ExtPrecond (on v's shard) pair connected by a runtime event
(SPEC.md:468, 484).  On B200 the pair collapses into the message itself: the
worker that executes u adds ``(1<<48) + term(u)`` to v's mailbox word in v's
shard's memory over NVLink (one ``red.relaxed.sys.add.u64`` through the
cudaIpcOpenMemHandle mapping), so a cross-shard edge costs exactly one remote
atomic -- the input travels inside it -- and no host or NCCL involvement.
``ext_pairs`` still reports the reference's pair count for the SPEC.md:471
known answers.

Partition: a ShardingPlan maps each resource (worker) to a shard; the default
is contiguous blocks of workers, i.e. blocks of Task Bench points
(SURVEY.md §8(e)).  One process per GPU; the IPC handle exchange uses any
``allgather(obj) -> list`` callable (torch.distributed.all_gather_object in
practice; gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ResourceError
from .flat import FlatGraph


@dataclass(frozen=True)
class ShardingPlan:
    """mapping resource(worker) -> shard id, total and onto."""
    shard_of_worker: tuple
    n_shards: int
    devices: tuple | None = None   # in-process multi-GPU replay: device of each shard

    @staticmethod
    def blocks(n_workers: int, n_shards: int) -> "ShardingPlan":
        if n_shards < 1 or n_shards > 8:
            raise ResourceError("1..8 shards supported")
        return ShardingPlan(tuple(int(w * n_shards // n_workers) for w in range(n_workers)), n_shards)

    def validate(self, n_workers: int) -> None:
        if len(self.shard_of_worker) != n_workers:
            raise ResourceError("plan references unknown processors")
        s = set(self.shard_of_worker)
        if s != set(range(self.n_shards)):
            raise ResourceError("sharding plan must be onto 0..n_shards-1")


def node_shards(g: FlatGraph, plan: ShardingPlan) -> np.ndarray:
    plan.validate(g.n_workers)
    return np.asarray(plan.shard_of_worker, dtype=np.uint8)[g.worker]


def local_programs(g: FlatGraph, plan: ShardingPlan, rank: int):
    """(work_ptr, work, global worker ids) of shard `rank`: its workers' node
    lists in one global topological order."""
    workers = np.flatnonzero(np.asarray(plan.shard_of_worker) == rank)
    remap = np.full(g.n_workers, -1, dtype=np.int64)
    remap[workers] = np.arange(len(workers))
    mine = np.flatnonzero(remap[g.worker] >= 0)
    rank_order = g.topo_rank()
    lw = remap[g.worker[mine]]
    order = np.lexsort((rank_order[mine], lw))
    work = mine[order].astype(np.int32)
    counts = np.bincount(lw, minlength=len(workers))
    ptr = np.zeros(len(workers) + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    return ptr, work, workers


@dataclass
class HaloGraph:
    """A graph extended with halo replicas (see :func:`replicate_halo`)."""
    graph: FlatGraph          # n_real original nodes, then the replicas
    node_rank: np.ndarray     # owning shard of every node (replicas: the shard that runs them)
    ident: np.ndarray         # int32: the node each id computes (itself, or the replicated node)
    plan: ShardingPlan        # the original plan plus one worker per replica stream
    n_real: int
    k: int


def replicate_halo(g: FlatGraph, plan: ShardingPlan, k: int, max_frac: float = 0.05) -> HaloGraph | None:
    """Halo replication for sharded replay (communication-avoiding lowering).

    Without it, a stencil-like graph crosses the GPU boundary on EVERY level,
    so each level pays the NVLink mailbox hop (1.0 us vs 0.3 us on-chip).
    With period k, shard b re-computes the remote predecessors of its nodes
    whose level is not a multiple of k, transitively, from real remote
    inputs at the last multiple-of-k level: for stencil_1d a cone of k-1, k-2,
    ..., 1 columns per boundary and period.  A replica is an ordinary node
    with its own id >= n and identity u (td_csr.ident): it hashes as u, gets
    u's inputs (each predecessor copy on shard b, or the real remote one) and
    therefore computes u's token bit-exactly.  Messages that reach shard b
    come from b's copy of the producer when there is one, else from the real
    producer, so the cross-GPU hop is on the critical path once per k levels.

    Replicas of one original worker run on one extra warp of shard b, in that
    worker's order.  Needs unit-level edges (every predecessor one level
    up: all Task Bench patterns); returns None when the graph does not
    qualify or the replicas would exceed ``max_frac`` of the nodes."""
    from .flat import IntervalCSR, kahn_levels
    if k < 2 or plan.n_shards < 2:
        return None
    n = g.n
    owner = np.asarray(plan.shard_of_worker, dtype=np.int64)[g.worker]
    level = kahn_levels(g.pred, g.succ)
    dst, src = g.pred.expand()
    if len(dst) and not (level[dst] == level[src] + 1).all():
        return None
    phase = level % k
    S = plan.n_shards
    # closure: (b, u) for remote u with phase != 0 that a node on b (or a replica on b) consumes
    cross = (owner[src] != owner[dst]) & (phase[src] != 0)
    frontier = np.unique(src[cross] * S + owner[dst[cross]])
    rkeys = np.zeros(0, np.int64)
    while len(frontier):
        frontier = np.setdiff1d(frontier, rkeys, assume_unique=True)
        rkeys = np.union1d(rkeys, frontier)
        if len(rkeys) > max_frac * n:
            return None
        fu, fb = frontier // S, frontier % S
        i, p = _expand_rows(g.pred, fu)
        b = fb[i]
        keep = (owner[p] != b) & (phase[p] != 0)
        frontier = np.unique(p[keep] * S + b[keep])
    if not len(rkeys):
        return None
    r_u, r_b = rkeys // S, rkeys % S
    nr = len(rkeys)
    rid = n + np.arange(nr, dtype=np.int64)

    def copy_on(x, b):
        """id of the copy of node x that messages landing on shard b come from"""
        key = x * S + b
        i = np.searchsorted(rkeys, key)
        i = np.minimum(i, nr - 1)
        hit = rkeys[i] == key
        return np.where(hit, rid[i], x)

    # edges into real nodes: sender = the consumer's shard's copy of the producer
    e_src = [copy_on(src, owner[dst])]
    e_dst = [dst]
    # edges into replicas: every predecessor p of u, from shard b's copy of p
    j, p = _expand_rows(g.pred, r_u)
    e_src.append(copy_on(p, r_b[j]))
    e_dst.append(rid[j])
    e_src = np.concatenate(e_src)
    e_dst = np.concatenate(e_dst)
    n2 = n + nr
    pred = IntervalCSR.from_edges(n2, e_dst, e_src)
    succ = IntervalCSR.from_edges(n2, e_src, e_dst)
    # one extra worker per (shard, original worker) stream of replicas
    streams = np.unique(r_b * g.n_workers + g.worker[r_u])
    sw = np.searchsorted(streams, r_b * g.n_workers + g.worker[r_u])
    worker = np.concatenate([g.worker, g.n_workers + sw]).astype(np.int32)
    plan2 = ShardingPlan(tuple(plan.shard_of_worker) + tuple(int(x) for x in streams // g.n_workers),
                         plan.n_shards, plan.devices)
    order = g.topo_rank()
    g2 = FlatGraph(n=n2, pred=pred, succ=succ, kind=np.concatenate([g.kind, g.kind[r_u]]),
                   arg=np.concatenate([g.arg, g.arg[r_u]]), worker=worker, n_workers=g.n_workers + len(streams),
                   col=None if g.col is None else np.concatenate([g.col, np.full(nr, -1, np.int32)]),
                   n_cols=g.n_cols, order=np.concatenate([order, order[r_u]]),
                   meta={**g.meta, "halo": k, "n_real": n})
    node_rank = np.concatenate([owner, r_b]).astype(np.uint8)
    ident = np.concatenate([np.arange(n), r_u]).astype(np.int32)
    return HaloGraph(g2, node_rank, ident, plan2, n, k)


def _expand_rows(csr, rows: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(index into rows, neighbour) for every neighbour of the given rows"""
    rows = np.asarray(rows, dtype=np.int64)
    nk = csr.ptr[rows + 1] - csr.ptr[rows]
    k = np.repeat(csr.ptr[rows], nk) + (np.arange(int(nk.sum())) - np.repeat(np.cumsum(nk) - nk, nk))
    owner_row = np.repeat(np.arange(len(rows)), nk)
    lo = csr.iv[k, 0].astype(np.int64)
    ln = csr.iv[k, 1].astype(np.int64) - lo + 1
    idx = np.repeat(owner_row, ln)
    nb = np.repeat(lo, ln) + (np.arange(int(ln.sum())) - np.repeat(np.cumsum(ln) - ln, ln))
    return idx, nb


def lowering_stats(g: FlatGraph, node_rank: np.ndarray) -> dict:
    """Reference-side view of the lowering: per-shard node counts and the
    ExtPostcond->ExtPrecond pairs (one per shard-crossing edge)."""
    v, u = g.pred.expand()
    cross = node_rank[u] != node_rank[v]
    n_sh = int(node_rank.max()) + 1 if len(node_rank) else 1
    pairs = np.zeros((n_sh, n_sh), dtype=np.int64)
    np.add.at(pairs, (node_rank[u[cross]], node_rank[v[cross]]), 1)
    return dict(nodes_per_shard=np.bincount(node_rank, minlength=n_sh).tolist(),
                ext_pairs=int(cross.sum()), pairs_matrix=pairs.tolist())


class ShardedGraph:
    """This rank's shard of a graph, uploaded and wired to its peers."""

    def __init__(self, g: FlatGraph, n_ranks: int, rank: int, device: int, plan: ShardingPlan | None = None,
                 allgather=None, n_ext_pre: int = 0, n_ext_post: int = 0, stencil2d: tuple | None = None,
                 halo: int | tuple = 0, halo_max_frac: float = 0.05):
        from .executor import DeviceGraph
        self.graph = g
        self.plan = plan or ShardingPlan.blocks(g.n_workers, n_ranks)
        if self.plan.n_shards != n_ranks:
            raise ResourceError("plan shard count != number of ranks")
        self.rank = rank
        self.n_real = g.n
        self.halo = None
        gx, plan_x, ident = g, self.plan, None
        # halo: a period, or candidate periods tried in order (the first whose
        # replicas fit in halo_max_frac); every rank derives the same replicas
        periods = () if stencil2d is not None else (halo,) if isinstance(halo, int) else tuple(halo)
        for k in periods:
            if k and self.halo is None:
                self.halo = replicate_halo(g, self.plan, k, max_frac=halo_max_frac)
        if self.halo is not None:
            gx, plan_x, ident = self.halo.graph, self.halo.plan, self.halo.ident
        self.node_rank = node_shards(gx, plan_x)
        ptr, work, self.workers = local_programs(gx, plan_x, rank)
        self.dev = DeviceGraph(gx, device, n_ranks=n_ranks, my_rank=rank, node_rank=self.node_rank,
                               work_ptr=ptr, work=work, n_ext_pre=n_ext_pre, n_ext_post=n_ext_post, ident=ident)
        if stencil2d is not None:  # grid buffers must exist before their IPC handles are exported
            self.dev.attach_stencil2d(*stencil2d)
        if n_ranks > 1:
            if allgather is None:
                allgather = _torch_allgather
            handles = allgather(self.dev.ipc_export())
            for r, h in enumerate(handles):
                if r != rank:
                    self.dev.ipc_attach(r, h)

    def local_nodes(self) -> np.ndarray:
        """ids of the (original) nodes this rank owns; halo replicas excluded"""
        return np.flatnonzero(self.node_rank[:self.n_real] == self.rank)


def _torch_allgather(obj):
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


class InProcessShards:
    """All shards of a graph in ONE process, one per device:
    shard r runs on devices[r]; peers are wired with direct peer pointers.
    A device may host several shards (each then launches on its own stream,
    so their persistent kernels run concurrently)."""

    def __init__(self, g: FlatGraph, plan: ShardingPlan, devices, stencil2d: tuple | None = None, halo: int = 0):
        from .executor import DeviceGraph
        if len(devices) != plan.n_shards:
            raise ResourceError("one device per shard is required")
        self.graph = g
        self.plan = plan
        self.halo = replicate_halo(g, plan, halo) if (halo and stencil2d is None) else None
        gx, plan_x, ident = (g, plan, None) if self.halo is None else (self.halo.graph, self.halo.plan,
                                                                      self.halo.ident)
        self.node_rank = node_shards(gx, plan_x)
        self.shards = []
        for r, dev in enumerate(devices):
            ptr, work, _ = local_programs(gx, plan_x, r)
            d = DeviceGraph(gx, dev, n_ranks=plan.n_shards, my_rank=r, node_rank=self.node_rank,
                            work_ptr=ptr, work=work, ident=ident)
            if stencil2d is not None:
                d.attach_stencil2d(*stencil2d)
            self.shards.append(d)
        for r, d in enumerate(self.shards):
            for q, peer in enumerate(self.shards):
                if q != r:
                    d.attach_direct(q, peer)
        self._streams = [None] * len(devices)
        if len(set(devices)) < len(devices):
            import torch
            self._keep = [torch.cuda.Stream(device=dev) for dev in devices]
            self._streams = [st.cuda_stream for st in self._keep]

    def run(self, seed: int = 0, flags: int = 0, spin_limit: int = 0) -> None:
        for d, st in zip(self.shards, self._streams):   # every shard's persistent kernel
            d.launch(seed, flags=flags, spin_limit=spin_limit, stream=st)
        for d in self.shards:
            d.wait()

    def tokens(self) -> np.ndarray:
        n = self.graph.n
        out = np.zeros(n, dtype=np.uint64)
        for r, d in enumerate(self.shards):
            mine = self.node_rank[:n] == r
            out[mine] = d.tokens()[:n][mine]
        return out

    def close(self) -> None:
        for d in self.shards:
            d.close()

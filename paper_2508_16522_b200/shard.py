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
                 allgather=None, n_ext_pre: int = 0, n_ext_post: int = 0, stencil2d: tuple | None = None):
        from .executor import DeviceGraph
        self.graph = g
        self.plan = plan or ShardingPlan.blocks(g.n_workers, n_ranks)
        if self.plan.n_shards != n_ranks:
            raise ResourceError("plan shard count != number of ranks")
        self.rank = rank
        self.node_rank = node_shards(g, self.plan)
        ptr, work, self.workers = local_programs(g, self.plan, rank)
        self.dev = DeviceGraph(g, device, n_ranks=n_ranks, my_rank=rank, node_rank=self.node_rank,
                               work_ptr=ptr, work=work, n_ext_pre=n_ext_pre, n_ext_post=n_ext_post)
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
        return np.flatnonzero(self.node_rank == self.rank)


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

    def __init__(self, g: FlatGraph, plan: ShardingPlan, devices, stencil2d: tuple | None = None):
        from .executor import DeviceGraph
        if len(devices) != plan.n_shards:
            raise ResourceError("one device per shard is required")
        self.graph = g
        self.plan = plan
        self.node_rank = node_shards(g, plan)
        self.shards = []
        for r, dev in enumerate(devices):
            ptr, work, _ = local_programs(g, plan, r)
            d = DeviceGraph(g, dev, n_ranks=plan.n_shards, my_rank=r, node_rank=self.node_rank,
                            work_ptr=ptr, work=work)
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
        out = np.zeros(self.graph.n, dtype=np.uint64)
        for r, d in enumerate(self.shards):
            mine = self.node_rank == r
            out[mine] = d.tokens()[mine]
        return out

    def close(self) -> None:
        for d in self.shards:
            d.close()

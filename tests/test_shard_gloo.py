"""CPU: sharded-lowering host logic, including a world_size-2 gloo run of the
IPC-handle exchange and partition bookkeeping."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_16522_b200.flat import FlatGraph, IntervalCSR, transpose
from paper_2508_16522_b200.shard import ShardingPlan, _torch_allgather, local_programs, lowering_stats, node_shards
from paper_2508_16522_b200.taskbench import generate_graph


def _diamond():
    pred = IntervalCSR.from_lists(4, [[], [0], [0], [1, 2]])
    return FlatGraph(n=4, pred=pred, succ=transpose(pred), kind=np.zeros(4, np.uint8),
                     arg=np.zeros(4, np.uint32), worker=np.array([0, 1, 0, 1], np.int32), n_workers=2)


def test_diamond_two_shards_two_pairs():
    g = _diamond()
    nr = node_shards(g, ShardingPlan((0, 1), 2))
    assert lowering_stats(g, nr)["ext_pairs"] == 2


def test_one_shard_zero_pairs():
    g = _diamond()
    nr = node_shards(g, ShardingPlan((0, 0), 1))
    assert lowering_stats(g, nr)["ext_pairs"] == 0


@pytest.mark.parametrize("G,cross", [(2, 594), (4, 1782), (8, 4158)])
def test_nearest_cross_gpu_edges(G, cross):
    g = generate_graph("nearest", 8192, 100, n_workers=8192)
    nr = node_shards(g, ShardingPlan.blocks(8192, G))
    assert lowering_stats(g, nr)["ext_pairs"] == cross


def test_local_programs_partition_nodes():
    g = generate_graph("fft", 64, 9, n_workers=16)
    plan = ShardingPlan.blocks(16, 4)
    seen = []
    for r in range(4):
        ptr, work, workers = local_programs(g, plan, r)
        assert len(workers) == 4 and ptr[-1] == len(work)
        assert (node_shards(g, plan)[work] == r).all()
        for w in range(4):  # each worker's list is in topological (id) order
            lst = work[ptr[w]:ptr[w + 1]]
            assert (np.diff(lst) > 0).all()
        seen.append(work)
    allw = np.sort(np.concatenate(seen))
    assert np.array_equal(allw, np.arange(g.n))


def test_plan_validation():
    with pytest.raises(Exception):
        ShardingPlan((0, 0, 2), 3).validate(3)  # not onto
    with pytest.raises(Exception):
        ShardingPlan((0, 1), 2).validate(3)     # unknown processors


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    g = generate_graph("stencil_1d", 64, 10, n_workers=64)
    plan = ShardingPlan.blocks(64, ws)
    ptr, work, workers = local_programs(g, plan, rank)
    handle = bytes([rank]) * 192  # stand-in for 3 cudaIpcMemHandle_t
    got = _torch_allgather(handle)
    counts = _torch_allgather(int(len(work)))
    q.put((rank, [h[0] for h in got], sum(counts), g.n, int(workers.min()), int(workers.max())))
    dist.destroy_process_group()


def test_gloo_two_ranks_exchange_and_partition():
    ws = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for rank, handles, total, n, wmin, wmax in res:
        assert handles == [0, 1]
        assert total == n
        assert (wmin, wmax) == ((0, 31) if rank == 0 else (32, 63))

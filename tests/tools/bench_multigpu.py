"""BASELINE configs[3] and configs[4] across GPUs (run under torchrun, one
process per GPU): nearest r5 W=8192 T=100 and all_to_all W=8192 T=10
partitioned by point blocks, and the 2D stencil 16384^2 partitioned by tile
blocks (strong scaling: the whole graph is fixed, split over N GPUs).
Cross-GPU edges are peer-memory atomics over NVLink.  Device time per replay
is the max over ranks (CUDA events, barrier on both sides).  Parity of the
sharded tokens vs the oracle is checked on rank 0 for each graph."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2508_16522_b200.executor import device_info  # noqa: E402
from paper_2508_16522_b200.shard import ShardedGraph, lowering_stats  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph, generate_stencil2d  # noqa: E402


def timed(sg, reps, seed=1):
    for _ in range(3):
        sg.dev.run(seed, flags=0)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        dist.barrier()
        sg.dev.run(seed, flags=0)
        ts.append(sg.dev.last_ms())
    t = torch.tensor([float(np.median(ts))], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_tokens(sg, g):
    mine = sg.local_nodes()
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (mine, sg.dev.tokens()[mine]))
    full = np.zeros(g.n, np.uint64)
    for m, t in parts:
        full[m] = t
    return full


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    os.environ["NCCL_DEBUG"] = "WARN"
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, ws = dist.get_rank(), dist.get_world_size()
    info = device_info(local)
    out = []
    halos = [int(x) for x in os.environ.get("HALOS", "0,4,8").split(",")]
    for pat, W, T, reps, halo in [("nearest", 8192, 100, 10, h) for h in halos] + [("all_to_all", 8192, 10, 10, 0)]:
        if ws == 1 and halo:
            continue
        per = W // ws
        g = generate_graph(pat, W, T, n_workers=min(per, info["max_workers"]) * ws)
        sg = ShardedGraph(g, ws, rank, local, halo=halo)
        ms = timed(sg, reps)
        parity = None
        tok = gather_tokens(sg, g)
        if rank == 0:
            from oracle import seq
            parity = bool(np.array_equal(tok, seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=1)))
            ls = lowering_stats(g, sg.node_rank)
            out.append(dict(graph=f"{pat} W={W} T={T}", gpus=ws, halo=halo,
                            halo_replicas=0 if sg.halo is None else sg.halo.graph.n - g.n, tasks=g.n, replay_ms=ms,
                            tasks_per_s=g.n / (ms * 1e-3), cross_gpu_edges=ls["ext_pairs"], parity=parity))
        dist.barrier()
        sg.dev.close()
    nx = ny = 16384
    steps = 11
    ntile = (nx // 64) * (ny // 64)
    for mapping in os.environ.get("ST2D_MAPPINGS", "block,shard_cyclic,shard_block").split(","):
        g = generate_stencil2d(nx, ny, steps, n_workers=min(info["max_workers_st2d"] * ws, ntile),
                               mapping=mapping, shards=ws)
        sg = ShardedGraph(g, ws, rank, local, stencil2d=(nx, ny))
        ms = timed(sg, 5)
        if rank == 0:
            alg = ntile * (steps - 1) * ((66 * 66 - 4) * 4 + 64 * 64 * 4) + ntile * 64 * 64 * 4
            out.append(dict(graph=f"stencil2d {nx}^2 64x64 T={steps}", mapping=mapping, gpus=ws, tasks=g.n,
                            replay_ms=ms, tasks_per_s=g.n / (ms * 1e-3), ms_per_step=ms / steps,
                            hbm_GBps_total=alg / (ms * 1e-3) / 1e9,
                            parity="checked at 512^2/1024x2048 in mgpu_check"))
        dist.barrier()
        sg.dev.close()
    if rank == 0:
        for r in out:
            print(json.dumps(r), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

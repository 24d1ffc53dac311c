"""METG(50) at the paper's small widths (§6.1: stencil, width 8 and
32 on one node), on 1..N B200 (torchrun, one process per GPU; N=1 runs
without torchrun).  The stencil_1d graph is sharded by point blocks (one
column per worker); every granularity point re-parameterises the compute
body in place (set_body_arg) and times replays on the device, max over
ranks.  granularity = wall * executors / tasks with executors = the resident
worker warps of all GPUs; efficiency = rate / the sweep's best rate
(SPEC.md:536-544)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.flat import KIND_COMPUTE  # noqa: E402
from paper_2508_16522_b200.metg import Sample, compute_metg  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402


def main():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        os.environ["NCCL_DEBUG"] = "WARN"
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    iters = sorted({int(round(2 ** (k / 4))) for k in range(0, 4 * 16 + 1)})
    out = []
    for W in (8, 32):
        if W % ws:
            continue
        samples = []
        graphs = {}
        for it in iters:
            steps = 1000 if it <= 256 else (200 if it <= 8192 else 40)
            if steps not in graphs:
                g = generate_graph("stencil_1d", W, steps, n_workers=W, kind=KIND_COMPUTE, arg=1)
                if ws > 1:
                    from paper_2508_16522_b200.shard import ShardedGraph
                    halo = int(os.environ.get("METG_HALO", "0"))
                    sg = ShardedGraph(g, ws, rank, local, halo=halo, halo_max_frac=1.0)
                    graphs[steps] = (g, sg.dev, sg)
                else:
                    graphs[steps] = (g, DeviceGraph(g, local), None)
            g, dg, _ = graphs[steps]
            dg.set_body_arg(it)
            for _ in range(2):
                dg.run(1, flags=0)
            ts = []
            for _ in range(5):
                torch.cuda.synchronize()
                if dist:
                    dist.barrier()
                dg.run(1, flags=0)
                ts.append(dg.last_ms())
            t = torch.tensor([float(np.median(ts))], device="cuda")
            if dist:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall_ms = float(t.item())
            rate = g.n * it * 64 / (wall_ms * 1e-3)
            samples.append(Sample(granularity_ns=wall_ms * 1e6 * W / g.n, wall_ns=wall_ms * 1e6, rate=rate,
                                  iterations=it, tasks=g.n, executors=W))
        r = compute_metg(samples, 0.5)
        if rank == 0:
            out.append({"pattern": "stencil_1d", "width": W, "gpus": ws, "executors": W,
                        "halo": int(os.environ.get("METG_HALO", "0")) if ws > 1 else 0,
                        "metg50_us": None if r.metg_ns is None else r.metg_ns / 1e3,
                        "curve": [[round(s.granularity_ns / 1e3, 3), round(s.efficiency, 4), s.iterations]
                                  for s in r.curve]})
        for _, dg, sg in graphs.values():
            dg.close()
    if rank == 0:
        for x in out:
            print(json.dumps(x), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Cost of the sharded (MULTI) kernel itself, without NVLink: stencil_1d
1024x1000 on ONE GPU as a single graph vs as 2 shards on the same device
(two persistent kernels, peer pointers to the same memory), halo 0 and 16."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.shard import InProcessShards, ShardingPlan  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402

g = generate_graph("stencil_1d", 1024, 1000, n_workers=1024, kind=2, arg=1)
with DeviceGraph(g) as dg:
    for _ in range(3):
        dg.run(1, flags=0)
    ts = []
    for _ in range(10):
        dg.run(1, flags=0)
        ts.append(dg.last_ms())
    print("single", np.median(ts))
for halo in (0, 16):
    sh = InProcessShards(g, ShardingPlan.blocks(1024, 2), [0, 0], halo=halo)
    for _ in range(3):
        sh.run(1)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sh.run(1)
        e1.record()
        torch.cuda.synchronize()
        ts.append(max(d.last_ms() for d in sh.shards))
    print("2 shards same GPU halo", halo, np.median(ts))
    sh.close()

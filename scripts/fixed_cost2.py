"""Fixed replay cost vs CTA count: one-level no_comm graphs at several worker
counts, and the same graph on a full (placed) grid.  python scripts/fixed_cost2.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
out = {}
for place in ("0", "1"):
    os.environ["TD_PLACE"] = place
    for wk in (148, 592, 1184, 2368, 4736):
        g = generate_graph("no_comm", wk, 1, n_workers=wk)
        with DeviceGraph(g) as dg:
            for _ in range(3):
                dg.run(1, flags=0)
            ts = []
            for _ in range(11):
                flush.zero_()
                torch.cuda.synchronize()
                dg.run(1, flags=0)
                ts.append(dg.last_ms() * 1e3)
            out[f"place{place} w{wk} ctas{(wk + 3) // 4}"] = round(float(np.median(ts)), 2)
print(json.dumps(out))

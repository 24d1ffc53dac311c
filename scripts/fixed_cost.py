"""Fixed cost of one replay (launch, prologue, epilogue, copies): replay time of
tiny graphs, L2 flushed before each replay like the bench.
python scripts/fixed_cost.py"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_16522_b200 import _native as N  # noqa: E402
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
out = {}
for pat, W, T, wk in [("no_comm", 1024, 1, 1024), ("no_comm", 1024, 2, 1024), ("stencil_1d", 1024, 2, 1024),
                      ("stencil_1d", 1024, 10, 1024), ("no_comm", 8192, 2, 2048), ("nearest", 8192, 2, 2048),
                      ("nearest", 8192, 10, 2048), ("all_to_all", 8192, 2, 4096), ("no_comm", 148, 2, 148),
                      ("no_comm", 4736, 2, 4736)]:
    g = generate_graph(pat, W, T, n_workers=wk, kind=0, arg=0)
    with DeviceGraph(g) as dg:
        for _ in range(3):
            dg.run(1, flags=0)
        res = {}
        for fl_name, fl in (("noflush", False), ("flush", True)):
            ts = []
            for _ in range(11):
                if fl:
                    flush.zero_()
                torch.cuda.synchronize()
                dg.run(1, flags=0)
                ts.append(dg.last_ms() * 1e3)
            res[fl_name] = round(float(np.median(ts)), 2)
        out[f"{pat} {W}x{T} w{wk} g{dg.info()['group']}"] = res
print(json.dumps(out, indent=0))

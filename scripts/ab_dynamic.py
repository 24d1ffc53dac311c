"""Same-box A/B: static per-worker lists vs arrival-order dispatch
(TD_F_DYNAMIC, per-SM ready queues) on balanced Task Bench graphs and on
imbalanced ones (random busy_wait bodies on multi-column workers, tree with
block mapping).  Median of 9 replays each, L2 flushed; tokens checked."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_16522_b200 import _native as N  # noqa: E402
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402
from oracle import seq  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
CASES = [  # name, pattern, W, T, workers, kind, arg, busy_max_ns (random per node if > 0)
    ("stencil_busy_rand2us_w128", "stencil_1d", 1024, 1000, 128, 1, 0, 2000),
    ("stencil_busy_rand2us_w256", "stencil_1d", 1024, 1000, 256, 1, 0, 2000),
    ("stencil_busy_rand2us_w1024", "stencil_1d", 1024, 1000, 1024, 1, 0, 2000),
    ("nearest_busy_rand4us_w512", "nearest", 2048, 200, 512, 1, 0, 4000),
    ("tree_empty_w256", "tree", 4096, 1000, 256, 0, 0, 0),
    ("stencil_compute1_w1024", "stencil_1d", 1024, 1000, 1024, 2, 1, 0),
    ("fft_empty_w4096", "fft", 4096, 1000, 4096, 0, 0, 0),
]
out = {}
for name, pat, W, T, wk, kind, arg, busy in CASES:
    g = generate_graph(pat, W, T, n_workers=wk, mapping="block", kind=kind, arg=arg)
    if busy:
        g.arg[:] = np.random.default_rng(1).integers(0, busy, size=g.n).astype(np.uint32)
    want = seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=1)
    res = {}
    with DeviceGraph(g, dynamic=True) as dg:
        for mode, fl in (("static", 0), ("dynamic", N.TD_F_DYNAMIC)):
            for _ in range(2):
                dg.run(1, flags=fl, spin_limit=1 << 26)
            ts = []
            for _ in range(9):
                flush.zero_()
                torch.cuda.synchronize()
                dg.run(1, flags=fl, spin_limit=1 << 26)
                ts.append(dg.last_ms())
            res[mode] = round(float(np.median(ts)), 4)
            res[mode + "_ok"] = bool(np.array_equal(dg.tokens(), want))
    res["dynamic_over_static"] = round(res["dynamic"] / res["static"], 3)
    out[name] = res
    print(name, json.dumps(res), flush=True)
print(json.dumps(out))

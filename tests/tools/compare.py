"""Claim direction of the paper on B200: per-task
overhead of the compiled persistent executor vs a CUDA Graph of the same DAG
vs a generic event-driven per-task runtime, all parity-checked."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_16522_b200.comparators import CudaGraphReplay, event_runtime  # noqa: E402
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402
from oracle import seq  # noqa: E402

rows = []
for pat, W, T in [("stencil_1d", 8, 100), ("stencil_1d", 32, 100), ("stencil_1d", 128, 100), ("fft", 64, 100),
                  ("stencil_1d", 1024, 10)]:
    g = generate_graph(pat, W, T, n_workers=W, kind=2, arg=1)
    want = seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=4)
    with DeviceGraph(g) as dg:
        for _ in range(3):
            dg.run(4, flags=0)
        ts = []
        for _ in range(20):
            dg.run(4, flags=0)
            ts.append(dg.last_ms())
        ours = float(np.median(ts))
        ok_ours = np.array_equal(dg.tokens(), want)
    cg = CudaGraphReplay(g, seed=4)
    for _ in range(3):
        cg.run()
    cg_ms = float(np.median([cg.run() for _ in range(10)]))
    ok_cg = np.array_equal(cg.tokens(), want)
    cg.close()
    evs = []
    for _ in range(3):
        ms, tok = event_runtime(g, min(W, 32), seed=4)
        evs.append(ms)
    ev_ms = float(np.median(evs))
    ok_ev = np.array_equal(tok, want)
    r = dict(graph=f"{pat} {W}x{T}", tasks=g.n, ours_ms=ours, cuda_graph_ms=cg_ms, event_runtime_ms=ev_ms,
             ours_us_per_step=1e3 * ours / T, cuda_graph_us_per_step=1e3 * cg_ms / T,
             event_us_per_step=1e3 * ev_ms / T, speedup_vs_cuda_graph=cg_ms / ours,
             speedup_vs_event_runtime=ev_ms / ours, parity=[bool(ok_ours), bool(ok_cg), bool(ok_ev)])
    rows.append(r)
    print(json.dumps(r), flush=True)

"""Quick GPU probe: roofline microbenchmarks + replay timings of the configs."""
import json, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2508_16522_b200.executor import DeviceGraph, device_info
from paper_2508_16522_b200.taskbench import generate_graph
from paper_2508_16522_b200 import roofline

info = device_info(0)
print(json.dumps(info))
rf = roofline.measure(0, info["sm_count"])
print(json.dumps(rf))
res = {}
for pat, W, T, kind, arg, workers in [("stencil_1d", 8, 100, 0, 0, 8), ("stencil_1d", 1024, 1000, 0, 0, 1024),
                                      ("no_comm", 1024, 1000, 0, 0, 1024), ("fft", 4096, 1000, 0, 0, 4096),
                                      ("tree", 4096, 1000, 0, 0, 4096), ("nearest", 8192, 100, 0, 0, None), ("all_to_all", 8192, 10, 0, 0, None),
                                      ("stencil_1d", 1024, 1000, 2, 64, 1024), ("stencil_1d", 1024, 1000, 2, 1024, 1024)]:
    mw = info["max_workers"]
    wk = min(workers or mw, mw, W)
    g = generate_graph(pat, W, T, n_workers=wk, kind=kind, arg=arg)
    with DeviceGraph(g) as dg:
        for _ in range(3):
            dg.run(seed=1)
        ts = []
        for _ in range(5):
            dg.run(seed=1)
            ts.append(dg.last_ms())
        ms = float(np.median(ts))
        print(f"{pat} W={W} T={T} kind={kind} arg={arg} workers={wk}: {ms:.3f} ms, {g.n/ms*1e3:.3e} tasks/s, per-step {ms*1e3/T:.2f} us", flush=True)

"""Is the METG plateau clock-limited?  Burst vs sustained LCG peak, and the
SM clock while a long compute_bound replay (1024 executors) runs."""
import json
import sys
import threading
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2508_16522_b200 import roofline as RF  # noqa: E402
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402

out = {"compute_peak": RF.compute_peak(0, 148, sustained_s=4.0)}
g = generate_graph("stencil_1d", 1024, 1000, n_workers=1024, kind=2, arg=1)
with DeviceGraph(g) as dg:
    for it in (1, 256, 2048, 8192):
        dg.set_body_arg(it)
        dg.run(1, flags=0)
        with bench.Clocks(0) as clk:
            t0 = time.time()
            ts = []
            while time.time() - t0 < 3.0:
                dg.run(1, flags=0)
                ts.append(dg.last_ms())
        c = clk.summary()
        rate = g.n * it * 64 / (sorted(ts)[len(ts) // 2] * 1e-3)
        out[f"iters_{it}"] = {"replay_ms_median": sorted(ts)[len(ts) // 2], "rate": rate,
                              "eff_vs_burst": rate / out["compute_peak"]["lane_updates_per_s"],
                              "eff_vs_sustained": rate / out["compute_peak"]["sustained_lane_updates_per_s"],
                              "clocks": c}
        print(it, json.dumps(out[f"iters_{it}"]), flush=True)
print(json.dumps(out))

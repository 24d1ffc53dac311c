"""Per-level timeline of a replay from TD_F_TRACE (%globaltimer per node:
entry, inputs observed, before sends, after bookkeeping): when each level's
nodes start, see their inputs and finish, and how long the last producer's
send takes to be observed by the next level.  Diagnostic:
python scripts/trace_levels.py all_to_all 8192 20 4736 [kind arg]"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_16522_b200 import _native as N  # noqa: E402
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402

pat, W, T, wk = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
kind, arg = (int(sys.argv[5]), int(sys.argv[6])) if len(sys.argv) > 6 else (0, 0)
g = generate_graph(pat, W, T, n_workers=wk, kind=kind, arg=arg)
with DeviceGraph(g) as dg:
    for _ in range(3):
        dg.run(1, flags=0)
    plain_ms = dg.last_ms()
    dg.run(1, flags=N.TD_F_TRACE)
    tr = dg.trace().reshape(-1, 4)[: g.n].astype(np.int64)
    info = dg.info()
lv = np.arange(g.n) // W  # Task Bench ids: level-major
t0 = tr[:, 0].min()
rows = []
for t in range(T):
    m = lv == t
    e, i, s, b = (tr[m, k] - t0 for k in range(4))
    rows.append({"t": t, "entry_min": int(e.min()), "in_min": int(i.min()), "in_med": int(np.median(i)),
                 "in_max": int(i.max()), "send_max": int(s.max()), "done_max": int(b.max()),
                 "wait_med": int(np.median(i - e)), "body_med": int(np.median(s - i)), "send_book_med": int(np.median(b - s))})
for r in rows:
    print(json.dumps(r))
d = [rows[t + 1]["in_min"] - rows[t]["send_max"] for t in range(T - 1)]
per = [rows[t + 1]["in_max"] - rows[t]["in_max"] for t in range(T - 1)]
print(json.dumps({"graph": f"{pat} {W}x{T} workers {wk}", "info": info, "replay_ms_untraced": plain_ms,
                  "ns_per_level_median": float(np.median(per)),
                  "last_send_to_first_observe_ns_median": float(np.median(d)),
                  "spread_in_observed_ns_median": float(np.median([r["in_max"] - r["in_min"] for r in rows]))}))

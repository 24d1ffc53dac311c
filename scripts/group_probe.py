"""Per-pass cycle breakdown of GROUP mode (diagnostic; -DTD_CYCLE_PROBE build
via TD_LIB): entry -> inputs ready (wait) -> term (proc) -> sends issued ->
end (tail), the gap to the warp's next pass, and the number of poll rounds.
python scripts/group_probe.py nearest 8192 100 2048 [kind arg]"""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
PROBE = os.path.join(HERE, "paper_2508_16522_b200", "libtdexec_probe.so")
os.environ["TD_LIB"] = os.environ.get("TD_PROBE_LIB", PROBE)
from paper_2508_16522_b200 import _native as N  # noqa: E402
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402

pat, W, T, wk = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
kind, arg = (int(sys.argv[5]), int(sys.argv[6])) if len(sys.argv) > 6 else (0, 0)
mapping = sys.argv[7] if len(sys.argv) > 7 else "block"
g = generate_graph(pat, W, T, n_workers=wk, kind=kind, arg=arg, mapping=mapping)
with DeviceGraph(g) as dg:
    for _ in range(3):
        dg.run(1, flags=0)
    plain_ms = dg.last_ms()
    dg.run(1, flags=N.TD_F_TRACE)
    traced_ms = dg.last_ms()
    import ctypes as C
    raw = np.zeros(8 * g.n + 8, dtype=np.uint64)
    N.check(N.lib().td_graph_trace(dg._h, raw.ctypes.data_as(C.c_void_p), raw.size))
    tr = raw[: 8 * g.n].reshape(g.n, 8).astype(np.int64)
    k_entry = int(~raw[8 * g.n + 5] & np.uint64(0xFFFFFFFFFFFFFFFF))
    k_exit = int(raw[8 * g.n + 6])
    info = dg.info()
rows = np.nonzero(tr[:, 0])[0]
t = tr[rows]
wait, proc, send, tail = t[:, 1] - t[:, 0], t[:, 2] - t[:, 1], t[:, 3] - t[:, 2], t[:, 4] - t[:, 3]
polls = t[:, 5] & 0xFFFFFFFF
smid = t[:, 5] >> 32
# gap: same worker, next pass by start time
wkr = np.asarray(g.worker)[rows]
order = np.lexsort((t[:, 0], wkr))
ws, t0, t4 = wkr[order], t[order, 0], t[order, 4]
same = ws[1:] == ws[:-1]
gap = (t0[1:] - t4[:-1])[same]
st = lambda a: {"p50": float(np.median(a)), "mean": float(np.mean(a))}  # noqa: E731
# per warp: cycles from its first pass's entry to its last pass's end; globally
# (%globaltimer) the first entry to the last end, against the kernel time
first = np.r_[True, ~same]
last = np.r_[~same, True]
span_cycles = t4[last] - t0[first]
g_span_us = (t[:, 7].max() - t[:, 6].min()) / 1e3
g_first_entry_us = np.sort(t[:, 6] - t[:, 6].min())
# the workers that end last: their SM, how many workers share that SM, their mean pass cycles
wl = ws[last]
end_us = (t[order][last][:, 7] - t[:, 6].min()) / 1e3
sm_of_w = smid[order][last]
wpsm = np.bincount(sm_of_w.astype(np.int64), minlength=200)
pass_mean = {}
dur = (t4 - t0)
for w_, d_ in zip(ws, dur):
    pass_mean.setdefault(int(w_), []).append(d_)
idx = np.argsort(-end_us)[:12]
straggle = [{"worker": int(wl[i]), "end_us": round(float(end_us[i]), 1), "sm": int(sm_of_w[i]),
             "workers_on_sm": int(wpsm[sm_of_w[i]]), "mean_pass_cycles": round(float(np.mean(pass_mean[int(wl[i])])), 0)}
            for i in idx]
load_of_pass = wpsm[smid.astype(np.int64)]
by_load = {}
for L in np.unique(load_of_pass):
    m = load_of_pass == L
    by_load[int(L)] = {"passes": int(m.sum()), "wait": round(float(wait[m].mean())), "proc": round(float(proc[m].mean())),
                       "send": round(float(send[m].mean())), "tail": round(float(tail[m].mean())),
                       "poll_rounds": round(float(polls[m].mean()), 3)}
straggle.append({"phases_by_workers_on_sm": by_load})
wids = np.array(sorted(pass_mean))
pm = np.array([np.mean(pass_mean[w_]) for w_ in wids])
wait_by_w = {}
for w_, a_ in zip(wkr, wait):
    wait_by_w.setdefault(int(w_), []).append(a_)
wm = np.array([np.mean(wait_by_w[w_]) for w_ in wids])
straggle.append({"mean_pass_cycles_by_worker_32tiles": [round(float(x)) for x in [pm[i::1][:0].sum() or np.mean(c) for i, c in enumerate(np.array_split(pm, 32))]],
                 "mean_wait_cycles_by_worker_32tiles": [round(float(np.mean(c))) for c in np.array_split(wm, 32)],
                 "last_16_workers_pass": [round(float(x)) for x in pm[-16:]],
                 "first_16_workers_pass": [round(float(x)) for x in pm[:16]]})
straggle.append({"median_workers_on_sm": float(np.median(wpsm[wpsm > 0])),
                 "median_mean_pass_cycles": float(np.median([np.mean(v) for v in pass_mean.values()]))})
print(json.dumps({"graph": f"{pat} {W}x{T} workers {wk} kind {kind} arg {arg} {mapping}", "group": info["group"],
                  "passes": int(len(rows)), "plain_ms": plain_ms, "traced_ms": traced_ms,
                  "wait": st(wait), "proc": st(proc), "send": st(send), "tail": st(tail), "gap": st(gap),
                  "poll_rounds": st(polls), "frac_one_round": float(np.mean(polls == 0)),
                  "warp_span_us_at_1965MHz": st(span_cycles / 1965.0),
                  "global_first_entry_to_last_end_us": float(g_span_us),
                  "kernel_minus_span_us": float(traced_ms * 1e3 - g_span_us),
                  "event_ms_minus_kernel_entry_to_exit_us": float(traced_ms * 1e3 - (k_exit - k_entry) / 1e3),
                  "kernel_entry_to_first_pass_us": float((t[:, 6].min() - k_entry) / 1e3),
                  "last_pass_to_kernel_exit_us": float((k_exit - t[:, 7].max()) / 1e3),
                  "warp_first_entry_us_pct": [round(float(x), 2) for x in np.percentile(
                      (t[order][first][:, 6] - t[:, 6].min()) / 1e3, [0, 10, 50, 90, 99, 100])],
                  "warp_last_end_us_pct": [round(float(x), 2) for x in np.percentile(
                      (t[order][last][:, 7] - t[:, 6].min()) / 1e3, [0, 10, 50, 90, 99, 100])],
                  "stragglers": straggle,
                  "first_entry_by_worker_decile_us": [round(float(np.mean(x)), 2) for x in np.array_split(
                      (t[order][first][:, 6] - t[:, 6].min()) / 1e3, 10)]}))

"""Per-task cycle breakdown of the executor's critical path (diagnostic).

Needs the -DTD_CYCLE_PROBE build (libtdexec_probe.so, built here) loaded via
TD_LIB.  With TD_F_TRACE every task's lane 0 records %clock64 at:
  p0 entry  p1 inputs observed  p2 h  p3 body  p4 term  p5 sends issued
  p6 stores done  p7 = number of mailbox polls
All deltas are within one warp (one SM clock).  `gap` is p0 of a worker's
next task minus p6 of its previous one (descriptor fetch + identity hashes)."""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
PROBE = os.path.join(HERE, "paper_2508_16522_b200", "libtdexec_probe.so")


def build():
    from paper_2508_16522_b200 import _native as N
    if not os.path.exists(PROBE) or os.path.getmtime(PROBE) < os.path.getmtime(N.SRC_PATH):
        subprocess.run(["nvcc", *N.NVCC_FLAGS, "-DTD_CYCLE_PROBE", "-o", PROBE, N.SRC_PATH], check=True)


def main():
    build()
    os.environ["TD_LIB"] = PROBE
    from paper_2508_16522_b200 import _native as N
    from paper_2508_16522_b200.executor import DeviceGraph
    from paper_2508_16522_b200.taskbench import generate_graph
    out = {}
    if "--multi" in sys.argv:  # the sharded kernel: 2 shards of stencil_1d on the same GPU
        from paper_2508_16522_b200.shard import InProcessShards, ShardingPlan
        g = generate_graph("stencil_1d", 1024, 1000, n_workers=1024, kind=2, arg=1)
        sh = InProcessShards(g, ShardingPlan.blocks(1024, 2), [0, 0], halo=16)
        for _ in range(3):
            sh.run(1)
        sh.run(1, flags=N.TD_F_TRACE)
        gx = sh.halo.graph
        tr = np.zeros((gx.n, 8), np.int64)
        for r, d in enumerate(sh.shards):
            mine = sh.node_rank == r
            tr[mine] = d.trace(8).astype(np.int64)[mine]
        has = gx.pred.degrees() > 0
        keys = ["wait", "h", "body", "term", "send", "tail"]
        r = {k: float(np.mean((tr[:, i + 1] - tr[:, i])[has])) for i, k in enumerate(keys)}
        r["polls"] = float(tr[has, 7].mean())
        print("multi 2 shards same GPU", json.dumps(r), flush=True)
        sh.close()
        return out
    cases = [("stencil_1d", 1024, 1000, 2, 1), ("no_comm", 1024, 1000, 2, 1), ("stencil_1d", 1024, 1000, 0, 0),
             ("fft", 4096, 300, 2, 1)]
    for pat, W, T, kind, arg in cases:
        g = generate_graph(pat, W, T, n_workers=min(W, 4736), kind=kind, arg=arg)
        with DeviceGraph(g) as dg:
            for _ in range(3):
                dg.run(1, flags=0)
            dg.run(1, flags=0)
            plain = dg.last_ms()
            dg.run(1, flags=N.TD_F_TRACE)
            traced = dg.last_ms()
            tr = dg.trace(8).astype(np.int64)
        has = g.pred.degrees() > 0
        d = {
            "wait": tr[:, 1] - tr[:, 0], "h": tr[:, 2] - tr[:, 1], "body": tr[:, 3] - tr[:, 2],
            "term": tr[:, 4] - tr[:, 3], "send": tr[:, 5] - tr[:, 4], "tail": tr[:, 6] - tr[:, 5],
        }
        # next task of the same worker: the worker lists are in g.order per worker
        order = np.argsort(g.worker, kind="stable")
        wk = g.worker[order]
        same = wk[1:] == wk[:-1]
        gap = tr[order[1:], 0] - tr[order[:-1], 6]
        r = {k: {"p50": float(np.median(a[has])), "mean": float(a[has].mean())} for k, a in d.items()}
        r["gap"] = {"p50": float(np.median(gap[same])), "mean": float(gap[same].mean())}
        polls = tr[has, 7]
        r["polls"] = {"p50": float(np.median(polls)), "mean": float(polls.mean()),
                      "frac_first_poll": float((polls == 1).mean())}
        per_task = sum(r[k]["mean"] for k in ("wait", "h", "body", "term", "send", "tail", "gap"))
        r["sum_mean_cycles"] = per_task
        r["plain_ms"], r["traced_ms"] = plain, traced
        r["cycles_per_step_at_1965MHz"] = plain * 1e-3 * 1.965e9 / (g.n / W) if pat != "fft" else None
        out[f"{pat}_{W}x{T}_kind{kind}"] = r
        print(f"{pat} {W}x{T} kind={kind}", json.dumps(r), flush=True)
    return out


if __name__ == "__main__":
    main()

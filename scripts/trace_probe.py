"""Per-task latency breakdown of a replay from the TD_F_TRACE timestamps.

For every node v with predecessors:
  detect  = ts1(v) - max_u ts3(u)   last predecessor signalled -> v observed ready
  gather  = ts2(v) - ts1(v)         input token loads
  publish = ts3(v) - ts2(v)         body + token store + release fence + RED issue
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_16522_b200 import _native as N  # noqa: E402
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402


def analyze(g, tr):
    v, u = g.pred.expand()
    last = np.zeros(g.n, dtype=np.int64)
    np.maximum.at(last, v, tr[u, 3].astype(np.int64))
    has = g.pred.degrees() > 0
    det = (tr[:, 1].astype(np.int64) - last)[has]
    gat = (tr[:, 2].astype(np.int64) - tr[:, 1].astype(np.int64))[has]
    pub = (tr[:, 3].astype(np.int64) - tr[:, 2].astype(np.int64))[has]
    q = lambda a: {p: float(np.percentile(a, p)) for p in (10, 50, 90, 99)}  # noqa: E731
    span = (tr[:, 3].max() - tr[:, 0].min()) / 1e3
    lsb = int(np.gcd.reduce(np.diff(np.unique(tr[:, 1]))[:10000].astype(np.int64)))
    return dict(detect_ns=q(det), gather_ns=q(gat), publish_ns=q(pub), span_us=float(span), timer_gcd_ns=lsb)


def main():
    out = {}
    for pat, W, T, kind, arg in [("stencil_1d", 1024, 1000, 2, 1), ("fft", 4096, 300, 2, 1),
                                 ("no_comm", 1024, 1000, 2, 1)]:
        g = generate_graph(pat, W, T, n_workers=min(W, 4736), kind=kind, arg=arg)
        with DeviceGraph(g) as dg:
            for _ in range(3):
                dg.run(1, flags=0)
            dg.run(1, flags=0)
            plain = dg.last_ms()
            dg.run(1, flags=N.TD_F_TRACE)
            traced = dg.last_ms()
            r = analyze(g, dg.trace())
        r.update(plain_ms=plain, traced_ms=traced)
        out[f"{pat}_{W}x{T}"] = r
        print(pat, json.dumps(r), flush=True)
    return out


if __name__ == "__main__":
    main()

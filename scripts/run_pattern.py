"""Replay one Task Bench graph a few times on cuda:0 (for ncu captures of
patterns other than the bench headline): python scripts/run_pattern.py fft 4096 1000
[kind arg [workers]] -- workers < W puts several columns on each worker (PAIR mode)"""
import sys

sys.path.insert(0, ".")
from paper_2508_16522_b200.executor import DeviceGraph, device_info  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402

pat, W, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
kind, arg = (2, 1) if len(sys.argv) < 5 else (int(sys.argv[4]), int(sys.argv[5]))
nw = int(sys.argv[6]) if len(sys.argv) > 6 else min(W, device_info(0)["max_workers"])
g = generate_graph(pat, W, T, n_workers=nw, kind=kind, arg=arg)
with DeviceGraph(g) as dg:
    for _ in range(4):
        dg.run(1, flags=0)
    print(pat, W, T, "replay ms", dg.last_ms())

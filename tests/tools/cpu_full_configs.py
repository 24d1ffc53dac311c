"""CPU reference (PAPER Alg. 1 restated on the reference's own
taskdual.machine) at FULL size on BASELINE configs[0]-[2], median of 5
executions after 2 warm-ups (SURVEY 8(d) CPU timing plan),
tokens checked against the C oracle.  Too slow for bench.py's default run
(configs[2] is 4M tasks per execution); run once on the GPU box's host:
python tests/tools/cpu_full_configs.py > profiles/r02_cpu_full_configs.jsonl"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402

for pattern, W, T, iters in (("stencil_1d", 8, 100, 0), ("stencil_1d", 1024, 1000, 1), ("no_comm", 1024, 1000, 1),
                             ("fft", 4096, 1000, 0), ("tree", 4096, 1000, 0)):
    r = bench.cpu_reference(W, T, iters, reps=5, warmups=2, pattern=pattern)
    print(json.dumps({"config": f"{pattern} W={W} T={T} {'compute_bound(%d)' % iters if iters else 'empty'}",
                      "tasks": r["tasks"], "tasks_per_s": r["value"], "median_s": r["seconds"], "times_s": r["times"],
                      "cores": r["cores"], "sample": r["sample"]}), flush=True)

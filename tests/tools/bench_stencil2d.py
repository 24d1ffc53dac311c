"""BASELINE configs[4] mini-app on one GPU (or one shard per rank under
torchrun): 2D 5-point stencil, 64x64-cell tasks, one persistent-kernel
launch per replay.  Reports tasks/s and the HBM roofline of the tile bodies
(33,808 algorithmic bytes per interior tile: read 66x66x4 - corners, write
64x64x4).  Parity vs the C oracle at a reduced size."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2508_16522_b200 import _native as N  # noqa: E402
from paper_2508_16522_b200.executor import DeviceGraph, device_info  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_stencil2d  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=11)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--workers", type=int, default=0)
    a = ap.parse_args()
    info = device_info(0)
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "MEASURED_PEAKS.json")))
    # parity at a reduced size first
    from oracle import seq
    gs = generate_stencil2d(1024, 1024, 4)
    want, _ = seq.stencil2d_tokens(gs, seed=3)
    with DeviceGraph(gs) as dg:
        dg.attach_stencil2d(1024, 1024)
        dg.run(seed=3)
        parity = bool(np.array_equal(dg.tokens(), want))
    st2_workers = a.workers or None
    g = generate_stencil2d(a.n, a.n, a.steps, n_workers=st2_workers or min(info["max_workers_st2d"], (a.n // 64) ** 2))
    nt = (a.n // 64) ** 2
    with DeviceGraph(g) as dg:
        dg.attach_stencil2d(a.n, a.n)
        for _ in range(2):
            dg.run(seed=1, flags=0)
        ts = []
        for _ in range(a.reps):
            dg.run(seed=1, flags=0)
            ts.append(dg.last_ms())
    ms = float(np.median(ts))
    upd_steps = a.steps - 1  # step 0 initialises
    tile_bytes = (66 * 66 - 4) * 4 + 64 * 64 * 4
    alg = nt * upd_steps * tile_bytes + nt * 64 * 64 * 4  # + init writes
    out = dict(workload=f"stencil2d {a.n}^2, 64x64 tiles ({nt} tasks/step), {a.steps} steps (1 init + {upd_steps} updates)",
               tasks=g.n, replay_ms=ms, tasks_per_s=g.n / (ms * 1e-3), ms_per_update_step=ms / a.steps,
               workers=g.n_workers, achieved_GBps=alg / (ms * 1e-3) / 1e9, hbm_peak_GBps=peaks["hbm_gbs"],
               frac=alg / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], parity_1024=parity)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

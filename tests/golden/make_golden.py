"""Generate the golden token fixtures (tests/golden/golden.npz).

Run in the BUILD container (where the reference is importable):
    python tests/golden/make_golden.py
Each case is executed by the CPU reference executor — PAPER Alg. 1 restated
on the reference's own taskdual.machine substrate (oracle/alg1_cpu.py) — and
cross-checked against both sequential oracles (numpy per-timestep and plain
C) before being written.  The fixtures then pin the oracle in tests that run
anywhere (including the GPU box, where /root/reference does not exist).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import alg1_cpu, seq, taskbench_np as tnp  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402

CASES = [
    # name, pattern, width, steps, kind, arg, seed, processors
    ("stencil_8x100_s0", "stencil_1d", 8, 100, 0, 0, 0, 8),
    ("stencil_8x100_s1", "stencil_1d", 8, 100, 0, 0, 1, 4),
    ("stencil_8x100_s2", "stencil_1d", 8, 100, 0, 0, 2, 2),
    ("stencil_8x100_s3", "stencil_1d", 8, 100, 0, 0, 3, 1),
    ("no_comm_16x20_c5", "no_comm", 16, 20, 2, 5, 4, 4),
    ("fft_32x24", "fft", 32, 24, 0, 0, 5, 4),
    ("tree_32x10_c3", "tree", 32, 10, 2, 3, 6, 4),
    ("nearest5_40x12", "nearest", 40, 12, 0, 0, 7, 4),
    ("all_to_all_24x5", "all_to_all", 24, 5, 0, 0, 8, 4),
    ("spread5_20x8", "spread", 20, 8, 0, 0, 9, 4),
    ("stencil_1024x4_c1", "stencil_1d", 1024, 4, 2, 1, 1, 8),
]


def main():
    out = {}
    for name, pat, W, T, kind, arg, seed, P in CASES:
        g = generate_graph(pat, W, T, n_workers=P, mapping="round_robin", kind=kind, arg=arg)
        rows = [g.pred.row(v) for v in range(g.n)]
        tok, stats, _ = alg1_cpu.run_flat(g.n, rows, g.worker, kind=g.kind, arg=g.arg, seed=seed, processors=P)
        c = seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=seed)
        n = tnp.run(pat, W, T, seed=seed, kind=kind, arg=arg)
        assert np.array_equal(tok, c) and np.array_equal(c, n), name
        assert stats["cross_worker_messages"] == g.cross_worker_edges(), name
        out[name] = tok
        out[name + "__stats"] = np.array([stats["cross_worker_messages"], stats["local_decrements"],
                                          stats["init_messages"]], dtype=np.int64)
        print(name, g.n, hex(int(np.bitwise_xor.reduce(tok))), stats)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz"), **out)


if __name__ == "__main__":
    main()

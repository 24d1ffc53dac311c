"""Small cases of every kernel path (DIAG, plain, PLAIN, sharded, tile body,
comparators, implicit runtime), each checked against the oracle."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import seq  # noqa: E402
from paper_2508_16522_b200 import _native as N  # noqa: E402
from paper_2508_16522_b200.comparators import CudaGraphReplay, event_runtime  # noqa: E402
from paper_2508_16522_b200.executor import DeviceGraph  # noqa: E402
from paper_2508_16522_b200.implicit import ImplicitRuntime  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph, generate_stencil2d  # noqa: E402
from paper_2508_16522_b200.tasks import DeviceBody, TaskRegistry  # noqa: E402

ok = True
for pat, W, T, k in [("stencil_1d", 32, 8, 2), ("all_to_all", 96, 3, 0), ("fft", 16, 6, 0), ("no_comm", 8, 70, 2)]:
    g = generate_graph(pat, W, T, n_workers=min(W, 8), kind=k, arg=3)
    with DeviceGraph(g) as dg:
        # the DIAG kernel, then the plain one (PLAIN where the graph qualifies)
        for s, fl in ((1, N.TD_F_CHECKSUM | N.TD_F_STATS | N.TD_F_TALLY | N.TD_F_TRACE), (2, 0), (3, N.TD_F_CHECKSUM)):
            dg.run(s, flags=fl)
            ok &= np.array_equal(dg.tokens(), seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=s))
# the sharded kernels (plain + PLAIN + halo replicas) with two shards on this GPU
from paper_2508_16522_b200.shard import InProcessShards, ShardingPlan  # noqa: E402
for pat, W, T, halo in [("stencil_1d", 64, 12, 3), ("all_to_all", 128, 3, 0)]:
    g = generate_graph(pat, W, T, n_workers=W, kind=2, arg=2)
    sh = InProcessShards(g, ShardingPlan.blocks(W, 2), [0, 0], halo=halo)
    try:
        for s, fl in ((1, N.TD_F_TALLY), (2, 0)):
            sh.run(s, flags=fl, spin_limit=1 << 30)
            ok &= np.array_equal(sh.tokens(), seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=s))
    finally:
        sh.close()
# GROUP passes (2 and 4 nodes), a padded GROUP layout, the arrival-order
# kernel, memory_bound bodies, and the sharded GROUP kernel
for pat, W, T, wk, k in [("stencil_1d", 64, 6, 16, 2), ("nearest", 64, 6, 32, 0), ("tree", 64, 8, 16, 2)]:
    g = generate_graph(pat, W, T, n_workers=wk, mapping="block", kind=k, arg=2)
    with DeviceGraph(g, dynamic=True) as dg:
        for s, fl in ((1, 0), (2, N.TD_F_DYNAMIC | N.TD_F_TALLY), (3, N.TD_F_CHECKSUM | N.TD_F_STATS)):
            dg.run(s, flags=fl, spin_limit=1 << 28)
            ok &= np.array_equal(dg.tokens(), seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=s))
g = generate_graph("no_comm", 16, 4, n_workers=4, mapping="block", kind=6, arg=128)
with DeviceGraph(g) as dg:
    dg.attach_scratch(128)
    dg.run(5)
    ok &= np.array_equal(dg.tokens(), seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=5))
g = generate_graph("nearest", 128, 8, n_workers=32, kind=2, arg=2)
sh = InProcessShards(g, ShardingPlan.blocks(32, 2), [0, 0])
try:
    sh.run(6, flags=0, spin_limit=1 << 30)
    ok &= np.array_equal(sh.tokens(), seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=6))
finally:
    sh.close()
g = generate_stencil2d(256, 128, 3, n_workers=5)
with DeviceGraph(g) as dg:
    dg.attach_stencil2d(256, 128)
    dg.run(4)
    ok &= np.array_equal(dg.tokens(), seq.stencil2d_tokens(g, 4)[0])
reg = TaskRegistry()
reg.register_task(1, DeviceBody.compute_bound(2))
rt = ImplicitRuntime(reg, capacity=1024)
r = [rt.region() for _ in range(3)]
rt.begin_trace(1)
for i in range(12):
    rt.issue(1, i % 2, accesses=[(r[i % 3], "write"), (r[(i + 1) % 3], "read")])
rt.end_trace(1)
rt.replay(1, "memoized")
rt.replay(1, "compiled").wait()
img = rt.memory_image()
rt.close()
g = generate_graph("stencil_1d", 8, 10, kind=2, arg=1)
cg = CudaGraphReplay(g, seed=2)
cg.run()
ok &= np.array_equal(cg.tokens(), seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=2))
cg.close()
ms, tok = event_runtime(g, 4, seed=2)
ok &= np.array_equal(tok, seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=2))
print("sanitize cases parity:", ok)
sys.exit(0 if ok else 1)

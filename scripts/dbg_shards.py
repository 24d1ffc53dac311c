import sys, numpy as np
sys.path.insert(0, ".")
from paper_2508_16522_b200 import _native as N
from paper_2508_16522_b200.shard import InProcessShards, ShardingPlan
from paper_2508_16522_b200.taskbench import generate_graph
W, T, S = 256, 20, 8
g = generate_graph("stencil_1d", W, T, n_workers=W)
sh = InProcessShards(g, ShardingPlan.blocks(W, S), [0] * S)
seq = __import__("oracle.seq", fromlist=["seq"])
for mode in sys.argv[1:]:
    try:
        if mode == "diag":
            sh.run(1, flags=N.TD_F_TALLY | N.TD_F_STATS, spin_limit=1 << 26)
        else:
            sh.run(7, flags=int(mode), spin_limit=1 << 26)
        ok = np.array_equal(sh.tokens(), seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=1 if mode == "diag" else 7))
        print(mode, "ok", ok, "device poison", [d.stats()["poisoned"] for d in sh.shards], flush=True)
    except Exception as e:
        print(mode, "ERR", e, [d.info()["plain"] for d in sh.shards], flush=True)
        for d in sh.shards:
            try: d.wait()
            except Exception as e2: print("  shard wait", e2)
sh.close()

"""METG(50) of the configs[1] patterns vs executor density (columns per worker)."""
import json
import sys

sys.path.insert(0, ".")
from paper_2508_16522_b200.metg import BenchConfig, compute_metg, run_bench  # noqa: E402

iters = tuple(sorted({int(round(2 ** (k / 4))) for k in range(0, 81)}))
for pat in ("stencil_1d", "no_comm"):
    for k in (1, 2, 4, 8, 16):
        cfg = BenchConfig(pattern=pat, width=1024, steps=1000, iterations=iters, repetitions=3, warmups=1,
                          n_workers=1024 // k)
        res = compute_metg(run_bench(cfg))
        print(json.dumps({"pattern": pat, "cols_per_worker": k, "executors": 1024 // k,
                          "metg50_us": None if res.metg_ns is None else round(res.metg_ns / 1e3, 3),
                          "peak": res.peak_rate,
                          "curve": [(round(s.granularity_ns / 1e3, 3), round(s.efficiency, 3)) for s in res.curve[:14]]}),
              flush=True)

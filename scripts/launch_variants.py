"""Event-timed replay of tiny graphs under launch variants (diagnostic; each
variant in its own process).  The TD_DEBUG_LAUNCH switches it drove (bit 1:
cudaLaunchKernel instead of the cooperative launch; bit 2: no dynamic
shared-memory pad; bit 4: no D2H copy behind the kernel) were temporary and are
no longer in tdexec.cu; the results are profiles/r02_launch_variants.log, and
the copy they singled out is gone (the poison mirror)."""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2508_16522_b200.executor import DeviceGraph
from paper_2508_16522_b200.taskbench import generate_graph
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
out = {}
for pat, W, T, wk in [("nearest", 8192, 2, 2048), ("no_comm", 1024, 1, 1024), ("stencil_1d", 1024, 1000, 1024)]:
    g = generate_graph(pat, W, T, n_workers=wk, kind=2 if pat == "stencil_1d" else 0, arg=1 if pat == "stencil_1d" else 0)
    with DeviceGraph(g) as dg:
        for _ in range(3): dg.run(1, flags=0)
        ts = []
        for _ in range(15):
            flush.zero_(); torch.cuda.synchronize()
            dg.run(1, flags=0); ts.append(dg.last_ms() * 1e3)
        out[f"{pat} {W}x{T}"] = round(float(np.median(ts)), 2)
print(json.dumps(out))
'''
res = {}
for v in (0, 1, 2, 4, 7):
    env = dict(os.environ, TD_DEBUG_LAUNCH=str(v))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    res[v] = r.stdout.strip() or r.stderr[-300:]
    print(v, res[v], flush=True)

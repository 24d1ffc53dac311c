"""Where the e2e time of a public-API replay goes (execute / wait / checksums)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2508_16522_b200 import _native as N  # noqa: E402
from paper_2508_16522_b200.compiler import compile as td_compile  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402

g = generate_graph("stencil_1d", 1024, 1000, kind=2, arg=1)
cg = td_compile(g)
for _ in range(5):
    cg.execute(seed=1, flags=N.TD_F_CHECKSUM)[0].wait()
t_ex, t_wait, t_cs, t_tot, kern = [], [], [], [], []
for _ in range(50):
    t0 = time.perf_counter()
    done, _ = cg.execute(seed=1, flags=N.TD_F_CHECKSUM)
    t1 = time.perf_counter()
    done.wait()
    t2 = time.perf_counter()
    cs = cg.checksums()
    t3 = time.perf_counter()
    t_ex.append(t1 - t0), t_wait.append(t2 - t1), t_cs.append(t3 - t2), t_tot.append(t3 - t0)
    kern.append(cg.dev.last_ms())
med = lambda a: 1e3 * float(np.median(a))  # noqa: E731
print(f"execute {med(t_ex):.3f} ms  wait {med(t_wait):.3f} ms  checksums {med(t_cs):.3f} ms  total {med(t_tot):.3f} ms  kernel {np.median(kern):.3f} ms")
# the same replay through the DeviceGraph handle directly (no compiler wrapper)
dev = cg.dev
t_l, t_w, t_t = [], [], []
for _ in range(50):
    t0 = time.perf_counter()
    dev.launch(1, flags=N.TD_F_CHECKSUM)
    t1 = time.perf_counter()
    dev.wait()
    t2 = time.perf_counter()
    t_l.append(t1 - t0), t_w.append(t2 - t1), t_t.append(t2 - t0)
print(f"DeviceGraph.launch {med(t_l):.3f} ms  wait {med(t_w):.3f} ms  total {med(t_t):.3f} ms")
cg.close()

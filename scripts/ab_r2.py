"""Same-box A/B of executor variants (env switches read at upload time) over a
case list that covers the headline, the METG region and the wide graphs.
python scripts/ab_r2.py base noplace group2 ..."""
import json
import os
import subprocess
import sys

CASES = [  # pattern, W, T, kind, arg, workers
    ("stencil_1d", 1024, 1000, 2, 1, 1024), ("no_comm", 1024, 1000, 2, 1, 1024),
    ("stencil_1d", 1024, 1000, 2, 1, 512), ("stencil_1d", 1024, 1000, 2, 1, 256), ("stencil_1d", 1024, 1000, 2, 1, 128),
    ("no_comm", 1024, 1000, 2, 1, 512), ("no_comm", 1024, 1000, 2, 1, 256),
    ("stencil_1d", 1024, 1000, 2, 64, 1024), ("stencil_1d", 1024, 1000, 2, 256, 1024),
    ("no_comm", 1024, 1000, 2, 64, 1024), ("stencil_1d", 1024, 1000, 2, 256, 512),
    ("nearest", 8192, 100, 0, 0, 4736), ("nearest", 8192, 100, 0, 0, 4096), ("nearest", 8192, 100, 0, 0, 2048),
    ("fft", 4096, 1000, 0, 0, 4096), ("fft", 4096, 1000, 0, 0, 2048), ("fft", 4096, 1000, 0, 0, 1024),
    ("tree", 4096, 1000, 0, 0, 4096), ("tree", 4096, 1000, 0, 0, 2048), ("tree", 4096, 1000, 0, 0, 1024),
    ("all_to_all", 8192, 10, 0, 0, 4736),
    ("stencil_1d", 1024, 1000, 2, 2048, 1024), ("no_comm", 1024, 1000, 2, 2048, 1024),
    ("stencil_1d", 1024, 1000, 2, 2048, 512), ("stencil_1d", 1024, 1000, 2, 128, 1024),
]

CHILD = r'''
import json, os, sys, numpy as np, torch
sys.path.insert(0, ".")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
from paper_2508_16522_b200.executor import DeviceGraph
from paper_2508_16522_b200.taskbench import generate_graph
cases = json.loads(os.environ["AB_CASES"])
res = {}
for pat, W, T, kind, arg, wk in cases:
    g = generate_graph(pat, W, T, n_workers=wk, kind=kind, arg=arg)
    with DeviceGraph(g) as dg:
        for _ in range(3): dg.run(1, flags=0)
        ts = []
        for _ in range(11):
            flush.zero_(); torch.cuda.synchronize()
            dg.run(1, flags=0); ts.append(dg.last_ms())
        tk = dg.tokens()
        grp = dg.info()["group"]
    d = int(np.bitwise_xor.reduce(tk * np.uint64(0x9E3779B97F4A7C15) + np.arange(tk.size, dtype=np.uint64)))
    ms = float(np.median(ts))
    key = f"{pat}{W}x{T}/c{arg}/w{wk}"
    res[key] = {"ms": round(ms, 4), "g": grp, "d": f"{d & 0xFFFF:04x}"}
    if kind == 2 and arg >= 16:
        res[key]["eff"] = round(g.n * arg * 64 / (ms * 1e-3) / float(os.environ.get("AB_PEAK", "4.5e12")), 4)
print(json.dumps(res))
'''

VARIANTS = {
    "base": {}, "base2": {}, "base3": {}, "noplace": {"TD_PLACE": "0"}, "place": {"TD_PLACE": "1"}, "group2": {"TD_GROUP": "2"}, "nogroup": {"TD_NO_PAIR": "1"},
    "noplain": {"TD_NO_PLAIN": "1"}, "nopad": {"TD_NO_PAD": "1"},
    "f256": {"TD_SHARE_FANOUT": "256"}, "f1024": {"TD_SHARE_FANOUT": "1024"}, "f2048": {"TD_SHARE_FANOUT": "2048"},
    "f8192": {"TD_SHARE_FANOUT": "8192"},
    "bo32": {"TD_SHARED_BACKOFF": "32"}, "bo64": {"TD_SHARED_BACKOFF": "64"}, "bo128": {"TD_SHARED_BACKOFF": "128"},
    "oldlib": {"TD_LIB": "paper_2508_16522_b200/libtdexec_old.so"},  # (previous builds, A/B of kernel changes)
    "midlib": {"TD_LIB": "paper_2508_16522_b200/libtdexec_mid.so"},
    "xopt": {"TD_LIB": "paper_2508_16522_b200/libtdexec_xopt.so"},  # -Xptxas --allow-expensive-optimizations
    "xo3": {"TD_LIB": "paper_2508_16522_b200/libtdexec_xo3.so"},  # the previous build (A/B of kernel changes)
    "ss4": {"TD_SHARE_STRIDE": "4"}, "ss8": {"TD_SHARE_STRIDE": "8"}, "ss16": {"TD_SHARE_STRIDE": "16"},
    "mixring": {"TD_MIXED_RING": "1"}, "forcemulti": {"TD_FORCE_MULTI": "1"},
    "comb0": {"TD_COMBINE": "0"}, "comb1": {"TD_COMBINE": "1"}, "ss32": {"TD_SHARE_STRIDE": "32"},
    "comb1ss32": {"TD_COMBINE": "1", "TD_SHARE_STRIDE": "32"},
    "bo256": {"TD_SHARED_BACKOFF": "256"}, "bo512": {"TD_SHARED_BACKOFF": "512"},
    "slot1": {"TD_SLOT_SHIFT": "1"}, "slot3": {"TD_SLOT_SHIFT": "3"},
    "slot0": {"TD_SLOT_SHIFT": "0"}, "slot2": {"TD_SLOT_SHIFT": "2"},  # mailbox spacing override
}
if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["base", "noplace"]
    sel = os.environ.get("AB_SELECT")
    cases = [c for c in CASES if not sel or any(s in c[0] for s in sel.split(","))]
    if os.environ.get("AB_CASES_JSON"):  # explicit case list: [[pattern, W, T, kind, arg, workers], ...]
        cases = json.loads(os.environ["AB_CASES_JSON"])
    out_all = {}
    for rep in range(2):
        for name in names:
            env = dict(os.environ, **VARIANTS.get(name, {}), AB_CASES=json.dumps(cases))
            out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            line = out.stdout.strip() or out.stderr[-800:]
            print(name, rep, line, flush=True)
            try:
                out_all.setdefault(name, []).append(json.loads(line))
            except Exception:
                pass
    # summary: per case, best-of-reps ms per variant
    keys = list(next(iter(out_all.values()))[0]) if out_all else []
    for k in keys:
        row = []
        for name in names:
            vals = [r[k]["ms"] for r in out_all.get(name, []) if k in r]
            g = [r[k]["g"] for r in out_all.get(name, []) if k in r]
            e = [r[k].get("eff") for r in out_all.get(name, []) if k in r]
            dg = {r[k]["d"] for r in out_all.get(name, []) if k in r}
            row.append(f"{name}={min(vals) if vals else None}(g{g[0] if g else '-'}{',e' + str(max(x for x in e if x)) if any(e) else ''},{'/'.join(sorted(dg))})")
        print(f"{k:40s} " + "  ".join(row))

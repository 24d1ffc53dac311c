#!/bin/bash
# PAIR mode: parity tests, same-box timing of multi-column graphs, METG with and without.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pair or plain" > gpurun_out/pair_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pair_tests.log
cat > /tmp/pair_time.py <<'PY'
import json, os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2508_16522_b200.executor import DeviceGraph
from paper_2508_16522_b200.taskbench import generate_graph
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {}
for pat, W, T, wk, kind, arg in [("stencil_1d", 1024, 1000, 128, 2, 1), ("no_comm", 1024, 1000, 128, 2, 1), ("stencil_1d", 1024, 1000, 512, 2, 1), ("stencil_1d", 1024, 1000, 128, 2, 64)]:
    g = generate_graph(pat, W, T, n_workers=wk, mapping="block", kind=kind, arg=arg)
    with DeviceGraph(g) as dg:
        for _ in range(3): dg.run(1, flags=0)
        ts = []
        for _ in range(15):
            flush.zero_(); torch.cuda.synchronize()
            dg.run(1, flags=0); ts.append(dg.last_ms())
        tk = dg.tokens()
    res[f"{pat}{W}x{T}/w{wk}/it{arg}"] = round(float(np.median(ts)), 4)
res["digest"] = f"{int(np.bitwise_xor.reduce(tk)):016x}"
print(json.dumps(res))
PY
for rep in 1 2; do
  timeout 300 python /tmp/pair_time.py 2>&1 | tail -1; echo " <- pair"
  TD_NO_PAIR=1 timeout 300 python /tmp/pair_time.py 2>&1 | tail -1; echo " <- no pair"
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-extra --no-cpu --no-parity > gpurun_out/metg_pair.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/metg_pair.json').readlines()[-1]); print('pair METG', {k:(round(v['metg50_us'],3), v['executors']) for k,v in d['metg'].items()})"
TD_NO_PAIR=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-extra --no-cpu --no-parity > gpurun_out/metg_nopair.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/metg_nopair.json').readlines()[-1]); print('no-pair METG', {k:(round(v['metg50_us'],3), v['executors']) for k,v in d['metg'].items()})"

#!/bin/bash
# replay kernel launched as a one-node CUDA graph (TD_GRAPH_LAUNCH=1) vs cudaLaunchCooperativeKernel
O=gpurun_out/r2gl; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
TD_GRAPH_LAUNCH=1 timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest_gl.log 2>&1; echo "pytest graph-launch rc=$?"; tail -1 $O/pytest_gl.log
for gl in 0 1; do
  echo "--- TD_GRAPH_LAUNCH=$gl"
  TD_GRAPH_LAUNCH=$gl python scripts/e2e_probe.py 2>&1 | tail -2
  TD_GRAPH_LAUNCH=$gl python scripts/fixed_cost.py > $O/fixed_$gl.json; python -c "import json; d=json.load(open('$O/fixed_$gl.json')); print({k: v['flush'] for k, v in d.items()})"
  TD_GRAPH_LAUNCH=$gl timeout 300 python bench.py --steps 20 --warmup 5 --no-metg --no-extra --no-cpu > $O/bench_$gl.json 2> $O/bench_$gl.err; python -c "import json;d=json.load(open('$O/bench_$gl.json'));print('bench', d['value'], 'e2e', d['e2e']['value'], d['ms_per_step'])"
done

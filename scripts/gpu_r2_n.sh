#!/bin/bash
O=gpurun_out/r2n; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for spec in "fft 4096 1000 0 0 1024" "stencil_1d 1024 1000 2 1 1024" "tree 4096 1000 0 0 1024"; do
  TD_UPLOAD_PROFILE=1 timeout 120 python scripts/run_pattern.py $spec >> $O/upload_profile.log 2>&1
done; cat $O/upload_profile.log
timeout 2400 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -3 $O/bench.err
python -c "
import json; d=json.loads(open('$O/bench.json').read()); print(d['value'], d['compile_ms']); print(json.dumps(d['other_configs']['comparators'])[:600])
for k,v in d['other_configs'].items():
  if 'compile' in v: print(k, v['compile'], v['replay_ms'])
"

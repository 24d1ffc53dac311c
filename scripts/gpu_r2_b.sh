#!/bin/bash
# round 2: long-body parity + METG with a fixed chip peak
O=gpurun_out/r2b; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_native_abi.py -m gpu -x -q -k "long_bodies or group" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
python -m paper_2508_16522_b200.roofline > $O/microbench.json 2>&1
python -c "
import json
from paper_2508_16522_b200 import roofline as RF
print(json.dumps(RF.compute_peak(0)))" > $O/compute_peak.json 2>&1; cat $O/compute_peak.json
timeout 1500 python bench.py --steps 5 --warmup 3 --no-cpu --no-parity > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -30 $O/bench.err | grep -v "^\s" ; head -c 600 $O/bench.json

#!/bin/bash
# Multi-GPU session (run with gpurun --gpus N): sharded parity + scaling bench.
mkdir -p gpurun_out
NG=$(python -c "import torch; print(torch.cuda.device_count())")
echo "GPUs: $NG"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 tests/tools/mgpu_check.py > gpurun_out/mgpu_check.log 2>&1; echo "mgpu rc=$?"; grep -E "parity|Error|error" gpurun_out/mgpu_check.log | tail -40
for N in 2 4; do
  if [ $N -le $NG ]; then
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench N=$N rc=$?"; head -c 700 gpurun_out/bench_n$N.json; echo
  fi
done
timeout 300 python -c "
import json, sys; sys.path.insert(0,'.')
from paper_2508_16522_b200 import roofline as R
print(json.dumps(R.measure(0, 148, p2p_peer=1)))" 2>&1 | tail -2

#!/bin/bash
# 4-GPU session (gpurun --gpus 4): sharded parity, weak scaling of the bench
# headline, strong scaling of configs[3]/[4], microbenchmarks incl. P2P.
mkdir -p gpurun_out
NG=$(python -c "import torch; print(torch.cuda.device_count())")
echo "GPUs: $NG"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 tests/tools/mgpu_check.py > gpurun_out/mgpu_check.log 2>&1; echo "mgpu rc=$?"; grep -E "parity|Error|error" gpurun_out/mgpu_check.log | tail -40
for N in 2 4; do
  if [ $N -le $NG ]; then
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench N=$N rc=$?"; head -c 400 gpurun_out/bench_n$N.json; echo
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --impl reference --gpus $N --steps 2 --warmup 1 > gpurun_out/bench_ref_n$N.json 2> gpurun_out/bench_ref_n$N.err; echo "ref N=$N rc=$?"; head -c 200 gpurun_out/bench_ref_n$N.json; echo
  fi
done
for N in 1 2 4; do
  HALOS=0,16 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N tests/tools/bench_multigpu.py > gpurun_out/strong_n$N.jsonl 2> gpurun_out/strong_n$N.err; echo "strong N=$N rc=$?"; cat gpurun_out/strong_n$N.jsonl | cut -c1-200
done
timeout 300 python -c "
import json, sys; sys.path.insert(0,'.')
from paper_2508_16522_b200 import roofline as R
print(json.dumps(R.measure(0, 148, p2p_peer=1)))" > gpurun_out/rf4.json 2>&1; tail -c 1500 gpurun_out/rf4.json

#!/bin/bash
# Multi-GPU re-check of the current tree: sharded parity at N=2 (and N=4 when
# 4 GPUs are visible) and the weak-scaling bench at each N.
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l); echo "gpus=$NG"
for N in 2 4; do
  [ "$N" -le "$NG" ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 295$N tests/tools/mgpu_check.py > gpurun_out/mgpu_check_n$N.log 2>&1; echo "mgpu N=$N rc=$?"; grep -c "parity=True" gpurun_out/mgpu_check_n$N.log; grep -E "parity=False|Error|error" gpurun_out/mgpu_check_n$N.log | head
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 296$N bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench N=$N rc=$?"; head -c 400 gpurun_out/bench_n$N.json; echo
done

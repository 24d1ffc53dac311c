#!/bin/bash
# 2-GPU check: GPU tests, sharded parity, weak-scaling bench at N=2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tests/tools/mgpu_check.py > gpurun_out/mgpu_check.log 2>&1; echo "mgpu rc=$?"; grep -c "parity=True" gpurun_out/mgpu_check.log; grep -E "parity=False|Error|error" gpurun_out/mgpu_check.log | head
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench N=2 rc=$?"; head -c 400 gpurun_out/bench_n2.json; echo

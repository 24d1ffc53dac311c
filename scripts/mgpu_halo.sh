#!/bin/bash
# 4-GPU halo-period sweep: nearest strong scaling and the weak-scaling headline.
mkdir -p gpurun_out
HALOS=16,32,64 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 tests/tools/bench_multigpu.py > gpurun_out/halo_strong_n4.jsonl 2> gpurun_out/halo_strong_n4.err; echo "strong rc=$?"; grep nearest gpurun_out/halo_strong_n4.jsonl | cut -c1-200
for K in 16 32 64; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$((K % 10)) bench.py --gpus 4 --steps 20 --warmup 3 --halo $K --no-parity > gpurun_out/halo_bench_k$K.json 2> gpurun_out/halo_bench_k$K.err; echo "bench k=$K rc=$?"; head -c 250 gpurun_out/halo_bench_k$K.json; echo
done

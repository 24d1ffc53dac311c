#!/bin/bash
# 4-GPU session (gpurun --gpus 4): weak scaling of the bench headline (both
# arms), METG at the paper's widths on 2/4 GPUs.
mkdir -p gpurun_out
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench N=$N rc=$? lines=$(wc -l < gpurun_out/bench_n$N.json)"; head -c 400 gpurun_out/bench_n$N.json; echo
done
timeout 600 python scripts/metg_sharded.py > gpurun_out/metg_w_n1.jsonl 2> gpurun_out/metg_w_n1.err; echo "metg N=1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N scripts/metg_sharded.py > gpurun_out/metg_w_n$N.jsonl 2> gpurun_out/metg_w_n$N.err; echo "metg N=$N rc=$?"
  METG_HALO=16 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N scripts/metg_sharded.py > gpurun_out/metg_w_n${N}_h16.jsonl 2> gpurun_out/metg_w_n${N}_h16.err; echo "metg halo N=$N rc=$?"
done
grep -h "^{" gpurun_out/metg_w_n*.jsonl | cut -c1-120

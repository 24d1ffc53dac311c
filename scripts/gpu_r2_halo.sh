#!/bin/bash
# weak-scaling headline on 2 GPUs at several halo periods
O=gpurun_out/r2halo; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
for h in 32 64 128 256; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$((h % 10)) bench.py --gpus 2 --steps 20 --warmup 5 --no-metg --no-extra --no-cpu --halo $h > $O/b_$h.json 2> $O/b_$h.err
  echo "halo $h rc=$? $(python -c "import json;d=json.load(open('$O/b_$h.json'));print(d['value'], d['ms_per_step'], d['config'].get('halo_replicas'))" 2>&1 | tail -1)"
done

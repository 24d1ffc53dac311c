#!/bin/bash
# sharded headline (stencil_1d 1024*N x 1000, halo 64) at mailbox spacing 8 B vs 32 B
O=gpurun_out/r2n2s; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
for rep in 1 2 3; do for sh in 0 2; do
  TD_SLOT_SHIFT=$sh timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$sh bench.py --gpus 2 --steps 20 --warmup 5 --no-metg --no-extra --no-cpu > $O/b_${sh}_$rep.json 2> $O/b_${sh}_$rep.err
  echo "shift $sh rep $rep rc=$? $(python -c "import json;d=json.load(open('$O/b_${sh}_$rep.json'));print(d['value'], d['ms_per_step'])")"
done; done
TD_SLOT_SHIFT=2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29530 tests/tools/mgpu_check.py > $O/mgpu_check.log 2>&1; echo "mgpu_check rc=$?"; tail -2 $O/mgpu_check.log

#!/bin/bash
# round 2: bench at N=2 (and the reference arm under torchrun) as the driver runs them
O=gpurun_out/r2n${1:-2}${2:-}; mkdir -p $O
N=${1:-2}
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --impl reference --gpus $N --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"; head -c 300 $O/ref.json; echo
start=$(date +%s); timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$? $(( $(date +%s) - start )) s"; grep -v "^\s*$" $O/bench.err | tail -8; head -c 1200 $O/bench.json; echo

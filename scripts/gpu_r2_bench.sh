#!/bin/bash
# round 2: both bench arms as the driver runs them (N=1)
O=gpurun_out/r2bench; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"; head -c 600 $O/ref.json; echo
start=$(date +%s); timeout 2400 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$? $(( $(date +%s) - start )) s"; tail -30 $O/bench.err; head -c 1500 $O/bench.json; echo

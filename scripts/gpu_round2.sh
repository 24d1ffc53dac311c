#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; head -c 600 gpurun_out/bench.json; echo
CMD="python tests/tools/bench_stencil2d.py --n 4096 --steps 5 --reps 1"
timeout 300 $CMD > gpurun_out/plain_st.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 4 -c 1 -o gpurun_out/prof_st2d $CMD > gpurun_out/ncu_st.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_st.log

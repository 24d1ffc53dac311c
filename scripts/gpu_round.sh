#!/bin/bash
# One GPU session: parity tests, smoke, bench, comparators, ncu launch list + full capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; head -c 1500 gpurun_out/bench.json; echo
timeout 600 python tests/tools/compare.py > gpurun_out/compare.jsonl 2>&1; echo "compare rc=$?"; cat gpurun_out/compare.jsonl
CMD="python bench.py --steps 3 --warmup 3 --no-metg --no-cpu --no-parity --no-extra"
if [ "${NCU:-1}" = "1" ]; then
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 3 -c 1 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
fi

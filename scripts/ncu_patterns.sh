#!/bin/bash
# full ncu captures of the executor on fft 4096x1000 and no_comm 1024x1000
mkdir -p gpurun_out
for spec in "fft 4096 1000 0 0" "no_comm 1024 1000 2 1"; do
  set -- $spec
  timeout 300 python scripts/run_pattern.py $spec > gpurun_out/run_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 2 -c 1 -o gpurun_out/prof_$1 python scripts/run_pattern.py $spec > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?"; cat gpurun_out/run_$1.log
done
timeout 600 python tests/tools/sanitize_cases.py > gpurun_out/cases.log 2>&1; echo "cases rc=$?"; tail -2 gpurun_out/cases.log

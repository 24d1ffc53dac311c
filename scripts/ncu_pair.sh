#!/bin/bash
# ncu full captures of the PAIR-mode node loop vs the unpaired PLAIN loop on the
# METG configuration (stencil_1d 1024x1000, 128 workers = 8 columns per worker,
# compute_bound(23), i.e. the granularity at METG(50)).
mkdir -p gpurun_out
SPEC="stencil_1d 1024 1000 2 23 128"
for mode in pair nopair; do
  if [ $mode = nopair ]; then export TD_NO_PAIR=1; else unset TD_NO_PAIR; fi
  timeout 300 python scripts/run_pattern.py $SPEC > gpurun_out/run_$mode.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 2 -c 1 -o gpurun_out/prof_$mode python scripts/run_pattern.py $SPEC > gpurun_out/ncu_$mode.log 2>&1
  echo "$mode rc=$?"; cat gpurun_out/run_$mode.log
done

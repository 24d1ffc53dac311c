#!/bin/bash
# round 2 ncu: launch list of the headline bench command; full captures of the
# headline kernel, nearest 8192x100 (2048 workers, GROUP 4 and 4736 workers),
# fft 4096x1000 (1024 workers) and the config-5 tile kernel.  Each command is
# first run without ncu.
O=gpurun_out/r2ncu; mkdir -p $O
CMD="python bench.py --steps 3 --warmup 3 --no-metg --no-cpu --no-parity --no-extra"
timeout 300 $CMD > $O/plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 3 -c 1 -o $O/prof_headline $CMD > $O/ncu_headline.log 2>&1; echo "headline rc=$?"
for spec in "nearest 8192 100 0 0 2048" "nearest 8192 100 0 0 4736" "fft 4096 1000 0 0 1024"; do
  name=$(echo $spec | awk '{print $1"_"$6}')
  timeout 120 python scripts/run_pattern.py $spec > $O/run_$name.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 3 -c 1 -o $O/prof_$name python scripts/run_pattern.py $spec > $O/ncu_$name.log 2>&1; echo "$name rc=$?"
done
timeout 120 python tests/tools/bench_stencil2d.py --reps 2 > $O/run_st2d.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 3 -c 1 -o $O/prof_st2d python tests/tools/bench_stencil2d.py --reps 2 > $O/ncu_st2d.log 2>&1; echo "st2d rc=$?"
ls -la $O

#!/bin/bash
# round 2 final pass: poison mirror (placement counter reverted): tests, smoke, both bench arms, ncu captures
O=gpurun_out/r2final7; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; cat $O/smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
timeout 2400 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -16 $O/bench.err
CMD="python bench.py --steps 3 --warmup 3 --no-metg --no-cpu --no-parity --no-extra"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 3 -c 1 -o $O/prof_headline $CMD > $O/ncu_headline.log 2>&1; echo "headline rc=$?"
for spec in "nearest 8192 100 0 0 2048" "fft 4096 1000 0 0 1024" "tree 4096 1000 0 0 1024"; do
  name=$(echo $spec | awk '{print $1"_"$6}')
  timeout 120 python scripts/run_pattern.py $spec > $O/run_$name.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 3 -c 1 -o $O/prof_$name python scripts/run_pattern.py $spec > $O/ncu_$name.log 2>&1; echo "$name rc=$?"
done
for spec in "all_to_all 8192 10 0 0 4096"; do
  name=$(echo $spec | awk '{print $1"_"$6}')
  timeout 120 python scripts/run_pattern.py $spec > $O/run_$name.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 3 -c 1 -o $O/prof_$name python scripts/run_pattern.py $spec > $O/ncu_$name.log 2>&1; echo "$name rc=$?"
done

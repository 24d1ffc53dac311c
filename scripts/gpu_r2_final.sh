#!/bin/bash
# round 2 final single-GPU pass: tests, smoke, both bench arms, ncu of the
# GROUP kernels after the empty-body skip, cycle probe of the headline
O=gpurun_out/r2final; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; cat $O/smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
timeout 2400 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -16 $O/bench.err; head -c 800 $O/bench.json; echo
for spec in "nearest 8192 100 0 0 2048" "fft 4096 1000 0 0 1024" "tree 4096 1000 0 0 1024"; do
  name=$(echo $spec | awk '{print $1"_"$6}')
  timeout 120 python scripts/run_pattern.py $spec > $O/run_$name.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 3 -c 1 -o $O/prof_$name python scripts/run_pattern.py $spec > $O/ncu_$name.log 2>&1; echo "$name rc=$?"
done
for spec in "fft 4096 1000 0 0 1024" "stencil_1d 1024 1000 2 1 1024" "all_to_all 8192 10 0 0 4736"; do
  TD_UPLOAD_PROFILE=1 timeout 120 python scripts/run_pattern.py $spec >> $O/upload_profile.log 2>&1
done; cat $O/upload_profile.log
timeout 600 python scripts/cycle_probe.py > $O/cycle_probe.log 2>&1; echo "probe rc=$?"; tail -5 $O/cycle_probe.log | cut -c1-400

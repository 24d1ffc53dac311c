#!/bin/bash
O=gpurun_out/r2m; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for spec in "fft 4096 1000 0 0 1024" "stencil_1d 1024 1000 2 1 1024" "nearest 8192 100 0 0 2048" "all_to_all 8192 10 0 0 4736"; do
  TD_UPLOAD_PROFILE=1 timeout 120 python scripts/run_pattern.py $spec >> $O/upload_profile.log 2>&1
done; cat $O/upload_profile.log
nproc

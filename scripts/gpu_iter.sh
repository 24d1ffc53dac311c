#!/bin/bash
# One development iteration on one B200: GPU tests, same-box A/B against the
# previous build (libtdexec_prev.so), one full ncu capture of the headline kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python scripts/ab.py base prev > gpurun_out/ab.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab.log
CMD="python bench.py --steps 3 --warmup 3 --no-metg --no-cpu --no-parity --no-extra"
if [ "${NCU:-1}" = "1" ]; then
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 3 -c 1 -o gpurun_out/prof_iter $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log
fi

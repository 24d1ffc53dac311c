#!/bin/bash
# Same-box A/B of the config-5 tile kernel: base build vs a variant library.
# usage: bash scripts/ab_st2d.sh <variant>   (libtdexec_<variant>.so built by scripts/ab.py)
mkdir -p gpurun_out
V=paper_2508_16522_b200/libtdexec_$1.so
TD_LIB=$V timeout 900 python -m pytest tests/test_gpu_stencil2d.py tests/test_gpu_shards.py -q -x -k "stencil2d" > gpurun_out/st2d_var_tests.log 2>&1; echo "variant tests rc=$?"; tail -2 gpurun_out/st2d_var_tests.log
for rep in 1 2; do
  timeout 600 python tests/tools/bench_stencil2d.py --reps 5 2>/dev/null | tail -1 | cut -c1-400; echo " <- base"
  TD_LIB=$V timeout 600 python tests/tools/bench_stencil2d.py --reps 5 2>/dev/null | tail -1 | cut -c1-400; echo " <- $1"
done

#!/bin/bash
# same-box A/B of executor build variants: bash scripts/ab_run.sh base nodiag ...
mkdir -p gpurun_out
timeout 1500 python scripts/ab.py "$@" > gpurun_out/ab.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab.log

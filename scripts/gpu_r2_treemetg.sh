#!/bin/bash
O=gpurun_out/r2tm; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
AB_CASES_JSON='[["tree",4096,1000,2,64,4096],["tree",4096,1000,2,256,4096],["tree",4096,1000,2,64,4096]]' timeout 900 python scripts/ab_r2.py base oldlib midlib > $O/ab.log 2>&1; tail -4 $O/ab.log

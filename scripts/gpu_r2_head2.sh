#!/bin/bash
O=gpurun_out/r2head2; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
AB_CASES_JSON='[["stencil_1d",1024,1000,2,1,1024],["stencil_1d",1024,1000,2,1,512]]' timeout 900 python scripts/ab_r2.py base base2 base3 > $O/ab.log 2>&1; tail -2 $O/ab.log

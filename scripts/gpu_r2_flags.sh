#!/bin/bash
O=gpurun_out/r2flags; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
AB_CASES_JSON='[["stencil_1d",1024,1000,2,1,1024],["no_comm",1024,1000,2,1,1024],["nearest",8192,100,0,0,2048],["fft",4096,1000,0,0,1024],["tree",4096,1000,0,0,1024],["all_to_all",8192,10,0,0,4096],["stencil_1d",1024,1000,2,256,1024]]' timeout 900 python scripts/ab_r2.py base xopt xo3 > $O/ab.log 2>&1; tail -7 $O/ab.log

#!/bin/bash
# mailbox spacing for GROUP graphs after the ring changes
O=gpurun_out/r2gslot; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
AB_CASES_JSON='[["nearest",8192,100,0,0,2048],["fft",4096,1000,0,0,1024],["tree",4096,1000,0,0,1024],["stencil_1d",8192,100,0,0,2048],["stencil_1d",1024,1000,2,1,512],["no_comm",1024,1000,2,1,512]]' timeout 900 python scripts/ab_r2.py base slot1 slot2 > $O/ab.log 2>&1; tail -6 $O/ab.log

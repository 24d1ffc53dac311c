#!/bin/bash
# headline stencil_1d 1024x1000 compute(1): one node per warp (1024 w) vs
# GROUP 2 (512 w) after the GROUP ring changes, at several mailbox spacings
O=gpurun_out/r2head; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
AB_CASES_JSON='[["stencil_1d",1024,1000,2,1,1024],["stencil_1d",1024,1000,2,1,512],["stencil_1d",1024,1000,2,1,256],["no_comm",1024,1000,2,1,1024],["no_comm",1024,1000,2,1,512]]' \
  timeout 900 python scripts/ab_r2.py base slot0 slot1 slot2 slot3 > $O/ab.log 2>&1; echo "ab rc=$?"; tail -5 $O/ab.log

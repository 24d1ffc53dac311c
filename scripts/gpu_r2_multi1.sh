#!/bin/bash
# per-node overhead of the sharded kernel on one shard (TD_FORCE_MULTI=1)
O=gpurun_out/r2m1; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
AB_CASES_JSON='[["stencil_1d",1024,1000,2,1,1024],["no_comm",1024,1000,2,1,1024]]' timeout 900 python scripts/ab_r2.py base forcemulti > $O/ab.log 2>&1; tail -2 $O/ab.log

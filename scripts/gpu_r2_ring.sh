#!/bin/bash
# GROUP ring adds: match + warp reductions instead of 64-bit shared CAS loops
O=gpurun_out/r2ring; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
TD_LIB=paper_2508_16522_b200/libtdexec_checks.so timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest_checks.log 2>&1; echo "checks rc=$?"; tail -1 $O/pytest_checks.log
timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
AB_CASES_JSON='[["stencil_1d",8192,100,0,0,2048],["nearest",8192,100,0,0,2048],["nearest",8192,100,0,0,1024],["fft",4096,1000,0,0,1024],["tree",4096,1000,0,0,1024],["tree",4096,1000,0,0,2048],["stencil_1d",1024,1000,2,1,512],["stencil_1d",1024,1000,2,1,256],["no_comm",1024,1000,2,1,512],["stencil_1d",1024,1000,2,1,1024],["stencil_1d",1024,1000,2,256,512]]' \
  timeout 1200 python scripts/ab_r2.py base mixring > $O/ab.log 2>&1; echo "ab rc=$?"; tail -11 $O/ab.log
for spec in "stencil_1d 8192 100 2048" "nearest 8192 100 2048"; do timeout 120 python scripts/group_probe.py $spec >> $O/probe.log 2>&1; done
python -c "
import json
for l in open('$O/probe.log'):
    d=json.loads(l); print(d['graph'], {k: round(d[k]['mean']) for k in ('wait','proc','send','tail','gap')}, d['warp_last_end_us_pct'])"

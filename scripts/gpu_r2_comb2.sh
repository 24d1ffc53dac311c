#!/bin/bash
# deferred completion of combiner adds
O=gpurun_out/r2comb2; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
TD_LIB=paper_2508_16522_b200/libtdexec_checks.so timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest_checks.log 2>&1; echo "checks rc=$?"; tail -1 $O/pytest_checks.log
timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
AB_CASES_JSON='[["all_to_all",8192,10,0,0,4096],["all_to_all",8192,100,0,0,4736],["all_to_all",4096,100,0,0,4096],["all_to_all",8192,10,2,1,4096],["stencil_1d",1024,1000,1,0,1024]]' timeout 900 python scripts/ab_r2.py base oldlib > $O/ab.log 2>&1; tail -5 $O/ab.log

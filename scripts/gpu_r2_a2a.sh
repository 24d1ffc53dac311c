#!/bin/bash
# all_to_all (BASELINE configs[3]): combiners (default policy / forced / off);
# bundled tests on the bounds-checked build, then the GPU suite
O=gpurun_out/r2a2a; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
TD_LIB=paper_2508_16522_b200/libtdexec_checks.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "combiner or all_to_all" > $O/pytest_checks.log 2>&1; echo "checks rc=$?"; tail -1 $O/pytest_checks.log
timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
AB_CASES_JSON='[["all_to_all",1024,100,0,0,1024],["all_to_all",2048,100,0,0,2048],["all_to_all",2048,100,0,0,1024],["all_to_all",4096,100,0,0,4096],["all_to_all",4096,100,0,0,2048],["all_to_all",8192,100,0,0,4736],["all_to_all",8192,100,0,0,2048],["all_to_all",8192,10,0,0,4736],["all_to_all",8192,10,0,0,4096],["all_to_all",8192,10,0,0,2048],["all_to_all",8192,10,2,1,4736],["all_to_all",16384,10,0,0,4736]]' \
  timeout 1200 python scripts/ab_r2.py base comb0 > $O/ab_comb3.log 2>&1; echo "ab rc=$?"; tail -12 $O/ab_comb3.log

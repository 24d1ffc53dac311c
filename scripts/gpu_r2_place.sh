#!/bin/bash
# placement arrival counters: one returning add per CTA (banked) instead of a CAS loop
O=gpurun_out/r2place; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
TD_LIB=paper_2508_16522_b200/libtdexec_checks.so timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest_checks.log 2>&1; echo "checks rc=$?"; tail -1 $O/pytest_checks.log
TD_PLACE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dynamic.py -q -x -m gpu > $O/pytest_place.log 2>&1; echo "forced placement rc=$?"; tail -1 $O/pytest_place.log
timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
python scripts/fixed_cost2.py | tee $O/fixed_cost2.json
AB_CASES_JSON='[["fft",4096,1000,0,0,4096],["tree",4096,1000,0,0,4096],["nearest",8192,100,0,0,4736],["fft",4096,1000,0,0,1024],["stencil_1d",1024,1000,2,1,1024]]' timeout 900 python scripts/ab_r2.py base noplace > $O/ab.log 2>&1; tail -5 $O/ab.log

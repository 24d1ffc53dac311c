#!/bin/bash
O=gpurun_out/r2san; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
# the bounds-checked variant of the same source (-DTD_CHECKS: TD_CHECK asserts in tdexec.cu)
[ -f paper_2508_16522_b200/libtdexec_checks.so ] || (cd paper_2508_16522_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo \
  -Xcompiler -fPIC,-fopenmp -shared -std=c++17 -lgomp -DTD_CHECKS -o ../libtdexec_checks.so tdexec.cu) >> $O/build.log 2>&1
timeout 300 python tests/tools/sanitize_cases.py > $O/plain.log 2>&1; echo "plain rc=$?"; tail -1 $O/plain.log
TD_LIB=paper_2508_16522_b200/libtdexec_checks.so timeout 300 python tests/tools/sanitize_cases.py > $O/plain_checks.log 2>&1; echo "plain checks rc=$?"; tail -1 $O/plain_checks.log
# (compute-sanitizer is closed on the GPU pool; the -DTD_CHECKS build adds
# device-side bounds checks instead: run the whole GPU suite on it)
TD_LIB=paper_2508_16522_b200/libtdexec_checks.so timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_checks.log 2>&1; echo "checks rc=$?"; tail -3 $O/pytest_checks.log

#!/bin/bash
O=gpurun_out/r2p; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py tests/test_gpu_dynamic.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
TD_LIB=paper_2508_16522_b200/libtdexec_slot2.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py tests/test_gpu_dynamic.py -m gpu -q -x > $O/pytest_slot2.log 2>&1; echo "pytest slot2 rc=$?"; tail -2 $O/pytest_slot2.log
AB_SELECT=stencil,no_comm,tree,fft,nearest,all_to_all timeout 900 python scripts/ab_r2.py base slot2 slot4 > $O/ab.log 2>&1; echo "ab rc=$?"; tail -23 $O/ab.log

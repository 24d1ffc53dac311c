#!/bin/bash
O=gpurun_out/r2ss; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "combiner or all_to_all" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
TD_SHARE_STRIDE=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "combiner or all_to_all" > $O/pytest4.log 2>&1; echo "pytest ss4 rc=$?"; tail -1 $O/pytest4.log
AB_CASES_JSON='[["all_to_all",8192,10,0,0,4096],["all_to_all",8192,100,0,0,4736],["all_to_all",4096,100,0,0,4096],["all_to_all",2048,100,0,0,2048],["all_to_all",8192,10,0,0,2048]]' timeout 900 python scripts/ab_r2.py base ss4 ss8 ss16 > $O/ab.log 2>&1; tail -5 $O/ab.log

#!/bin/bash
O=gpurun_out/r2ring2; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
AB_CASES_JSON='[["no_comm",1024,1000,2,1,512],["stencil_1d",1024,1000,2,1,512],["nearest",8192,100,0,0,2048],["tree",4096,1000,0,0,1024],["fft",4096,1000,0,0,1024],["stencil_1d",8192,100,0,0,2048],["no_comm",1024,1000,2,64,512]]' timeout 900 python scripts/ab_r2.py base oldlib > $O/ab.log 2>&1; tail -7 $O/ab.log

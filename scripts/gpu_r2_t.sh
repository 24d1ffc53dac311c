#!/bin/bash
O=gpurun_out/r2t; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_stencil2d.py tests/test_gpu_shards.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 120 python tests/tools/bench_stencil2d.py --reps 5 > $O/st2d.json 2>&1; cat $O/st2d.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:td_exec -s 3 -c 1 -o $O/prof_st2d python tests/tools/bench_stencil2d.py --reps 2 > $O/ncu_st2d.log 2>&1; echo "ncu rc=$?"

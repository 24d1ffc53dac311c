#!/bin/bash
# round 2: dynamic fix, new GPU tests, dynamic A/B, early-poll A/B
O=gpurun_out/r2f; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_dynamic.py tests/test_gpu_formats_comparators.py tests/test_gpu_api.py tests/test_implicit.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -8 $O/pytest.log
timeout 400 python scripts/ab_dynamic.py > $O/ab_dynamic.log 2>&1; echo "ab rc=$?"; tail -9 $O/ab_dynamic.log | head -8
AB_SELECT=stencil,no_comm,nearest,fft,tree timeout 600 python scripts/ab_r2.py base early > $O/ab_early.log 2>&1; echo "ab early rc=$?"; tail -14 $O/ab_early.log

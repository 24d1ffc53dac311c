#!/bin/bash
# round 2: dynamic v2 tests + A/B, formats/comparators tests
O=gpurun_out/r2e; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dynamic.py tests/test_gpu_formats_comparators.py tests/test_gpu_api.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -8 $O/pytest.log
timeout 900 python scripts/ab_dynamic.py > $O/ab_dynamic.log 2>&1; echo "ab rc=$?"; tail -9 $O/ab_dynamic.log | head -8

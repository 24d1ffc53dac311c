#!/bin/bash
# round 2: full GPU suite (memory body, dynamic mode, sticky poison, replay state) + dynamic A/B
O=gpurun_out/r2d; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -8 $O/pytest.log
timeout 900 python scripts/ab_dynamic.py > $O/ab_dynamic.log 2>&1; echo "ab rc=$?"; tail -9 $O/ab_dynamic.log

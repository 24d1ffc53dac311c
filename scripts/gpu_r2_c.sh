#!/bin/bash
# round 2: placement + group mode tests and A/B
O=gpurun_out/r2c; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout 1500 python scripts/ab_r2.py base noplace group2 > $O/ab.log 2>&1; echo "ab rc=$?"; tail -16 $O/ab.log

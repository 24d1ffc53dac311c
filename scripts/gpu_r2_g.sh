#!/bin/bash
# round 2: full GPU suite, config-5 A/B, ncu captures
O=gpurun_out/r2g; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
timeout 900 bash scripts/ab_st2d_r2.sh > $O/ab_st2d.log 2>&1; echo "ab st2d rc=$?"; cat $O/ab_st2d.log | cut -c1-250
bash scripts/ncu_r2.sh

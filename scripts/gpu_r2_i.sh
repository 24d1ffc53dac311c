#!/bin/bash
O=gpurun_out/r2i; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
AB_SELECT=stencil,no_comm,tree timeout 900 python scripts/ab_r2.py base place > $O/ab.log 2>&1; echo "ab rc=$?"; tail -16 $O/ab.log

#!/bin/bash
O=gpurun_out/r2q; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
AB_SELECT=stencil,no_comm,tree,fft,nearest,all_to_all timeout 900 python scripts/ab_r2.py base slot0 > $O/ab.log 2>&1; echo "ab rc=$?"; tail -23 $O/ab.log

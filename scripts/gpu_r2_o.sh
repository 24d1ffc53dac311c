#!/bin/bash
O=gpurun_out/r2o; mkdir -p $O
AB_SELECT=stencil,no_comm,tree,fft,nearest timeout 900 python scripts/ab_r2.py base stagger > $O/ab.log 2>&1; echo "ab rc=$?"; tail -22 $O/ab.log

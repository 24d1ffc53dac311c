#!/bin/bash
O=gpurun_out/r2j; mkdir -p $O
AB_SELECT=stencil,no_comm,nearest,fft,tree timeout 900 python scripts/ab_r2.py base hoist > $O/ab.log 2>&1; echo "ab rc=$?"; tail -22 $O/ab.log

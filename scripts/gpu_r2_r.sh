#!/bin/bash
O=gpurun_out/r2r; mkdir -p $O
AB_SELECT=stencil,no_comm timeout 900 python scripts/ab_r2.py base xormix > $O/ab.log 2>&1; echo "ab rc=$?"; tail -14 $O/ab.log

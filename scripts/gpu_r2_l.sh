#!/bin/bash
O=gpurun_out/r2l; mkdir -p $O
AB_SELECT=all_to_all timeout 900 python scripts/ab_r2.py base f256 split16 split32 split32f256 split32f1024 > $O/ab.log 2>&1; echo "ab rc=$?"; tail -3 $O/ab.log

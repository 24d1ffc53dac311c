#!/bin/bash
# config-5 tile kernel A/B (same box): L2 promotion of the TMA box loads and
# the 64-wide aligned box (-DTD_ST2D_BOX64 build); parity at 1024^2 each time
for rep in 1 2; do
  for v in base promo0 promo64 promo128 box64 box64_promo128; do
    case $v in
      base) E="";; promo0) E="TD_TMA_PROMO=0";; promo64) E="TD_TMA_PROMO=64";; promo128) E="TD_TMA_PROMO=128";;
      box64) E="TD_LIB=paper_2508_16522_b200/libtdexec_box64.so";;
      box64_promo128) E="TD_LIB=paper_2508_16522_b200/libtdexec_box64.so TD_TMA_PROMO=128";;
    esac
    echo -n "$v $rep "; env $E timeout 120 python tests/tools/bench_stencil2d.py --reps 5 2>&1 | tail -1
  done
done

#!/bin/bash
# config-5: L2 eviction hints on the TMA box loads, streaming stores (same box, parity at 1024^2 each run)
for rep in 1 2; do
  for v in base hint1 hint2 hint3 stcs stcs_hint1; do
    case $v in base) E="";; *) E="TD_LIB=paper_2508_16522_b200/libtdexec_$v.so";; esac
    echo -n "$v $rep "; env $E timeout 120 python tests/tools/bench_stencil2d.py --reps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['replay_ms'],3), round(d['frac'],4), d['parity_1024'])"
  done
done

#!/bin/bash
# launch-path changes (checksum banks, merged D2H copy, no per-launch memsets):
# GPU suite on the bounds-checked and the release build, launch host-time
# profile, e2e probe, short bench
O=gpurun_out/r2e2e; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
TD_LIB=paper_2508_16522_b200/libtdexec_checks.so timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest_checks.log 2>&1; echo "checks rc=$?"; tail -1 $O/pytest_checks.log
timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
python scripts/e2e_probe.py > $O/e2e_probe.log 2>&1; cat $O/e2e_probe.log
TD_LIB=paper_2508_16522_b200/libtdexec_lprof.so python scripts/e2e_probe.py > $O/e2e_probe_lprof.log 2>&1; tail -1 $O/e2e_probe_lprof.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-metg --no-extra --no-cpu > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'], d['e2e']['value'], d['ms_per_step'])"

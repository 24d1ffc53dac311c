#!/bin/bash
# poison code mirrored into host-mapped memory by the kernel (no D2H copy behind a replay)
O=gpurun_out/r2poison; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
TD_LIB=paper_2508_16522_b200/libtdexec_checks.so timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest_checks.log 2>&1; echo "checks rc=$?"; tail -1 $O/pytest_checks.log
timeout 900 python -m pytest tests -q -x -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
python scripts/fixed_cost.py > $O/fixed_cost.json; python -c "import json; d=json.load(open('$O/fixed_cost.json')); print({k: v['flush'] for k, v in d.items()})"
timeout 300 python bench.py --steps 10 --warmup 3 --no-metg --no-extra --no-cpu > $O/bench.json 2> $O/bench.err; python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'], d['e2e']['value'], d['ms_per_step'])"

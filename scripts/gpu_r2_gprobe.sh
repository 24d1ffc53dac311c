O=gpurun_out/r2gp; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
rm -f $O/probe8.log
for lib in paper_2508_16522_b200/libtdexec_probe.so paper_2508_16522_b200/libtdexec_probe_old.so; do
for spec in "tree 4096 1000 1024" "no_comm 1024 1000 512 2 1"; do
  TD_PROBE_LIB=$lib timeout 120 python scripts/group_probe.py $spec >> $O/probe8.log 2>&1
done; done
python -c "
import json
for l in open('$O/probe8.log'):
    d=json.loads(l); print(d['graph'], round(d['plain_ms'],4), {k: round(d[k]['mean']) for k in ('wait','proc','send','tail','gap')}, 'polls', round(d['poll_rounds']['mean'],3))"

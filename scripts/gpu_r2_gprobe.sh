O=gpurun_out/r2gp; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
rm -f $O/probe9.log
for spec in "nearest 8192 100 2048" "nearest 8192 2 2048" "fft 4096 300 1024"; do
  timeout 120 python scripts/group_probe.py $spec >> $O/probe9.log 2>&1
done
python -c "
import json
for l in open('$O/probe9.log'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['graph'], 'plain', round(d['plain_ms']*1e3,1), 'traced', round(d['traced_ms']*1e3,1), 'us; event-minus-kernel', round(d['event_ms_minus_kernel_entry_to_exit_us'],2), 'entry->first pass', round(d['kernel_entry_to_first_pass_us'],2), 'last pass->exit', round(d['last_pass_to_kernel_exit_us'],2), 'span', round(d['global_first_entry_to_last_end_us'],1))"

O=gpurun_out/r2sh; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
echo "--- stats memset"; TD_DEBUG_STATS_MEMSET=1 timeout 120 python scripts/dbg_shards.py 0 0 0 2>&1 | grep -v "shard wait"
echo "--- sleep 200us"; TD_DEBUG_SLEEP_US=200 timeout 120 python scripts/dbg_shards.py 0 0 0 2>&1 | grep -v "shard wait"
echo "--- old lib"; TD_LIB=paper_2508_16522_b200/libtdexec_old.so timeout 120 python scripts/dbg_shards.py 0 0 0 2>&1 | grep -v "shard wait"

O=gpurun_out/r2abw; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
AB_CASES_JSON='[["nearest",8192,100,0,0,2048],["nearest",8192,100,0,0,1024],["nearest",8192,100,0,0,512],["fft",4096,1000,0,0,1024],["fft",4096,1000,0,0,512],["tree",4096,1000,0,0,1024],["tree",4096,1000,0,0,512],["tree",4096,1000,0,0,2048]]' timeout 900 python scripts/ab_r2.py base noplace place > $O/ab.log 2>&1; echo rc=$?; tail -8 $O/ab.log

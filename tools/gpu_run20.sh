python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
grep -q " failed\|rror" gpurun_out/t_all.log && { grep -E "^E |FAILED" gpurun_out/t_all.log | head -20; exit 1; }
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --kernel k2"
$SB --dtype f64 --slabs 8 --tag 8slabs-default

python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
grep -q " failed\|rror" gpurun_out/t_all.log && { grep -E "^E |FAILED" gpurun_out/t_all.log | head -20; exit 1; }
LBM_OVERLAP=0 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "local_slabs" 2>&1 | tail -1
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --kernel k2"
$SB --dtype f64 --tag 1slab
$SB --dtype f64 --slabs 8 --tag 8slabs-overlap
LBM_OVERLAP=0 $SB --dtype f64 --slabs 8 --tag 8slabs-serial
$SB --dtype f64 --bc periodic --tag periodic-1slab-overlap
LBM_OVERLAP=0 $SB --dtype f64 --bc periodic --tag periodic-1slab-serial

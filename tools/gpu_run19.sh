python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "local_slabs or kernel_choice or k2_equals" 2>&1 | tail -1
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --kernel k2"
$SB --dtype f64 --slabs 8 --tag 8slabs-overlap
LBM_OVERLAP=0 $SB --dtype f64 --slabs 8 --tag 8slabs-serial
$SB --dtype f64 --slabs 4 --tag 4slabs-overlap
LBM_OVERLAP=0 $SB --dtype f64 --slabs 4 --tag 4slabs-serial

python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
LBM_K2_WS=1 timeout 60 python -m pytest tests/test_gpu_parity.py -q -x -k "k2_equals_k1 and dims1" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "variants" 2>&1 | tail -2
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --kernel k2"
$SB --dtype f64 --tag k2
LBM_K2_WS=1 $SB --dtype f64 --tag k2w
LBM_K2_WS=1 LBM_K2_TILE=16x16 $SB --dtype f64 --tag k2w-16x16
LBM_K2_WS=1 LBM_K2_TILE=8x32 $SB --dtype f32 --tag k2w-8x32
LBM_K2_WS=1 LBM_K2_TILE=16x16 $SB --dtype f32 --tag k2w-16x16

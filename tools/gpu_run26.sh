python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --dtype f64 --kernel k2"
LBM_ZOFF=32 LBM_PALIGN=32 $SB --tag z32
LBM_ZOFF=32 LBM_PALIGN=32 LBM_NOFRAMES=1 $SB --tag z32-noframes
LBM_ZOFF=0 LBM_PALIGN=32 LBM_NOFRAMES=1 $SB --tag z0-noframes
LBM_ZOFF=0 LBM_PALIGN=32 $SB --tag z0-frames-corrupt

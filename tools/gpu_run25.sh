python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --dtype f64"
LBM_ZOFF=0 LBM_PALIGN=32 $SB --kernel k1 --tag k1-z0
LBM_ZOFF=0 LBM_PALIGN=32 LBM_PITCH_PAD=32 $SB --kernel k1 --tag k1-z0-pad32
LBM_ZOFF=0 LBM_PALIGN=32 LBM_PITCH_PAD=4 $SB --kernel k1 --tag k1-z0-pad4
LBM_ZOFF=32 LBM_PALIGN=32 $SB --kernel k1 --tag k1-z32
LBM_ZOFF=32 LBM_PALIGN=32 LBM_PITCH_PAD=-8 $SB --kernel k1 --tag k1-z32-pitch512
LBM_ZOFF=0 LBM_PALIGN=32 $SB --kernel k1 --bc periodic --tag k1-z0-per
LBM_ZOFF=32 LBM_PALIGN=32 LBM_PITCH_PAD=-8 $SB --kernel k2 --bc periodic --tag k2-z32-pitch512-per
LBM_ZOFF=32 LBM_PALIGN=32 $SB --kernel k2 --bc periodic --tag k2-z32-per
LBM_ZOFF=0 LBM_PALIGN=32 $SB --kernel k2 --bc periodic --tag k2-z0-per

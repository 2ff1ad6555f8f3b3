python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SB="timeout 120 python tools/sweep_bench.py --dims 256,512,512 --steps 40 --reps 3"
for ch in 0 8 16 32 64 128; do
LBM_K2_CHUNK=$ch $SB --dtype f64 --kernel k2tma --tag tma-ch$ch
LBM_K2_CHUNK=$ch LBM_K2_EARLY=1 $SB --dtype f64 --kernel k2tma --tag tma-early-ch$ch
done
for ch in 0 16 32; do
LBM_K2_CHUNK=$ch $SB --dtype f32 --kernel k2tma --tag tma-ch$ch
LBM_K2_CHUNK=$ch LBM_K2_EARLY=1 $SB --dtype f32 --kernel k2tma --tag tma-early-ch$ch
LBM_K2_CHUNK=$ch $SB --dtype f64 --kernel k2 --tag k2r-ch$ch
done

python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
export LBM_K2_EARLY=1
for dt in f64 f32; do
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --dtype $dt --kernel k2tma"
for ch in 16 24 32 40 48 64 96; do LBM_K2_CHUNK=$ch $SB --tag early-ch$ch; done
done
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --kernel k2tma"
LBM_K2_TILE=16x16 LBM_K2_CHUNK=32 $SB --dtype f64 --tag early16x16-ch32
LBM_K2_TILE=8x32 LBM_K2_CHUNK=32 $SB --dtype f32 --tag early8x32-ch32
LBM_K2_EARLY=0 LBM_K2_CHUNK=32 $SB --dtype f32 --tag late-ch32
LBM_K2_EARLY=0 LBM_K2_CHUNK=32 $SB --dtype f64 --tag late-ch32

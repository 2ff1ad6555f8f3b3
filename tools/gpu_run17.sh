python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 100 --reps 4 --power"
$SB --dtype f64 --kernel k2 --tag k2-sust
$SB --dtype f64 --kernel k1 --tag k1-sust
$SB --dtype f32 --kernel k2 --tag k2-sust
$SB --dtype f32 --kernel k1 --tag k1-sust
LBM_K2_TILE=16x16 $SB --dtype f64 --kernel k2 --tag k2-16x16-sust

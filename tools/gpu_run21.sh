python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --kernel k2"
$SB --dtype f64 --tag fix
LBM_K2_NOFIX=1 $SB --dtype f64 --tag nofix
$SB --dtype f32 --tag fix
LBM_K2_NOFIX=1 $SB --dtype f32 --tag nofix
$SB --dtype f64 --bc periodic --tag fix-per
LBM_K2_NOFIX=1 $SB --dtype f64 --bc periodic --tag nofix-per

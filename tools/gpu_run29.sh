python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
LBM_PER_REG=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "k2_equals_k1" 2>&1 | tail -1
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --bc periodic --kernel k2"
$SB --dtype f64 --tag per-fixup
LBM_PER_REG=1 $SB --dtype f64 --tag per-reg
$SB --dtype f32 --tag per-fixup
LBM_PER_REG=1 $SB --dtype f32 --tag per-reg
SB="timeout 300 python tools/sweep_bench.py --dims 256,256,256 --steps 20 --reps 2 --bc periodic --kernel k2"
$SB --dtype f64 --tag cfg3-fixup
LBM_PER_REG=1 $SB --dtype f64 --tag cfg3-reg

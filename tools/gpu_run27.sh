python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "k2_equals_k1 and dims1" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
grep -q " failed\|rror" gpurun_out/t_all.log && { grep -E "^E |FAILED|Error" gpurun_out/t_all.log | head -20; exit 1; }
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2"
$SB --dtype f64 --kernel k2 --tag k2
$SB --dtype f32 --kernel k2 --tag k2
$SB --dtype f64 --kernel k2 --bc periodic --tag k2-per

python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "k2_equals_k1 or variants or config" > gpurun_out/t_k2.log 2>&1; tail -1 gpurun_out/t_k2.log
grep -q " failed\|rror" gpurun_out/t_k2.log && { grep -E "^E |FAILED|Error" gpurun_out/t_k2.log | head -20; exit 1; }
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --kernel k2"
$SB --dtype f64 --tag rowmap
$SB --dtype f32 --tag rowmap
$SB --dtype f64 --bc periodic --tag rowmap-per

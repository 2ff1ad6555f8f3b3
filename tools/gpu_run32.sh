python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "aa_" > gpurun_out/t_aa.log 2>&1; tail -2 gpurun_out/t_aa.log
grep -q " failed\|rror" gpurun_out/t_aa.log && { grep -E "^E |FAILED|Error" gpurun_out/t_aa.log | head -20; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2"
$SB --dtype f64 --kernel aa --tag aa
$SB --dtype f32 --kernel aa --tag aa
$SB --dtype f64 --kernel k1 --tag k1
$SB --dtype f64 --kernel aa --dims 2048,512,512 --tag aa-2048

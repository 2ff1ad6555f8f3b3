python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "k2_equals_k1 or variants or local_slabs or kernel_choice" > gpurun_out/t_k2.log 2>&1; tail -2 gpurun_out/t_k2.log
grep -q " failed\|rror" gpurun_out/t_k2.log && exit 1
SB="timeout 120 python tools/sweep_bench.py --dims 256,512,512 --steps 40 --reps 3"
for dt in f64 f32; do
$SB --dtype $dt --kernel k2tma --tag tma
LBM_K2_EARLY=1 $SB --dtype $dt --kernel k2tma --tag tma-early
LBM_K2_TILE=16x16 $SB --dtype $dt --kernel k2tma --tag tma16x16
LBM_K2_TILE=16x16 LBM_K2_EARLY=1 $SB --dtype $dt --kernel k2tma --tag tma16x16-early
LBM_K2_TILE=8x16 $SB --dtype $dt --kernel k2tma --tag tma8x16
done

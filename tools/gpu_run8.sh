python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "k2_equals_k1 or local_slabs or kernel_choice" > gpurun_out/t_k2.log 2>&1; tail -2 gpurun_out/t_k2.log
grep -q " passed" gpurun_out/t_k2.log || exit 1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
show() { python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print('$1', d.get('value'), d.get('roofline',{}).get('frac'), d.get('clocks',{}).get('sm_mhz'))"; }
timeout 600 $B --kernel k2tma 2>&1 | show "f64 tma 8x32"
timeout 600 $B --kernel k2tma --dtype f32 2>&1 | show "f32 tma 16x32"
LBM_K2_TILE=8x16 timeout 600 $B --kernel k2tma 2>&1 | show "f64 tma 8x16"
LBM_K2_TILE=16x16 timeout 600 $B --kernel k2tma 2>&1 | show "f64 tma 16x16"
LBM_K2_TILE=8x32 timeout 600 $B --kernel k2tma --dtype f32 2>&1 | show "f32 tma 8x32"
CMD="python bench.py --config 4 --dims 64,512,512 --steps 1 --warmup 0 --lbm-steps 4 --no-cpu-baseline --no-e2e --kernel k2tma"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_sweep -s 1 -c 1 -o gpurun_out/prof_k2t_c $CMD > gpurun_out/ncu_k2t.log 2>&1
tail -1 gpurun_out/ncu_k2t.log

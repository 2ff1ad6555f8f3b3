python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 60 python -m pytest tests/test_gpu_parity.py -x -q -k "k2_equals_k1 and dims1" > gpurun_out/t_k2a.log 2>&1; tail -3 gpurun_out/t_k2a.log; grep -q " passed" gpurun_out/t_k2a.log || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "k2_equals_k1" > gpurun_out/t_k2.log 2>&1; tail -3 gpurun_out/t_k2.log
grep -q " passed" gpurun_out/t_k2.log || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k2r_shapes or local_slabs or kernel_choice" > gpurun_out/t_k2b.log 2>&1; tail -3 gpurun_out/t_k2b.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
show() { python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print('$1', d.get('value'), d.get('roofline',{}).get('frac'), d.get('clocks',{}).get('sm_mhz'))"; }
for cfg in 8x32s0 8x32s1; do
  LBM_K2R_CFG=$cfg timeout 600 $B 2>&1 | show "f64 $cfg"
  LBM_K2R_CFG=$cfg timeout 600 $B --dtype f32 2>&1 | show "f32 $cfg"
done
CMD="python bench.py --config 4 --dims 64,512,512 --steps 1 --warmup 0 --lbm-steps 4 --no-cpu-baseline --no-e2e"
export LBM_K2R_CFG=8x32s1
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2r_sweep -s 1 -c 1 -o gpurun_out/prof_k2r_b $CMD > gpurun_out/ncu_k2r.log 2>&1
tail -1 gpurun_out/ncu_k2r.log

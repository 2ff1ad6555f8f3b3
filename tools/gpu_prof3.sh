python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
CMD="python bench.py --config 4 --dims 64,512,512 --steps 1 --warmup 0 --lbm-steps 4 --no-cpu-baseline --no-e2e"
export LBM_K2R_CFG=8x32s0
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2r_sweep -s 1 -c 1 -o gpurun_out/prof_k2r_a $CMD > gpurun_out/ncu_k2r.log 2>&1
tail -3 gpurun_out/ncu_k2r.log

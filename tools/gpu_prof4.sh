python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
CMD="python tools/sweep_bench.py --dims 64,512,512 --steps 2 --reps 1 --kernel k2tma"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_sweep -s 2 -c 1 -o gpurun_out/prof_k2t_e0 $CMD > gpurun_out/ncu_e0.log 2>&1
export LBM_K2_EARLY=1
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_sweep -s 2 -c 1 -o gpurun_out/prof_k2t_e1 $CMD > gpurun_out/ncu_e1.log 2>&1
tail -1 gpurun_out/ncu_e0.log gpurun_out/ncu_e1.log

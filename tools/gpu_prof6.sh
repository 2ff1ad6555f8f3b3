python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
CMD="python tools/sweep_bench.py --dims 128,512,512 --steps 2 --reps 1 --kernel k2"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_sweep -s 2 -c 1 -o gpurun_out/prof_k2_f64_v3 $CMD > gpurun_out/ncu_v3.log 2>&1
$CMD --dtype f32 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_sweep -s 2 -c 1 -o gpurun_out/prof_k2_f32_v3 $CMD --dtype f32 > gpurun_out/ncu_v3f.log 2>&1
tail -n 1 gpurun_out/ncu_v3.log gpurun_out/ncu_v3f.log

set -x
CMD="python bench.py --config 4 --dims 64,512,512 --steps 1 --warmup 0 --lbm-steps 4 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_sweep -s 1 -c 1 -o gpurun_out/prof_k2_r1 $CMD > gpurun_out/ncu_k2.log 2>&1
$CMD --kernel k1 > gpurun_out/prof_plain_k1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_step -s 2 -c 1 -o gpurun_out/prof_k1_r1 $CMD --kernel k1 > gpurun_out/ncu_k1.log 2>&1
tail -3 gpurun_out/ncu_k2.log gpurun_out/ncu_k1.log
ls -la gpurun_out/

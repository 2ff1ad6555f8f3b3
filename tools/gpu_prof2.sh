set -x
CMD="python bench.py --config 4 --dims 64,512,512 --steps 1 --warmup 0 --lbm-steps 4 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_sweep -s 1 -c 1 -o gpurun_out/prof_k2_r1b $CMD > gpurun_out/ncu_k2.log 2>&1
$CMD --dtype f32 > gpurun_out/prof_plain32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_sweep -s 1 -c 1 -o gpurun_out/prof_k2f32_r1b $CMD --dtype f32 > gpurun_out/ncu_k2f32.log 2>&1
BCMD="python bench.py --steps 3 --warmup 3"
$BCMD > gpurun_out/bench_launchlist_plain.json 2>gpurun_out/bench_launchlist_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $BCMD > gpurun_out/ncu_launches.log 2>&1
ls -la gpurun_out

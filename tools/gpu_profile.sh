# ncu evidence for profiles/ (run under gpurun): one config-5 sweep launch of K2 (fp64, fp32) and K1
# under ncu --set full, and the launch list of the default bench command.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for dt in f64 f32; do
  CMD="python tools/sweep_bench.py --dims 1024,512,512 --steps 2 --reps 1 --kernel k2 --dtype $dt"
  $CMD > gpurun_out/plain_$dt.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k2_sweep -s 2 -c 1 -o gpurun_out/r01_k2_${dt}_cfg5 $CMD > gpurun_out/ncu_k2_$dt.log 2>&1
done
CMD="python tools/sweep_bench.py --dims 1024,512,512 --steps 2 --reps 1 --kernel k2sc --dtype f64"
$CMD > gpurun_out/plain_k2sc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_sweep -s 2 -c 1 -o gpurun_out/r01_k2sc_f64_cfg5 $CMD > gpurun_out/ncu_k2sc.log 2>&1
CMD="python tools/sweep_bench.py --dims 1024,512,512 --steps 2 --reps 1 --kernel k1 --dtype f64"
$CMD > gpurun_out/plain_k1.log 2>&1 && \
ncu --set full --clock-control none -k regex:k1_step -s 4 -c 1 -o gpurun_out/r01_k1_f64_cfg5 $CMD > gpurun_out/ncu_k1.log 2>&1
BCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$BCMD > gpurun_out/bench_ll_plain.json 2> gpurun_out/bench_ll_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_bench_f64.csv $BCMD > gpurun_out/ncu_ll.log 2>&1
ls -la gpurun_out | tail -12

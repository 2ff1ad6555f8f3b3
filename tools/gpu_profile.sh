# ncu evidence for profiles/ (run under gpurun; one GPU): one sweep launch per kernel/workload under
# ncu --set full, summarised ON the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back),
# plus the launch list of the default bench command.  Round-2 second pass: R=r02b.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
R=${R:-r02b}
cap() {  # cap <name> <kernel regex> <skip> <sweep_bench args...>
  local name=$1 kre=$2 skip=$3; shift 3
  local CMD="python tools/sweep_bench.py --steps 2 --reps 1 $*"
  $CMD > gpurun_out/plain_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o /tmp/${R}_$name $CMD \
    > gpurun_out/ncu_$name.log 2>&1
  python tools/ncu_summary.py rep /tmp/${R}_$name.ncu-rep "${R}_$name: $*" > gpurun_out/${R}_$name.txt 2>&1
  ncu -i /tmp/${R}_$name.ncu-rep --page raw --csv > gpurun_out/${R}_$name.raw.csv 2>/dev/null
  ncu -i /tmp/${R}_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${R}_$name.src.csv 2>/dev/null
}
for dt in f64 f32; do
  cap k2_${dt}_cfg5 k2_sweep 2 --dims 1024,512,512 --kernel k2 --dtype $dt
  cap k2_${dt}_cfg3 k2_sweep 2 --dims 256,256,256 --bc periodic --kernel k2 --dtype $dt
done
cp /tmp/${R}_k2_f64_cfg5.ncu-rep gpurun_out/
BCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$BCMD > gpurun_out/bench_ll_plain.json 2> gpurun_out/bench_ll_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_bench_f64.csv $BCMD > gpurun_out/ncu_ll.log 2>&1
du -sh gpurun_out

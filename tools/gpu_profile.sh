# ncu evidence for profiles/ (run under gpurun; one GPU): one sweep launch per
# kernel/workload under ncu --set full, and the launch list of the default
# bench command.  Summaries: python tools/ncu_summary.py rep gpurun_out/<name>.ncu-rep
# (round 2 captures: profiles/r02_*).
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
R=${R:-r02}
cap() {  # cap <name> <kernel regex> <skip> <sweep_bench args...>
  local name=$1 kre=$2 skip=$3; shift 3
  local CMD="python tools/sweep_bench.py --steps 2 --reps 1 $*"
  $CMD > gpurun_out/plain_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o gpurun_out/${R}_$name $CMD \
    > gpurun_out/ncu_$name.log 2>&1
}
for dt in f64 f32; do
  cap k2_${dt}_cfg5 k2_sweep 2 --dims 1024,512,512 --kernel k2 --dtype $dt
  cap k2_${dt}_cfg3 k2_sweep 2 --dims 256,256,256 --bc periodic --kernel k2 --dtype $dt
done
LBM_K2_TILE=8x32 cap k2_f32_cfg5_8x32 k2_sweep 2 --dims 1024,512,512 --kernel k2 --dtype f32
cap k3_f32_cfg3 k3_sweep 1 --dims 256,256,256 --bc periodic --kernel k3 --dtype f32 --steps 3
cap dqq27_f64_cfg4 k_dqq_step 3 --dims 512,512,512 --kernel k1 --dtype f64 --lattice 27
BCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$BCMD > gpurun_out/bench_ll_plain.json 2> gpurun_out/bench_ll_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_bench_f64.csv $BCMD > gpurun_out/ncu_ll.log 2>&1
ls -la gpurun_out | tail -12

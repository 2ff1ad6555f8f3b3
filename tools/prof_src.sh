# Source-level (SASS) stall attribution of one K2 sweep launch (run under gpurun; one GPU).
# usage: bash tools/prof_src.sh <name> <sweep_bench args...>
# -> gpurun_out/<name>.ncu-rep; read here with
#    ncu -i gpurun_out/<name>.ncu-rep --page source --csv --print-source sass > x.csv; python tools/sass_hist.py x.csv 40
name=$1; shift
CMD="python tools/sweep_bench.py --steps 2 --reps 1 $*"
$CMD > gpurun_out/plain_$name.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KRE:-k2_sweep} -s ${SKIP:-2} -c 1 -o gpurun_out/$name $CMD \
  > gpurun_out/ncu_$name.log 2>&1
tail -2 gpurun_out/ncu_$name.log

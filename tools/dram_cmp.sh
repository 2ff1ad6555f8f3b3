# DRAM bytes + duration of one K2 launch per variant (run under gpurun; one GPU):
#   ENVS="LBM_K2_ZBLOCK=255 LBM_K2_ZBLOCK=8" bash tools/dram_cmp.sh <tag> <sweep_bench args...>
tag=$1; shift
for e in $ENVS; do
  env $e ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:${KRE:-k2_sweep} -s 2 -c 1 --csv python tools/sweep_bench.py --steps 2 --reps 1 "$@" 2>/dev/null \
    | grep -E '"(dram__bytes|gpu__time)' | awk -F'","' -v e="$e" -v t="$tag" '{printf "%s %s %s %s %s\n", t, e, $(NF-2), $(NF-1), $NF}' | tr -d '"'
done

# A/B of a variant build against the in-tree library (run under gpurun; one GPU):
#   bash tools/ab_run.sh <variant>      (exp/<variant> from tools/build_variant.sh)
# bitwise gate, interleaved sustained sweeps (config 5 f64/f32, config 3 f64/f32),
# smem bank conflicts + DRAM bytes of one K2 launch, interleaved bench.py K2 frac.
v=$1
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
LBM_PKG_ROOT=exp/$v timeout 300 python tools/ab_bitwise.py || exit 1
for rep in 1 2; do
  for root in . exp/$v; do
    for dt in f64 f32; do
      LBM_PKG_ROOT=$root timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 400 --reps 3 --power --dtype $dt --tag "cfg5 $root"
      LBM_PKG_ROOT=$root timeout 300 python tools/sweep_bench.py --dims 256,256,256 --bc periodic --steps 400 --reps 3 --power --dtype $dt --tag "cfg3 $root"
    done
  done
done
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum
for root in . exp/$v; do
  for dt in f64 f32; do
    LBM_PKG_ROOT=$root ncu --metrics $M --clock-control none -k regex:k2_sweep -s 2 -c 1 --csv \
      python tools/sweep_bench.py --steps 2 --reps 1 --dims 1024,512,512 --dtype $dt 2>/dev/null \
      | grep -E '"(l1tex|dram|gpu__time|smsp)' | awk -F'","' -v t="$root $dt" '{printf "%s %s %s %s\n", t, $(NF-2), $(NF-1), $NF}' | tr -d '"'
  done
done
for rep in 1 2; do
  for root in . exp/$v; do
    LBM_PKG_ROOT=$root timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_bench.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_bench.json')); print('bench', sys.argv[1], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])" "$root"
  done
done

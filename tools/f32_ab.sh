# fp32 K2 A/B of variant builds (run under gpurun; one GPU): bitwise gate, smem conflicts and
# instructions of one config-5 launch, interleaved sweeps (config 5, config 3) and bench --dtype f32.
for v in "$@"; do LBM_PKG_ROOT=exp/$v timeout 600 python tools/ab_bitwise.py | grep -c bitwise || exit 1; done
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,gpu__time_duration.sum,smsp__inst_executed.sum
for root in . $(for v in "$@"; do echo exp/$v; done); do
  LBM_PKG_ROOT=$root ncu --metrics $M --clock-control none -k regex:k2_sweep -s 2 -c 1 --csv \
    python tools/sweep_bench.py --steps 2 --reps 1 --dims 1024,512,512 --dtype f32 2>/dev/null \
    | grep -E '"(l1tex|gpu__time|smsp)' | awk -F'","' -v t="$root" '{printf "%s %s %s\n", t, $(NF-2), $NF}' | tr -d '"'
done
for rep in 1 2; do for root in . $(for v in "$@"; do echo exp/$v; done); do
  LBM_PKG_ROOT=$root timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 40 --reps 3 --dtype f32 --tag "cfg5 $root"
  LBM_PKG_ROOT=$root timeout 300 python tools/sweep_bench.py --dims 256,256,256 --bc periodic --steps 100 --reps 3 --dtype f32 --tag "cfg3 $root"
  LBM_PKG_ROOT=$root timeout 900 python bench.py --dtype f32 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f32_bench.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/f32_bench.json')); print('bench f32', sys.argv[1], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])" $root
done; done

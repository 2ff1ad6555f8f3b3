# GPU tests + ncu evidence for the D3Q15/D3Q27 two-step sweep (run under gpurun; one GPU):
# full GPU suite, then one K2Q launch per lattice/dtype under ncu --set full (summarised on the
# box), and the one-step kernel of D3Q27 fp64 (AUTO's choice there).  R names the round.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
grep -E "^E |FAILED" gpurun_out/t_all.log | head -20
R=${R:-r02c}
cap() {  # cap <name> <kernel regex> <sweep_bench args...>
  local name=$1 kre=$2; shift 2
  local CMD="python tools/sweep_bench.py --steps 4 --reps 1 $*"
  $CMD > gpurun_out/plain_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -o /tmp/${R}_$name $CMD \
    > gpurun_out/ncu_$name.log 2>&1
  python tools/ncu_summary.py rep /tmp/${R}_$name.ncu-rep "${R}_$name: $*" > gpurun_out/${R}_$name.txt 2>&1
}
cap k2q15_f64_cfg4 k_dqq_k2 --dims 512,512,512 --lattice 15 --kernel k2 --dtype f64
cap k2q27_f32_cfg4 k_dqq_k2 --dims 512,512,512 --lattice 27 --kernel k2 --dtype f32
cap k2q27_f64_cfg4 k_dqq_k2 --dims 512,512,512 --lattice 27 --kernel k2 --dtype f64
for q in 15 27; do for dt in f64 f32; do for k in k1 k2; do
  timeout 300 python tools/sweep_bench.py --dims 512,512,512 --lattice $q --steps 200 --reps 3 --power --dtype $dt --kernel $k --tag "q$q $k sustained"
done; done; done

# ncu --set full of the final K2Q sweeps (run under gpurun; one GPU), summarised on the box.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
R=${R:-r02c}
for spec in "k2q27_f32_cfg4:27:f32" "k2q15_f32_cfg4:15:f32" "k2q15_f64_cfg4:15:f64"; do
  IFS=: read name q dt <<< "$spec"
  CMD="python tools/sweep_bench.py --steps 4 --reps 1 --dims 512,512,512 --lattice $q --kernel k2 --dtype $dt"
  $CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_dqq_k2 -s 1 -c 1 -o /tmp/${R}_$name $CMD > gpurun_out/ncu_$name.log 2>&1
  python tools/ncu_summary.py rep /tmp/${R}_$name.ncu-rep "${R}_$name: --dims 512,512,512 --lattice $q --kernel k2 --dtype $dt (final K2Q)" > gpurun_out/${R}_$name.txt 2>&1
  head -12 gpurun_out/${R}_$name.txt | tail -8
done

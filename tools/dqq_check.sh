# D3Q15/D3Q27 two-step sweep (K2Q) check (run under gpurun; one GPU): its GPU tests,
# then sweep MLUPS of K1 (one step per pass) vs K2 on the 512^3 cavity, both dtypes.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_dqq.py -q -x > gpurun_out/t_dqq.log 2>&1; tail -3 gpurun_out/t_dqq.log
grep -E "^E |FAILED|Error" gpurun_out/t_dqq.log | head -20
for q in 27 15; do
  for dt in f64 f32; do
    for k in k1 k2; do
      timeout 300 python tools/sweep_bench.py --dims 512,512,512 --lattice $q --steps 20 --reps 3 --dtype $dt --kernel $k --tag "q$q $k"
    done
  done
done
timeout 300 python tools/sweep_bench.py --dims 256,256,256 --bc periodic --lattice 27 --steps 20 --reps 3 --dtype f64 --kernel k2 --tag "q27 k2 per"

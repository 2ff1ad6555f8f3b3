# D3Q15/D3Q27 final check (run under gpurun; one GPU): GPU tests of the lattices, sweeps, ncu of D3Q27 fp64 K2Q.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_dqq.py -q -x > gpurun_out/t_dqq.log 2>&1; tail -2 gpurun_out/t_dqq.log
grep -E "^E |FAILED" gpurun_out/t_dqq.log | head
for q in 27 15; do for dt in f64 f32; do for k in k1 k2; do
  timeout 300 python tools/sweep_bench.py --dims 512,512,512 --lattice $q --steps 20 --reps 3 --dtype $dt --kernel $k --tag "q$q $k"
done; done; done
timeout 300 python tools/sweep_bench.py --dims 256,256,256 --bc periodic --lattice 27 --steps 20 --reps 3 --dtype f64 --kernel k2 --tag "q27 k2 per"
timeout 300 python tools/sweep_bench.py --dims 512,512,512 --lattice 27 --steps 200 --reps 3 --power --dtype f64 --kernel k2 --tag "q27 k2 sustained"
CMD="python tools/sweep_bench.py --steps 4 --reps 1 --dims 512,512,512 --lattice 27 --kernel k2 --dtype f64"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_dqq_k2 -s 1 -c 1 -o /tmp/r02c_k2q27ws_f64_cfg4 $CMD > gpurun_out/ncu_ws.log 2>&1
python tools/ncu_summary.py rep /tmp/r02c_k2q27ws_f64_cfg4.ncu-rep "r02c_k2q27ws_f64_cfg4: --dims 512,512,512 --lattice 27 --kernel k2 --dtype f64 (warp-specialised)" > gpurun_out/r02c_k2q27ws_f64_cfg4.txt 2>&1

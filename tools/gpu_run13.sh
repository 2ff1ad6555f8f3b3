python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
grep -q " failed\|rror" gpurun_out/t_all.log && exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err; echo rc=$?
cat gpurun_out/bench_r1d.json
timeout 900 python bench.py --steps 3 --warmup 3 --dtype f32 --no-cpu-baseline > gpurun_out/bench_r1d_f32.json 2> gpurun_out/bench_r1d_f32.err; echo rc=$?
cat gpurun_out/bench_r1d_f32.json

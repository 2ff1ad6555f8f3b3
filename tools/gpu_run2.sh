set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; echo rc=$?
cat gpurun_out/bench_r1c.json; tail -5 gpurun_out/bench_r1c.err
timeout 900 python bench.py --steps 3 --warmup 3 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/bench_r1c_f32.json 2>&1; cat gpurun_out/bench_r1c_f32.json
timeout 900 python bench.py --steps 3 --warmup 3 --config 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_r1c_c4.json 2>&1; cat gpurun_out/bench_r1c_c4.json
timeout 900 python bench.py --steps 3 --warmup 3 --config 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r1c_c3.json 2>&1; cat gpurun_out/bench_r1c_c3.json

set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; echo rc=$?
cat gpurun_out/bench_r1c.json; tail -5 gpurun_out/bench_r1c.err
timeout 900 python bench.py --steps 3 --warmup 3 --dtype f32 --no-cpu-baseline > gpurun_out/bench_r1c_f32.json 2> gpurun_out/bench_r1c_f32.err; echo rc=$?
cat gpurun_out/bench_r1c_f32.json

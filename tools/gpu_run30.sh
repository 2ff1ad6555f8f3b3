python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
grep -q " failed\|rror" gpurun_out/t_all.log && { grep -E "^E |FAILED|Error" gpurun_out/t_all.log | head -20; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r1e.json')); print('bench f64', d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
timeout 900 python bench.py --steps 3 --warmup 3 --dtype f32 --no-cpu-baseline > gpurun_out/bench_r1e_f32.json 2> gpurun_out/bench_r1e_f32.err
python -c "import json; d=json.load(open('gpurun_out/bench_r1e_f32.json')); print('bench f32', d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"

# Standard GPU check (run under gpurun): build, all GPU tests, sweep micro-bench; "bench" adds a bench.py line.
# standard GPU check: build, all GPU tests, sweep micro-bench, sustained bench (no CPU leg)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
grep -q " failed\|rror" gpurun_out/t_all.log && { grep -E "^E |FAILED" gpurun_out/t_all.log | head -20; exit 1; }
for dt in f64 f32; do
  timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --dtype $dt --kernel k2 --tag k2
done
timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --dtype f64 --kernel k1 --tag k1
if [ "$1" = "bench" ]; then
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_chk.json 2>gpurun_out/bench_chk.err
  python -c "import json; d=json.load(open('gpurun_out/bench_chk.json')); print('bench f64', d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
fi

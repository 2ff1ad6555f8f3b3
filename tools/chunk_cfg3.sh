# Config 3 (256^3 periodic) x-chunk length under the sustained bench (run under gpurun; one GPU):
# bench.py --config 3 K2 frac per LBM_K2_CHUNK value, both dtypes, interleaved twice.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for rep in 1 2; do
  for dt in f64 f32; do
    for ch in ${CHUNKS:-0 43 52 64}; do
      LBM_K2_CHUNK=$ch timeout 600 python bench.py --config 3 --dtype $dt --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
        > gpurun_out/ch_bench.json 2>/dev/null
      python -c "import json,sys; d=json.load(open('gpurun_out/ch_bench.json')); print('cfg3', sys.argv[1], 'chunk', sys.argv[2], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])" $dt $ch
    done
  done
done

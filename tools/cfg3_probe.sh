# Config 3 f32 probes (run under gpurun; one GPU): bench K2 frac per short chunk length,
# and sweep-only MLUPS of 256^3 periodic vs cavity and of a longer periodic box.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for dt in f32 f64; do
  for ch in 0 24 28 36 40; do
    LBM_K2_CHUNK=$ch timeout 600 python bench.py --config 3 --dtype $dt --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/ch_bench.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ch_bench.json')); print('cfg3', sys.argv[1], 'chunk', sys.argv[2], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])" $dt $ch
  done
done
for bc in periodic cavity; do
  for dims in 256,256,256 1024,256,256 256,512,512; do
    timeout 300 python tools/sweep_bench.py --dims $dims --bc $bc --steps 200 --reps 3 --dtype f32 --tag "$bc $dims"
  done
done
for t in 8x32 16x16; do
  LBM_K2_TILE=$t timeout 300 python tools/sweep_bench.py --dims 256,256,256 --bc periodic --steps 200 --reps 3 --dtype f32 --tag "tile $t"
done

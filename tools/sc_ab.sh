# A/B of single-copy K2_SC chunk caps (run under gpurun; one GPU): bitwise K2_SC == K1 of each
# variant, then interleaved bench.py --kernel k2sc lines (config 5 fp64).
for v in "$@"; do AB_KERNELS=1,5 LBM_PKG_ROOT=exp/$v timeout 600 python tools/ab_bitwise.py | grep -c bitwise || exit 1; done
for rep in 1 2; do for root in . $(for v in "$@"; do echo exp/$v; done); do
  LBM_PKG_ROOT=$root timeout 900 python bench.py --kernel k2sc --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sc_bench.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/sc_bench.json')); print('k2sc', sys.argv[1], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])" $root
done; done

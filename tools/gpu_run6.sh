set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "k2_equals_k1 and 5-17-31" 2>&1 | tail -5 || exit 1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
show() { python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print('$1', d.get('value'), d.get('roofline',{}).get('frac'), d.get('clocks',{}).get('sm_mhz'))"; }
for cfg in 8x32s1 8x32s0 8x16s1 4x32s1; do
  LBM_K2R_CFG=$cfg timeout 600 $B 2>&1 | show "f64 $cfg"
  LBM_K2R_CFG=$cfg timeout 600 $B --dtype f32 2>&1 | show "f32 $cfg"
done
timeout 600 $B --kernel k2tma 2>&1 | show "f64 tma"

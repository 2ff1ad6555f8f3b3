python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for t in 8x32 8x16 16x16; do
  LBM_K2_TILE=$t timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print('f64 $t', d.get('value'), d.get('roofline',{}).get('achieved'), d.get('clocks'))"
done
for t in 16x32 8x32 8x16 16x16; do
  LBM_K2_TILE=$t timeout 900 python bench.py --steps 3 --warmup 3 --dtype f32 --no-cpu-baseline --no-e2e 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print('f32 $t', d.get('value'), d.get('roofline',{}).get('achieved'), d.get('clocks'))"
done
for t in 8x16 16x16; do LBM_K2_TILE=$t timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "k2 or config" 2>&1 | tail -1; done

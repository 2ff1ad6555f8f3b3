python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for args in "" "--dtype f32"; do
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $args 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print('$args', d.get('value'), d.get('roofline',{}).get('achieved'), d.get('clocks'))"
done
for t in 16x16 8x16; do
  LBM_K2_TILE=$t timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print('f64 $t', d.get('value'), d.get('roofline',{}).get('achieved'))"
done

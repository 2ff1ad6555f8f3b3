python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for args in "" "--kernel k1" "--dtype f32" "--dtype f32 --kernel k1"; do
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $args 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]); print('$args', d['value'], d['roofline']['achieved'], d['roofline']['kernel'], d['clocks'])"
done

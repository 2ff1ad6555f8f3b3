python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
show() { python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; r=d.get('roofline',{}); print('$1', d.get('value'), r.get('achieved'), r.get('frac'), r.get('frac_mlups_x_single_step_bytes'), (d.get('e2e') or {}).get('value'), r.get('traffic'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))"; }
B="timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$B --config 3 2>&1 | show "cfg3-f64"
$B --config 3 --dtype f32 2>&1 | show "cfg3-f32"
$B --config 4 2>&1 | show "cfg4-f64"
$B --config 4 --dtype f32 2>&1 | show "cfg4-f32"
$B --kernel k1 2>&1 | show "cfg5-f64-k1"
$B --kernel k1 --dtype f32 2>&1 | show "cfg5-f32-k1"
$B 2>&1 | show "cfg5-f64"
$B --config 2 2>&1 | show "cfg2-f64"

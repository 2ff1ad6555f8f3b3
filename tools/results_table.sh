# DESIGN §9 results table (run under gpurun; one GPU): bench.py lines for configs 3-5, both dtypes,
# config 5's weak-scaling slab and K2_SC, D3Q15/D3Q27 on config 4, e2e included, no CPU leg.  One JSON line per run in gpurun_out/results.jsonl.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
: > gpurun_out/results.jsonl; : > gpurun_out/results_full.jsonl
for args in "--config 5 --dtype f64" "--config 5 --dtype f32" "--config 4 --dtype f64" "--config 4 --dtype f32" \
            "--config 3 --dtype f64" "--config 3 --dtype f32" "--config 5 --dtype f64 --weak" "--config 5 --dtype f64 --kernel k2sc" \
            "--config 4 --lattice 15 --dtype f64" "--config 4 --lattice 15 --dtype f32" \
            "--config 4 --lattice 27 --dtype f64" "--config 4 --lattice 27 --dtype f32"; do
  timeout 900 python bench.py $args --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/rt.json 2>/dev/null
  cat gpurun_out/rt.json >> gpurun_out/results_full.jsonl
  python - "$args" <<'PY' >> gpurun_out/results.jsonl
import json, sys
d = json.load(open("gpurun_out/rt.json"))
print(json.dumps({"args": sys.argv[1], "value": d["value"], "frac": d["roofline"]["frac"], "achieved": d["roofline"]["achieved"],
                  "e2e": (d.get("e2e") or {}).get("value"), "sm_mhz": d["clocks"]["sm_mhz"], "reasons": d["clocks"]["reasons"],
                  "ms_per_step": d["ms_per_step"]}))
PY
  tail -1 gpurun_out/results.jsonl
done

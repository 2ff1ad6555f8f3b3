python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "k2_equals_k1 or variants or local_slabs" 2>&1 | tail -1
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --kernel k2"
for ch in 0 24 32 48 64; do LBM_K2_CHUNK=$ch $SB --dtype f64 --tag grp-ch$ch; done
for gr in 74 296 100000; do LBM_K2_GROUP=$gr $SB --dtype f64 --tag grp$gr; done
for ch in 0 32; do LBM_K2_CHUNK=$ch $SB --dtype f32 --tag grp-ch$ch; done
M="dram__sectors_read.sum,gpu__time_duration.sum"
CMD="python tools/sweep_bench.py --dims 256,512,512 --steps 2 --reps 1 --kernel k2"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics $M --clock-control none -k regex:k2_sweep -s 2 -c 1 --csv $CMD 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print "grp", $(NF-2), $NF}'

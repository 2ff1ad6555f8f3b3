python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
M="dram__sectors_read.sum,gpu__time_duration.sum"
for pad in 0 32 64 256 4096; do
  LBM_PQ_PAD=$pad timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "k2_equals_k1 and dims5" 2>&1 | tail -1
  LBM_PQ_PAD=$pad timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --dtype f64 --kernel k2 --tag k2-pad$pad
  CMD="python tools/sweep_bench.py --dims 256,512,512 --steps 2 --reps 1 --kernel k2"
  LBM_PQ_PAD=$pad $CMD > gpurun_out/plain.log 2>&1 && LBM_PQ_PAD=$pad ncu --metrics $M --clock-control none -k regex:k2_sweep -s 2 -c 1 --csv $CMD 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' -v t="pad$pad" '{print t, $(NF-2), $NF}'
done
LBM_PQ_PAD=32 timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --dtype f32 --kernel k2 --tag k2-f32-pad32
LBM_PQ_PAD=32 timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --dtype f64 --kernel k1 --tag k1-pad32

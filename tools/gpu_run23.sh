python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SB="timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --steps 10 --reps 2 --kernel k2"
for pad in 0 8 24 56 120 504; do LBM_PITCH_PAD=$pad $SB --dtype f64 --tag pad$pad; done
for pad in 0 16 48; do LBM_PITCH_PAD=$pad $SB --dtype f32 --tag pad$pad; done
CMD="python tools/sweep_bench.py --dims 256,512,512 --steps 4 --reps 1 --kernel k2"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__sectors_read.sum,dram__sectors_write.sum --clock-control none -s 4 -c 6 --csv $CMD 2>/dev/null | grep -E "gpu__time|dram" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-150

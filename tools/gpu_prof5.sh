python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
M="dram__sectors_read.sum,dram__sectors_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum"
CMD="python tools/sweep_bench.py --dims 256,512,512 --steps 2 --reps 1"
for v in 256 none 64 128; do
  $CMD --kernel k2 > gpurun_out/plain.log 2>&1 && LBM_K2_L2PROMO=$v ncu --metrics $M --clock-control none -k regex:k2_sweep -s 2 -c 1 --csv $CMD --kernel k2 2>/dev/null | grep -E "dram__|gpu__time|lts__" | awk -F'","' -v t="promo-$v" '{print t, $(NF-2), $NF}'
done
$CMD --kernel k2reg > gpurun_out/plain.log 2>&1 && ncu --metrics $M --clock-control none -k regex:k2r_sweep -s 2 -c 1 --csv $CMD --kernel k2reg 2>/dev/null | grep -E "dram__|gpu__time|lts__" | awk -F'","' '{print "k2reg", $(NF-2), $NF}'
$CMD --kernel k1 > gpurun_out/plain.log 2>&1 && ncu --metrics $M --clock-control none -k regex:k1_step -s 2 -c 1 --csv $CMD --kernel k1 2>/dev/null | grep -E "dram__|gpu__time|lts__" | awk -F'","' '{print "k1", $(NF-2), $NF}'

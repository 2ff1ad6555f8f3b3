# A/B of a variant build on the D3Q15/D3Q27 kernels (run under gpurun; one GPU):
#   bash tools/dqq_ab.sh <variant>   -- bitwise K2Q == K1 of the variant, then sweeps, interleaved
v=$1
AB_LATTICES=15,27 LBM_PKG_ROOT=exp/$v timeout 600 python tools/ab_bitwise.py | tail -13 || exit 1
for rep in 1 2; do for root in . exp/$v; do
  for q in 27 15; do for dt in f64 f32; do for k in k1 k2; do
    LBM_PKG_ROOT=$root timeout 300 python tools/sweep_bench.py --dims 512,512,512 --lattice $q --steps 20 --reps 3 --dtype $dt --kernel $k --tag "$root q$q $k"
  done; done; done
done; done

set -o pipefail
AB_LATTICES=27 LBM_PKG_ROOT=exp/t8x8 timeout 600 python tools/ab_bitwise.py 2>&1 | tail -6 || exit 1
for rep in 1 2 3; do for root in . exp/t8x8; do
  LBM_PKG_ROOT=$root timeout 300 python tools/sweep_bench.py --dims 512,512,512 --lattice 27 --steps 20 --reps 3 --dtype f64 --kernel k2 --tag "$root q27 k2"
done; done
for root in . exp/t8x8; do
  LBM_PKG_ROOT=$root timeout 300 python tools/sweep_bench.py --dims 1024,512,512 --lattice 27 --steps 20 --reps 2 --dtype f64 --kernel k2 --tag "$root q27 cfg5 k2"
done

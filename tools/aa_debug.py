import numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lbm_inputs as li, paper_2208_05429_b200 as lbm
LID = (0.05, 0.0, 0.0)
for dims in [(1, 8, 32), (3, 9, 33), (2, 4, 4), (3, 4, 4)]:
    f0 = li.random_populations(47, *dims)
    with lbm.Lattice(*dims, 0.6, LID, "f64", kernel=lbm.LBM_KERNEL_K1) as ref, \
            lbm.Lattice(*dims, 0.6, LID, "f64", kernel=lbm.LBM_KERNEL_AA) as aa:
        ref.set_populations(f0); aa.set_populations(f0)
        print(dims, "t0 equal", np.array_equal(ref.populations(), aa.populations()))
        for n in range(1, 4):
            ref.step(1); aa.step(1)
            a, b = ref.populations(), aa.populations()
            d = np.argwhere(a != b)
            print(dims, "step", n, "ndiff", len(d), "maxdiff", np.max(np.abs(a - b)), d[:6].tolist())

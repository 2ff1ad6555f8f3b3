"""Cost of the D3Q15/27 NCCL x-slab path on one GPU:
a one-rank periodic NCCL context (ghost-plane pushes, self send/recv and the
merge every step) against the single-process one-step kernel (K1) and the
default two-step K2Q, 512^3, MLUPS from wall time around step + synchronize."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2208_05429_b200 as lbm  # noqa: E402

dims, n = (512, 512, 512), 20
for q in (15, 27):
    for dt in ("f64", "f32"):
        for tag, kw in [("K2Q", {}), ("K1", {"kernel": lbm.LBM_KERNEL_K1}),
                        ("NCCL", {"comm": lbm.LBM_COMM_NCCL, "nccl_id": lbm.lbm_nccl_unique_id()})]:
            with lbm.Lattice(*dims, 0.6, (0, 0, 0), dt, bc=lbm.LBM_BC_PERIODIC, lattice=q, **kw) as lat:
                lat.init_equilibrium(np.full(dims, 1.0), None)
                lat.step(4)
                lbm.lbm_synchronize(lat.ctx)
                best = 0.0
                for _ in range(3):
                    t0 = time.perf_counter()
                    lat.step(n)
                    lbm.lbm_synchronize(lat.ctx)
                    best = max(best, np.prod(dims) * n / (time.perf_counter() - t0) / 1e6)
                print(f"D3Q{q} {dt} {tag:5s} {best:9.0f} MLUPS", flush=True)

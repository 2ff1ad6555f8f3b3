"""A/B correctness gate for a variant build (LBM_PKG_ROOT=exp/<name>): K2 sweeps
of the variant must equal K1 steps of the same library bit for bit on ragged
cavity and periodic boxes, both dtypes (the product tests' K2 == K1 o K1
property, run before timing a variant).  Prints one line per case; exit 1 on
any mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("LBM_PKG_ROOT"):
    sys.path.insert(0, os.environ["LBM_PKG_ROOT"])

import numpy as np  # noqa: E402

import paper_2208_05429_b200 as lbm  # noqa: E402

print("library:", lbm.__file__)
bad = 0
rng = np.random.default_rng(7)
lattices = [int(v) for v in os.environ.get("AB_LATTICES", "19").split(",")]
for q, dims in [(q, d) for q in lattices for d in [(37, 45, 70), (20, 19, 97), (64, 64, 64)]]:
    for bc in (lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC):
        for dt in ("f64", "f32"):
            nx, ny, nz = dims
            rho = (1 + 1e-3 * rng.uniform(-1, 1, (nx, ny, nz))).astype(np.float64)
            u = (0.02 * rng.uniform(-1, 1, (nx, ny, nz, 3))).astype(np.float64)
            out = []
            for kern in [int(v) for v in os.environ.get("AB_KERNELS", "1,2").split(",")]:
                with lbm.Lattice(nx, ny, nz, 0.6, (0.05, 0, 0), dt, bc=bc, kernel=kern, lattice=q) as lat:
                    lat.init_equilibrium(rho, u)
                    lat.step(6)
                    out.append(lat.populations())
            same = np.array_equal(out[0], out[1])
            bad += not same
            print(f"q{q} {dims} bc={bc} {dt}: {'bitwise' if same else 'MISMATCH max %.3e' % np.max(np.abs(out[0] - out[1]))}")
sys.exit(1 if bad else 0)

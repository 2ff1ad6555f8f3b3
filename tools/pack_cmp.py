"""Probe: D3Q15 fp32 one-step and two-step results of the library at
LBM_PKG_ROOT, saved to <out>.npz (compare two builds bit for bit)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("LBM_PKG_ROOT"):
    sys.path.insert(0, os.environ["LBM_PKG_ROOT"])
import numpy as np  # noqa: E402

import lbm_inputs as li  # noqa: E402
import paper_2208_05429_b200 as lbm  # noqa: E402

q, dims = 15, (70, 21, 45)
f0 = li.uniform(105, q * int(np.prod(dims)), 0.01, 0.06).reshape(q, *dims)
res = {}
for name, kern, n in (("k1_1", 1, 1), ("k1_4", 1, 4), ("k2_4", 2, 4)):
    with lbm.Lattice(*dims, 0.6, (0.05, 0, 0), "f32", lattice=q, kernel=kern) as lat:
        lat.set_populations(f0)
        lat.step(n)
        res[name] = lat.populations()
np.savez(sys.argv[1], **res)
print(lbm.__file__, "k1_4 == k2_4:", np.array_equal(res["k1_4"], res["k2_4"]))

"""Small runs of every kernel family for compute-sanitizer (SURVEY.md §5
race detection): memcheck (out-of-bounds / misaligned global and shared
accesses), racecheck (shared-memory hazards in K2's / K3's rings and stage
buffers), synccheck (barrier misuse).  Each case also checks its result
against a K1 run of the same state, so a sanitizer-clean run is a correct
one.

    compute-sanitizer --tool memcheck  --error-exitcode 9 python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import lbm_inputs as li  # noqa: E402
import paper_2208_05429_b200 as lbm  # noqa: E402

LID = (0.05, 0.0, 0.0)
CASES = [
    # (name, dims, bc, dtype, kwargs)
    ("k2 cavity f64", (6, 17, 40), lbm.LBM_BC_CAVITY, "f64", dict(kernel=lbm.LBM_KERNEL_K2)),
    ("k2 periodic f32", (6, 17, 40), lbm.LBM_BC_PERIODIC, "f32", dict(kernel=lbm.LBM_KERNEL_K2)),
    ("k2 periodic f64", (5, 9, 33), lbm.LBM_BC_PERIODIC, "f64", dict(kernel=lbm.LBM_KERNEL_K2)),
    ("k2_sc cavity f64", (8, 12, 36), lbm.LBM_BC_CAVITY, "f64", dict(kernel=lbm.LBM_KERNEL_K2_SC)),
    ("aa cavity f64", (6, 10, 35), lbm.LBM_BC_CAVITY, "f64", dict(kernel=lbm.LBM_KERNEL_AA)),
    ("k3 periodic f32", (6, 13, 40), lbm.LBM_BC_PERIODIC, "f32", dict(kernel=lbm.LBM_KERNEL_K3)),
    ("local slabs periodic f64", (16, 10, 36), lbm.LBM_BC_PERIODIC, "f64",
     dict(comm=lbm.LBM_COMM_LOCAL, local_slabs=4)),
    ("x-y blocks cavity f32", (8, 16, 40), lbm.LBM_BC_CAVITY, "f32",
     dict(comm=lbm.LBM_COMM_LOCAL, local_slabs=2, local_blocks_y=2)),
    ("d3q27 cavity f64", (4, 9, 33), lbm.LBM_BC_CAVITY, "f64", dict(lattice=27)),
    ("d3q15 periodic f32", (4, 9, 33), lbm.LBM_BC_PERIODIC, "f32", dict(lattice=15)),
]


def run(dims, bc, dtype, kw, n=7):
    q = kw.get("lattice", 19)
    f0 = li.uniform(90, q * int(np.prod(dims)), 0.01, 0.06).reshape(q, *dims)
    with lbm.Lattice(*dims, 0.6, LID, dtype, bc=bc, **kw) as lat:
        lat.set_populations(f0)
        lat.step(n)
        out = lat.populations()
        lat.macroscopic()
    return f0, out


def main():
    bad = 0
    for name, dims, bc, dtype, kw in CASES:
        f0, got = run(dims, bc, dtype, kw)
        ref_kw = {"lattice": kw["lattice"]} if "lattice" in kw else {"kernel": lbm.LBM_KERNEL_K1}
        _, want = run(dims, bc, dtype, ref_kw)
        ok = np.array_equal(got, want) or (kw.get("kernel") == lbm.LBM_KERNEL_AA and np.allclose(got, want, 1e-12))
        bad += not ok
        print(f"{name:28s} {'ok' if ok else 'MISMATCH'}", flush=True)
    print("sanitize cases:", "all ok" if not bad else f"{bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())

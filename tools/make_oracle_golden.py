"""Write the oracle's state after the configured step count of a BASELINE
config, sampled, to tests/golden/cfg{N}_oracle_t{steps}.npz.

Calls only oracle/ (the plain CPU solver) and lbm_inputs (the seeded input
recipe); nothing here touches the CUDA path.  The GPU parity tests
(tests/test_gpu_golden.py) compare the library against these values after
the same number of steps (BASELINE.json:5 "after the configured step count";
PAPER.md:832-837 verifies solvers by comparing final fields).

Host memory: two fp64 lattices (2 * cells * 152 B) plus the input field and
the moments: ~47 GB for config 4 and ~95 GB for config 5.  Run config 5 on a
host with enough RAM (the GPU box: `gpurun -- python tools/make_oracle_golden.py
--config 5`).

What is stored (every value is the oracle's):
  origins[K,3], box[3], boxes[K,19,bx,by,bz]   canonical f(t_end) on K sampled
      boxes: the 8 domain corners, the 12 edge midpoints, the 6 face centres,
      x-chunk seams (x = m*c - 2 for the chunk lengths the planner may use),
      y % 8 / z % 32 tile seams and seeded interior points;
  line_x[19,nx], line_y[19,ny], line_z[19,nz]  three full lines through the
      domain (every x-chunk seam, every y tile seam, every z tile seam);
  plane_mass[nx], plane_mom[nx,3]              sum over each x plane of rho and
      rho*u (the oracle's moments, oracle.macroscopic).
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import lbm_inputs as li  # noqa: E402
import oracle  # noqa: E402

BOX = (4, 4, 4)
N_BOXES = 64
CHUNKS = (32, 48, 52, 54, 56)


def sample_origins(cfg) -> np.ndarray:
    nx, ny, nz = cfg.nx, cfg.ny, cfg.nz
    bx, by, bz = BOX
    xs = (0, nx // 2 - bx // 2, nx - bx)
    ys = (0, ny // 2 - by // 2, ny - by)
    zs = (0, nz // 2 - bz // 2, nz - bz)
    out = []
    # {lo, mid, hi} per axis except the centre: the 8 corners, the 12 edge
    # midpoints and the 6 face centres
    for i in range(3):
        for j in range(3):
            for k in range(3):
                if (i, j, k) != (1, 1, 1):
                    out.append((xs[i], ys[j], zs[k]))
    rng = np.random.default_rng(1000 + cfg.seed)
    # x-chunk seams with y/z tile seams
    for c in CHUNKS:
        for m in (1, 2, 3):
            x0 = m * c - 2
            if x0 + bx > nx:
                continue
            y0 = 8 * int(rng.integers(1, ny // 8)) - 2
            z0 = 32 * int(rng.integers(1, max(2, nz // 32))) - 2
            out.append((x0, min(max(y0, 0), ny - by), min(max(z0, 0), nz - bz)))
    while len(out) < N_BOXES:
        out.append((int(rng.integers(0, nx - bx + 1)), int(rng.integers(0, ny - by + 1)),
                    int(rng.integers(0, nz - bz + 1))))
    return np.array(out[:N_BOXES], dtype=np.int64)


def line_coords(cfg):
    """(y, z) of the x line, (x, z) of the y line, (x, y) of the z line."""
    nx, ny, nz = cfg.nx, cfg.ny, cfg.nz
    return (ny // 2 + 3, nz - 1), (nx // 2 + 1, 1), (nx // 3, ny - 1)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--steps", type=int, default=None, help="default: the config's own step count")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = li.CONFIGS[a.config]
    steps = cfg.steps if a.steps is None else a.steps
    out = a.out or os.path.join(ROOT, "tests", "golden", f"cfg{a.config}_oracle_t{steps}.npz")
    oracle.set_threads(a.threads)

    t0 = time.time()
    rho, u = li.init_fields(cfg)
    f = oracle.init_equilibrium(cfg.nx, cfg.ny, cfg.nz, rho, None if not np.any(u) else u)
    del rho, u
    t1 = time.time()
    oracle.run_inplace(f, cfg.bc, cfg.tau, cfg.u_lid, steps)
    t2 = time.time()

    origins = sample_origins(cfg)
    bx, by, bz = BOX
    boxes = np.stack([f[:, x:x + bx, y:y + by, z:z + bz] for x, y, z in origins])
    (ly, lz), (mx, mz), (nx_, ny_) = line_coords(cfg)
    line_x = np.ascontiguousarray(f[:, :, ly, lz])
    line_y = np.ascontiguousarray(f[:, mx, :, mz])
    line_z = np.ascontiguousarray(f[:, nx_, ny_, :])
    rho, vel = oracle.macroscopic(f)
    del f
    plane_mass = rho.sum(axis=(1, 2))
    plane_mom = (rho[..., None] * vel).sum(axis=(1, 2))
    t3 = time.time()

    src = open(os.path.join(ROOT, "oracle", "oracle.c"), "rb").read()
    np.savez_compressed(
        out, config=a.config, name=cfg.name, steps=steps, dims=np.array([cfg.nx, cfg.ny, cfg.nz]),
        origins=origins, box=np.array(BOX), boxes=boxes,
        line_coords=np.array(line_coords(cfg)), line_x=line_x, line_y=line_y, line_z=line_z,
        plane_mass=plane_mass, plane_mom=plane_mom,
        oracle_sha256=hashlib.sha256(src).hexdigest(), threads=oracle.get_threads(),
        seconds=np.array([t1 - t0, t2 - t1, t3 - t2]))
    print(f"{cfg.name}: {steps} steps on {oracle.get_threads()} threads: init {t1 - t0:.1f} s, "
          f"run {t2 - t1:.1f} s ({cfg.cells * steps / (t2 - t1) / 1e6:.2f} MLUPS), "
          f"sample {t3 - t2:.1f} s -> {out}")


if __name__ == "__main__":
    main()

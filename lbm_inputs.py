"""Seeded synthetic inputs shared by tests/ and bench.py.

This module holds NO arithmetic of the method (no collision, equilibrium or
streaming): only the BASELINE.json workload definitions and a counter-based
random generator that draws their initial fields.  Both the oracle side and
the CUDA side receive the same arrays from here.

Generator: splitmix64.  Draw k (k = 1, 2, ...) uses
state s_k = seed + k * 0x9E3779B97F4A7C15 (mod 2^64) and the output mix
  z = (s ^ (s >> 30)) * 0xBF58476D1CE4E5B9
  z = (z ^ (z >> 27)) * 0x94D049BB133111EB
  out = z ^ (z >> 31);
u01 = (out >> 11) * 2^-53 and U(a, b) = a + (b - a) * u01.  Cells are drawn
in canonical order (x slowest, z fastest); for a vector field the components
of one cell are consecutive draws.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

BC_CAVITY = 0
BC_PERIODIC = 1


def splitmix64(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Outputs number start+1 .. start+count of splitmix64 seeded with ``seed``."""
    k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + k * GAMMA
        z = (s ^ (s >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, count: int, a: float, b: float, start: int = 0) -> np.ndarray:
    u01 = (splitmix64(seed, count, start) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return a + (b - a) * u01


@dataclass(frozen=True)
class Config:
    """One BASELINE.json workload (BASELINE.json:7-11)."""
    name: str
    nx: int
    ny: int
    nz: int
    bc: int
    tau: float
    u_lid: tuple
    steps: int
    seed: int
    init: str  # "rho_noise" (rho = 1 + U(-1e-3, 1e-3), u = 0) or "u_noise" (rho = 1, u_a = U(-0.01, 0.01))
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def cells(self) -> int:
        return self.nx * self.ny * self.nz

    def with_dims(self, nx, ny, nz, steps=None) -> "Config":
        return Config(self.name + f"@{nx}x{ny}x{nz}", nx, ny, nz, self.bc, self.tau, self.u_lid,
                      self.steps if steps is None else steps, self.seed, self.init, self.note)


LID = (0.05, 0.0, 0.0)

CONFIGS = {
    1: Config("cfg1_cavity_16^3", 16, 16, 16, BC_CAVITY, 0.6, LID, 20, 0, "rho_noise",
              "BASELINE.json:7 - 16^3 lid-driven cavity, 20 steps"),
    2: Config("cfg2_cavity_64^3", 64, 64, 64, BC_CAVITY, 0.6, LID, 1000, 1, "rho_noise",
              "BASELINE.json:8 - 64^3 lid-driven cavity, 1000 steps"),
    3: Config("cfg3_periodic_256^3", 256, 256, 256, BC_PERIODIC, 0.55, (0.0, 0.0, 0.0), 200, 2, "u_noise",
              "BASELINE.json:9 - 256^3 fully periodic box, 200 steps"),
    4: Config("cfg4_cavity_512^3", 512, 512, 512, BC_CAVITY, 0.6, LID, 100, 3, "rho_noise",
              "BASELINE.json:10 - 512^3 lid-driven cavity, 100 steps"),
    5: Config("cfg5_cavity_1024x512x512", 1024, 512, 512, BC_CAVITY, 0.6, LID, 100, 4, "rho_noise",
              "BASELINE.json:11 - 1024x512x512 cuboid lid-driven cavity, 100 steps"),
}


def init_fields(cfg: Config, x0: int = 0, nx_local: int | None = None):
    """(rho[nxl,ny,nz], u[nxl,ny,nz,3]) float64 for planes [x0, x0 + nx_local).

    The draws are those of the whole domain (cell index = (x*ny + y)*nz + z),
    so a slab of a multi-GPU run sees exactly the values of the 1-GPU run.
    """
    nxl = cfg.nx - x0 if nx_local is None else nx_local
    plane = cfg.ny * cfg.nz
    n = nxl * plane
    if cfg.init == "rho_noise":
        rho = uniform(cfg.seed, n, -1e-3, 1e-3, start=x0 * plane) + 1.0
        u = np.zeros((n, 3))
    elif cfg.init == "u_noise":
        rho = np.ones(n)
        u = uniform(cfg.seed, 3 * n, -0.01, 0.01, start=3 * x0 * plane).reshape(n, 3)
    else:
        raise ValueError(cfg.init)
    return rho.reshape(nxl, cfg.ny, cfg.nz), u.reshape(nxl, cfg.ny, cfg.nz, 3)


def random_populations(seed: int, nx: int, ny: int, nz: int, lo=0.01, hi=0.06) -> np.ndarray:
    """Positive random f[19,nx,ny,nz] for parity cases off equilibrium."""
    return uniform(seed, 19 * nx * ny * nz, lo, hi).reshape(19, nx, ny, nz)

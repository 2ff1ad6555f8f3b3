"""Test-only numpy D3Q19 helpers for host-logic tests (halo plan, slabs).

Independent of both the oracle and the CUDA path: the BGK update is written
from the textbook form over whole arrays, streaming as per-direction pulls.
Arrays are canonical-direction f[19, x, y, z]; "A" arrays hold
post-collision populations (the library's storage form).
"""
import numpy as np

CVEC = [(0, 0, 0),
        (-1, 0, 0), (0, -1, 0), (0, 0, -1), (-1, -1, 0), (-1, 1, 0),
        (-1, 0, -1), (-1, 0, 1), (0, -1, -1), (0, -1, 1),
        (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, -1, 0),
        (1, 0, 1), (1, 0, -1), (0, 1, 1), (0, 1, -1)]
W = np.array([1 / 3] + [1 / 18 if sum(abs(a) for a in c) == 1 else 1 / 36 for c in CVEC[1:]])


def opp(i):
    return 0 if i == 0 else (i + 9 if i <= 9 else i - 9)


def bgk(f, tau):
    rho = f.sum(axis=0)
    j = np.stack([sum(CVEC[i][a] * f[i] for i in range(19)) for a in range(3)])
    u = j / rho
    usq = (u * u).sum(axis=0)
    feq = np.empty_like(f)
    for i in range(1, 19):
        cu = CVEC[i][0] * u[0] + CVEC[i][1] * u[1] + CVEC[i][2] * u[2]
        feq[i] = W[i] * rho * (1 + 3 * cu + 4.5 * cu * cu - 1.5 * usq)
    feq[0] = rho - feq[1:].sum(axis=0)
    return f - (f - feq) / tau


def pull(A, xs, periodic, u_lid, wall_lo=None, wall_hi=None, wrap_x=False):
    """Canonical f(t) on the planes xs of A (indices along A's x axis) from
    post-collision A.  x-neighbours come from A itself (ghost planes
    included); wall_lo / wall_hi are the indices of planes whose left /
    right neighbour is a cavity wall.  A missing source plane yields NaN so
    that an insufficient halo shows up."""
    _, nxa, ny, nz = A.shape
    out = np.empty((19, len(xs), ny, nz))
    for n, x in enumerate(xs):
        for i in range(19):
            cx, cy, cz = CVEC[i]
            xwall = (cx == 1 and x == wall_lo) or (cx == -1 and x == wall_hi)
            sx = (x - cx) % nxa if wrap_x else x - cx
            src = A[i, sx] if (0 <= sx < nxa and not xwall) else np.full((ny, nz), np.nan)
            if periodic:
                out[i, n] = np.roll(np.roll(src, cy, axis=0), cz, axis=1)
                continue
            v = np.full((ny, nz), np.nan)
            # v[y, z] = src[y - cy, z - cz] where the source is inside
            v[max(cy, 0):ny + min(cy, 0), max(cz, 0):nz + min(cz, 0)] = \
                src[max(-cy, 0):ny + min(-cy, 0), max(-cz, 0):nz + min(-cz, 0)]
            wall = np.zeros((ny, nz), dtype=bool)
            if cy == 1:
                wall[0, :] = True
            if cy == -1:
                wall[ny - 1, :] = True
            if cz == 1:
                wall[:, 0] = True
            if cz == -1:
                wall[:, nz - 1] = True
            if xwall:
                wall[:, :] = True
            v = np.where(wall, A[opp(i), x], v)
            if cz == -1:
                v[:, nz - 1] += 6.0 * W[i] * (cx * u_lid[0] + cy * u_lid[1] + cz * u_lid[2])
            out[i, n] = v
    return out


def step(A, tau, periodic, u_lid, xs, wall_lo=None, wall_hi=None, wrap_x=False):
    """One library step on the planes xs: f*(t) = C(S(f*(t-1)))."""
    return bgk(pull(A, xs, periodic, u_lid, wall_lo, wall_hi, wrap_x), tau)

"""Test-only restatements of the paper's in-place schedules (pure Python).

These are PINS for the oracle, not product code: the paper claims that its
single-copy swap schedules compute the same lattice update as a plain
collide-then-stream step.  Restating
those schedules from the paper and checking that they reproduce the oracle
bit for bit pins the oracle's streaming and boundary logic with an
independent data-movement scheme (swap + revert instead of a pull copy).

Conventions (SPEC.md module "lattice"/"kernels"): 1-based cell indices
(iX, iY, iZ) as in the paper's algorithms; the field is a numpy array
F[x, y, z, i] (0-based storage, cell-major, 19 slots per cell).

The per-cell collision is delegated to the oracle (``oracle.collide``):
the schedule, not the BGK arithmetic, is what these functions restate.
"""
from __future__ import annotations

import numpy as np

import oracle

# SPEC.md:109 direction order (retyped here; independent of the oracle's table)
CVEC = [(0, 0, 0),
        (-1, 0, 0), (0, -1, 0), (0, 0, -1), (-1, -1, 0), (-1, 1, 0),
        (-1, 0, -1), (-1, 0, 1), (0, -1, -1), (0, -1, 1),
        (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, -1, 0),
        (1, 0, 1), (1, 0, -1), (0, 1, 1), (0, 1, -1)]
WGT = [1 / 3] + [1 / 18 if sum(abs(a) for a in c) == 1 else 1 / 36 for c in CVEC[1:]]


def opp(i: int) -> int:
    return 0 if i == 0 else (i + 9 if i <= 9 else i - 9)


class SwapLattice:
    """Single-copy lattice with the paper's collide / revert / swap_stream.

    Optional instrumentation (``check=True``) records, per cell, how many
    collide+revert operations it has done and which links were swapped in
    which computation, and counts violations of the swap preconditions
    ("we must guarantee that the populations of neighbors
    involved in the swap are already in a post-collision state").
    """

    def __init__(self, f_canonical: np.ndarray, tau: float, u_lid, check: bool = False):
        # f_canonical: oracle layout (19, nx, ny, nz) -> cell-major F[x,y,z,i]
        self.F = np.ascontiguousarray(np.moveaxis(f_canonical, 0, -1)).copy()
        self.lx, self.ly, self.lz = self.F.shape[:3]
        self.omega = 1.0 / tau
        self.u_lid = tuple(float(v) for v in u_lid)
        self.check = check
        self.ncoll = np.zeros((self.lx, self.ly, self.lz), dtype=np.int64)
        self.swapped = {}  # (cell, i, comp) -> count
        self.violations = []
        self.log = []  # (kind, comp, (iX,iY,iZ))

    # -- geometry -------------------------------------------------------
    def inside(self, iX, iY, iZ) -> bool:
        return 1 <= iX <= self.lx and 1 <= iY <= self.ly and 1 <= iZ <= self.lz

    def on_boundary(self, iX, iY, iZ) -> bool:
        return iX in (1, self.lx) or iY in (1, self.ly) or iZ in (1, self.lz)

    def links(self, iX, iY, iZ) -> int:
        """Number of in-domain neighbours of a cell (its swappable links)."""
        return sum(self.inside(iX + c[0], iY + c[1], iZ + c[2]) for c in CVEC[1:])

    # -- primitives -----------------------------------------------------
    def collide_revert(self, iX, iY, iZ):
        """collide, then revert, then the lid correction."""
        x, y, z = iX - 1, iY - 1, iZ - 1
        comp = int(self.ncoll[x, y, z]) + 1
        if self.check and comp >= 2:
            done = sum(self.swapped.get(((iX, iY, iZ), j, comp - 1), 0) for j in range(1, 19))
            if done != self.links(iX, iY, iZ):
                self.violations.append(("collide-before-streamed", comp, (iX, iY, iZ)))
        post = oracle.collide(self.F[x, y, z, :], self.omega)
        rev = post.copy()
        for i in range(1, 10):  # revert: slots i and i+9 exchange
            rev[i], rev[i + 9] = post[i + 9], post[i]
        # moving lid at the top z face: slot i receives f*_opp(i) + 6 w_i rho_w (c_i.u)
        # for every i whose pull source lies beyond the lid
        for i in range(1, 19):
            if iZ - CVEC[i][2] > self.lz:
                cu = CVEC[i][0] * self.u_lid[0] + CVEC[i][1] * self.u_lid[1] + CVEC[i][2] * self.u_lid[2]
                rev[i] = rev[i] + 6.0 * WGT[i] * 1.0 * cu
        self.F[x, y, z, :] = rev
        self.ncoll[x, y, z] = comp
        self.log.append(("collide", comp, (iX, iY, iZ)))

    def swap_stream(self, iX, iY, iZ, boundary: bool):
        """Exchange slot opp(i) of this cell with slot i of the neighbour at
        +c_i, i = 1..9; boundary variant skips links that
        leave the box."""
        x, y, z = iX - 1, iY - 1, iZ - 1
        comp = int(self.ncoll[x, y, z])
        for i in range(1, 10):
            nX, nY, nZ = iX + CVEC[i][0], iY + CVEC[i][1], iZ + CVEC[i][2]
            if not self.inside(nX, nY, nZ):
                if not boundary:
                    raise AssertionError("bulk swap_stream on a boundary cell")
                continue
            if self.check:
                if self.ncoll[nX - 1, nY - 1, nZ - 1] != comp:
                    self.violations.append(("partner-not-collided", comp, (iX, iY, iZ), i))
                key = ((iX, iY, iZ), i + 9, comp)
                if self.swapped.get(key, 0):
                    self.violations.append(("link-twice", comp, (iX, iY, iZ), i))
                self.swapped[key] = self.swapped.get(key, 0) + 1
                nkey = ((nX, nY, nZ), i, comp)
                self.swapped[nkey] = self.swapped.get(nkey, 0) + 1
            a = self.F[x, y, z, i + 9]
            self.F[x, y, z, i + 9] = self.F[nX - 1, nY - 1, nZ - 1, i]
            self.F[nX - 1, nY - 1, nZ - 1, i] = a
        self.log.append(("stream", comp, (iX, iY, iZ)))

    # -- Alg. 2 helpers ---------------------------------
    def boundary_cell_comp(self, iX, iY, iZ):
        if not self.inside(iX, iY, iZ):
            return
        self.collide_revert(iX, iY, iZ)
        self.swap_stream(iX, iY, iZ, boundary=True)

    def adaptive_collide_stream(self, iX, iY, iZ):
        if self.on_boundary(iX, iY, iZ):
            self.boundary_cell_comp(iX, iY, iZ)
        else:
            self.collide_revert(iX, iY, iZ)
            self.swap_stream(iX, iY, iZ, boundary=False)

    def boundary_neighbor_handler(self, iX, iY, iZ, corrected: bool):
        lz, ly = self.lz, self.ly
        # condition 1: last cell of a row
        if iZ == lz:
            self.boundary_cell_comp(iX - 1, iY - 1, iZ)
        if not corrected:
            # condition 2 as printed
            if iY == ly and iZ > 1:
                self.boundary_cell_comp(iX - 1, iY, iZ - 1)
            # condition 3
            if iY == ly and iZ == lz:
                self.boundary_cell_comp(iX - 1, iY, iZ)
        else:
            # DESIGN.md R-12 (SURVEY C-12): the c_9 = (0,-1,+1) partner of
            # (iX-1, ly, iZ-1) is second-collided only at cursor (iX, ly, iZ+1)
            if iY == ly and iZ > 2:
                self.boundary_cell_comp(iX - 1, iY, iZ - 2)
            if iY == ly and iZ == lz:
                self.boundary_cell_comp(iX - 1, iY, iZ - 1)
                self.boundary_cell_comp(iX - 1, iY, iZ)

    def canonical(self) -> np.ndarray:
        return np.ascontiguousarray(np.moveaxis(self.F, -1, 0))


def fuse_swap_step(f: np.ndarray, tau: float, u_lid, check=False):
    """Alg. 1, "3D Fuse Swap LBM": one time step.

    Stage I: collide and revert on the 6 faces; Stage II: bulk collide &
    swap_stream in ascending X, Y, Z; Stage III: boundary_swap_stream on the
    bounding box."""
    L = SwapLattice(f, tau, u_lid, check)
    lx, ly, lz = L.lx, L.ly, L.lz
    cells = [(X, Y, Z) for X in range(1, lx + 1) for Y in range(1, ly + 1) for Z in range(1, lz + 1)]
    for c in cells:  # Stage I
        if L.on_boundary(*c):
            L.collide_revert(*c)
    for c in cells:  # Stage II
        if not L.on_boundary(*c):
            L.collide_revert(*c)
            L.swap_stream(*c, boundary=False)
    for c in cells:  # Stage III
        if L.on_boundary(*c):
            L.swap_stream(*c, boundary=True)
    return L


def prism_blocks(lx, ly, lz, tile, x0=1, x1=None):
    """Alg. 2 lines 3-5."""
    x1 = lx if x1 is None else x1
    for oX in range(x0, x1 + 1, tile):
        for oY in range(1, ly + tile - 1 + 1, tile):
            for oZ in range(1, lz + 2 * (tile - 1) + 1, tile):
                yield (oX, oY, oZ)


def prism_cells(lx, ly, lz, tile, block, x1=None, clamp_dy=False):
    """Alg. 2 lines 6-9.

    dx = innerX - outerX (dx is never initialised in the pseudocode).  dy is
    the row offset from the UNCLAMPED minY, so a window cut by the domain
    boundary is a truncated parallelogram ("we truncate the
    parallelograms") and the 4x16x16 example has 30 non-empty prisms
    ("from Prism 1 to Prism 30").  clamp_dy=True restarts dy
    at the clamped row, the literal placement of "dy = 0" on line 7, which
    leaves one of the 30 blocks empty (R-13)."""
    x1 = lx if x1 is None else x1
    oX, oY, oZ = block
    for dx, iX in enumerate(range(oX, min(oX + tile - 1, x1) + 1)):
        minY = oY - dx
        maxY = minY + tile - 1
        for iY in range(max(minY, 1), min(maxY, ly) + 1):
            dy = iY - (max(minY, 1) if clamp_dy else minY)
            minZ = oZ - dx - dy
            maxZ = minZ + tile - 1
            for iZ in range(max(minZ, 1), min(maxZ, lz) + 1):
                yield (iX, iY, iZ)


def traversal(lx, ly, lz, tile, clamp_dy=False):
    for b in prism_blocks(lx, ly, lz, tile):
        yield from prism_cells(lx, ly, lz, tile, b, clamp_dy=clamp_dy)


def two_step_cycle(f: np.ndarray, tau: float, u_lid, tile=None, corrected=True, check=False,
                   clamp_dy=False):
    """Alg. 2, "3D Sequential Memory-aware LBM": two time
    steps in one sweep.  tile=None is the single-prism ("2-step LBM") order."""
    L = SwapLattice(f, tau, u_lid, check)
    lx, ly, lz = L.lx, L.ly, L.lz
    if tile is None:
        tile = lx + ly + lz
    for (iX, iY, iZ) in traversal(lx, ly, lz, tile, clamp_dy):
        # (1) first computation at time step t
        L.adaptive_collide_stream(iX, iY, iZ)
        # (2) second computation at time step t+1, lagged by (1,1,1)
        if iX > 1 and iY > 1 and iZ > 1:
            L.adaptive_collide_stream(iX - 1, iY - 1, iZ - 1)
        # (3) second computation of neighbours at certain locations
        L.boundary_neighbor_handler(iX, iY, iZ, corrected)
    # second collide, revert & boundary_swap_stream on the top layer iX = lx
    for iY in range(1, ly + 1):
        for iZ in range(1, lz + 1):
            L.boundary_cell_comp(lx, iY, iZ)
    return L

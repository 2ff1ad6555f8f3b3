"""Pins for the CPU oracle (oracle/oracle.c), run without a GPU.

Each test checks the oracle against something the paper or the mathematics
fixes, not against a retyped copy of its own formulas (DESIGN.md section
"Oracle and its pins").  A plausible mistake anywhere in the oracle -- a
dropped equilibrium term, a wrong sign or index in the stream, a transposed
velocity, a mis-signed lid term, a wrong tau convention -- fails at least
one of them:

  table / weights     -> rational isotropy identities (closed form)
  equilibrium         -> exact rational moments + SPEC.md:81 printed value
  collide             -> conservation, fixed point, omega = 1 projection
  stream + bounce     -> independent numpy brute force on 4^3, Alg. 1 swap
                         schedule bit-for-bit
  lid                 -> closed-form one-step values (golden/lid_one_step.txt)
  two-step merge      -> corrected Alg. 2 bit-for-bit,
                         the paper's 4^3 walk-through order
  tau convention      -> shear-wave decay nu = (tau - 1/2)/3 (textbook)
  conservation        -> mass <= 1e-13 (BASELINE.json:5), periodic momentum
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import lbm_inputs as li
import oracle
import paper_algs as pa

LID = (0.05, 0.0, 0.0)


def read_table(golden_dir, name):
    rows = []
    with open(os.path.join(golden_dir, name)) as fh:
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if line:
                rows.append(line.split())
    return rows


# ---------------------------------------------------------------- lattice --
def test_table_matches_spec(golden_dir):
    c, w, opp = oracle.d3q19()
    rows = read_table(golden_dir, "d3q19_table.txt")
    assert len(rows) == 19
    for r in rows:
        i = int(r[0])
        assert tuple(c[i]) == (int(r[1]), int(r[2]), int(r[3]))
        assert w[i] == float(Fraction(r[4]))  # nearest double to the rational
        assert opp[i] == int(r[5])


def test_table_rational_isotropy():
    """Sum w = 1, sum w c = 0, sum w c c = I/3, odd third moments 0,
    sum w c c c c = (dd + dd + dd)/9 -- the D3Q19 closed forms."""
    c, w, opp = oracle.d3q19()
    wr = [Fraction(x).limit_denominator(100) for x in w]
    assert sum(wr) == 1
    for a in range(3):
        assert sum(wr[i] * c[i][a] for i in range(19)) == 0
        for b in range(3):
            assert sum(wr[i] * c[i][a] * c[i][b] for i in range(19)) == (Fraction(1, 3) if a == b else 0)
            for g in range(3):
                assert sum(wr[i] * c[i][a] * c[i][b] * c[i][g] for i in range(19)) == 0
                for d in range(3):
                    lhs = sum(wr[i] * c[i][a] * c[i][b] * c[i][g] * c[i][d] for i in range(19))
                    rhs = Fraction((a == b) * (g == d) + (a == g) * (b == d) + (a == d) * (b == g), 9)
                    assert lhs == rhs
    for i in range(19):
        assert opp[opp[i]] == i
        assert tuple(c[opp[i]]) == tuple(-c[i])
    # directions 1..9 are lexicographically negative
    for i in range(1, 10):
        first = next(v for v in c[i] if v != 0)
        assert first == -1


# ------------------------------------------------------------ equilibrium --
def test_equilibrium_printed_examples(golden_dir):
    for r in read_table(golden_dir, "equilibrium_examples.txt"):
        rho, ux, uy, uz = map(float, r[:4])
        slot, expected, tol = int(r[4]), float(r[5]), float(r[6])
        assert abs(oracle.equilibrium(rho, (ux, uy, uz))[slot] - expected) <= tol


@pytest.mark.parametrize("rho,u", [(1.2, (0.02, -0.01, 0.05)), (0.97, (0.1, 0.0, -0.07)),
                                   (1.0, (0.0, 0.0, 0.0)), (1.0005, (-0.03, 0.08, 0.01))])
def test_equilibrium_moments_closed_form(rho, u):
    """sum feq = rho, sum c feq = rho u, sum c c feq = rho (u u + I/3):
    the defining moments of the second-order equilibrium."""
    c, _, _ = oracle.d3q19()
    feq = oracle.equilibrium(rho, u)
    u = np.array(u)
    assert abs(math.fsum(feq) - rho) <= 1e-15
    j = c.T.astype(float) @ feq
    assert np.allclose(j, rho * u, atol=1e-15, rtol=0)
    P = np.einsum("ia,ib,i->ab", c.astype(float), c.astype(float), feq)
    assert np.allclose(P, rho * (np.outer(u, u) + np.eye(3) / 3), atol=2e-16 * 8, rtol=0)
    # projection fixed point
    r2, u2 = oracle.moments(feq)
    assert abs(r2 - rho) <= 1e-15 and np.allclose(u2, u, atol=1e-15)
    assert np.allclose(oracle.equilibrium(r2, u2), feq, atol=1e-15, rtol=0)


def test_moments_degenerate_is_an_error():
    with pytest.raises(ZeroDivisionError):
        oracle.moments(np.zeros(19))


# ---------------------------------------------------------------- collide --
def test_collide_invariants():
    """equilibrium is a fixed point; omega = 1 returns
    the equilibrium of the moments; rho and j are conserved."""
    c, _, _ = oracle.d3q19()
    rng_f = li.uniform(11, 19 * 20, 0.01, 0.08).reshape(20, 19)
    for f in rng_f:
        for omega in (1 / 0.55, 1 / 0.6, 1.0, 1.7):
            g = oracle.collide(f, omega)
            assert abs(math.fsum(g) - math.fsum(f)) <= 1e-15
            assert np.allclose(c.T @ g, c.T @ f, atol=1e-15, rtol=0)
        rho, u = oracle.moments(f)
        assert np.allclose(oracle.collide(f, 1.0), oracle.equilibrium(rho, u), atol=1e-16, rtol=0)
    feq = oracle.equilibrium(1.01, (0.02, -0.03, 0.01))
    assert np.allclose(oracle.collide(feq, 1.5), feq, atol=1e-16, rtol=0)


# --------------------------------------------------- stream + bounce-back --
def brute_force_step(f, tau, u_lid, periodic):
    """Independent numpy collide-then-stream on a small box.

    BGK written from the textbook form with numpy over all cells; streaming
    written per axis as explicit slice copies (no index arithmetic shared
    with the oracle's per-cell pull loop); walls by link-wise bounce-back."""
    cs = pa.CVEC
    w = np.array(pa.WGT)
    _, nx, ny, nz = f.shape
    rho = f.sum(axis=0)
    j = np.stack([sum(cs[i][a] * f[i] for i in range(19)) for a in range(3)])
    u = j / rho
    usq = (u * u).sum(axis=0)
    feq = np.empty_like(f)
    for i in range(1, 19):
        cu = cs[i][0] * u[0] + cs[i][1] * u[1] + cs[i][2] * u[2]
        feq[i] = w[i] * rho * (1 + 3 * cu + 4.5 * cu * cu - 1.5 * usq)
    feq[0] = rho - feq[1:].sum(axis=0)
    fs = f - (f - feq) / tau
    out = np.full_like(f, np.nan)

    def shifted(a, d, axis):
        """b[x] = a[x - d] along axis (d in -1, 0, 1); NaN where x - d leaves
        the box (cavity) or wrapped (periodic)."""
        if d == 0:
            return a.copy()
        if periodic:
            return np.roll(a, d, axis=axis)
        b = np.full_like(a, np.nan)
        src = [slice(None)] * 3
        dst = [slice(None)] * 3
        if d == 1:
            dst[axis], src[axis] = slice(1, None), slice(0, -1)
        else:
            dst[axis], src[axis] = slice(0, -1), slice(1, None)
        b[tuple(dst)] = a[tuple(src)]
        return b

    for i in range(19):
        b = fs[i]
        for axis in range(3):
            b = shifted(b, cs[i][axis], axis)
        out[i] = b
    if not periodic:
        for i in range(19):
            o = pa.opp(i)
            miss = np.isnan(out[i])
            out[i][miss] = fs[o][miss]
            if cs[i][2] == -1:  # source beyond the top z face: the moving lid
                top = np.zeros_like(miss)
                top[:, :, nz - 1] = True
                add = 6.0 * w[i] * (cs[i][0] * u_lid[0] + cs[i][1] * u_lid[1] + cs[i][2] * u_lid[2])
                out[i][top] += add
    return out


@pytest.mark.parametrize("dims", [(4, 4, 4), (3, 5, 4), (5, 6, 7)])
@pytest.mark.parametrize("periodic", [False, True])
def test_step_equals_brute_force(dims, periodic):
    f = li.random_populations(3, *dims)
    bc = oracle.BC_PERIODIC if periodic else oracle.BC_CAVITY
    got = oracle.step(f, bc, 0.6, LID)
    ref = brute_force_step(f, 0.6, LID, periodic)
    assert np.max(np.abs(got - ref)) <= 1e-15


@pytest.mark.parametrize("n", [1, 2, 3, 4])
@pytest.mark.parametrize("periodic", [False, True])
def test_run_equals_brute_force_steps(n, periodic):
    """oracle.run (two lattices, collide in place, pull, swap) equals n
    independent brute-force steps, odd and even n."""
    f = li.random_populations(4, 4, 5, 6)
    bc = oracle.BC_PERIODIC if periodic else oracle.BC_CAVITY
    ref = f
    for _ in range(n):
        ref = brute_force_step(ref, 0.6, LID, periodic)
    got = oracle.run(f, bc, 0.6, LID, n)
    assert np.max(np.abs(got - ref)) <= 1e-14 * n


@pytest.mark.parametrize("dims", [(3, 3, 3), (4, 4, 4), (5, 6, 7), (6, 4, 5)])
def test_step_equals_fuse_swap_alg1_bitwise(dims):
    """Alg. 1: Stage I collide+revert on the faces,
    Stage II bulk collide+swap_stream, Stage III boundary_swap_stream --
    identical bits to one oracle step, every link swapped once."""
    f = li.random_populations(5, *dims)
    L = pa.fuse_swap_step(f, 0.6, LID, check=True)
    assert L.violations == []
    assert np.array_equal(L.canonical(), oracle.step(f, oracle.BC_CAVITY, 0.6, LID))
    # link-once: every interior link swapped exactly once
    n_links = sum(L.links(X, Y, Z) for X in range(1, dims[0] + 1)
                  for Y in range(1, dims[1] + 1) for Z in range(1, dims[2] + 1))
    assert sum(L.swapped.values()) == n_links
    assert max(L.swapped.values()) == 1


def test_step_box_matches_full_step():
    """The sub-box step used for sampled full-size checks reproduces the full
    step on the box core (same arithmetic, only the source set differs)."""
    dims = (9, 8, 7)
    f = li.random_populations(6, *dims)
    for bc in (oracle.BC_CAVITY, oracle.BC_PERIODIC):
        full = oracle.step(f, bc, 0.6, LID)
        for origin, size in [((0, 0, 0), (4, 5, 7)), ((3, 2, 1), (5, 6, 6)), ((5, 3, 0), (4, 5, 7))]:
            box = f[:, origin[0]:origin[0] + size[0], origin[1]:origin[1] + size[1], origin[2]:origin[2] + size[2]]
            got = oracle.step_box(box, dims, origin, bc, 0.6, LID)
            ref = full[:, origin[0]:origin[0] + size[0], origin[1]:origin[1] + size[1], origin[2]:origin[2] + size[2]]
            known = ~np.isnan(got)
            assert np.array_equal(got[known], ref[known])
            # the core one cell in from every non-domain face is fully known
            core = [slice(1 if o > 0 else 0, s - (1 if o + s < n else 0)) for o, s, n in zip(origin, size, dims)]
            if bc == oracle.BC_PERIODIC:
                core = [slice(1, s - 1) if s < n else slice(None) for s, n in zip(size, dims)]
            assert known[(slice(None),) + tuple(core)].all()
    full = oracle.step(f, oracle.BC_CAVITY, 0.6, LID)
    assert np.array_equal(oracle.step_box(f, dims, (0, 0, 0), oracle.BC_CAVITY, 0.6, LID), full)


# -------------------------------------------------------------------- lid --
def test_lid_one_step_closed_form(golden_dir):
    nx, ny, nz = 5, 4, 6
    f = oracle.init_equilibrium(nx, ny, nz)
    _, w, _ = oracle.d3q19()
    g = oracle.step(f, oracle.BC_CAVITY, 0.6, LID)
    expected = {int(r[0]): float(r[1]) for r in read_table(golden_dir, "lid_one_step.txt")}
    for i in range(19):
        top = g[i, :, :, nz - 1]
        rest = g[i, :, :, :nz - 1]
        if i in expected:
            assert np.allclose(top, expected[i], atol=4e-16, rtol=0)  # including lid edges/corners
        else:
            assert np.allclose(top, w[i], atol=4e-16, rtol=0)
        assert np.allclose(rest, w[i], atol=4e-16, rtol=0)


def test_rest_state_invariant():
    """rho = 1, u = 0, still lid: a fixed point over 100 steps."""
    f = oracle.init_equilibrium(6, 5, 7)
    g = oracle.run(f, oracle.BC_CAVITY, 0.6, (0.0, 0.0, 0.0), 100)
    assert np.max(np.abs(g - f)) <= 1e-15
    g = oracle.run(f, oracle.BC_PERIODIC, 0.55, (0.0, 0.0, 0.0), 100)
    assert np.max(np.abs(g - f)) <= 1e-15


# ------------------------------------------------------------ conservation --
@pytest.mark.parametrize("tau", [0.55, 0.6])
def test_mass_conserved_cavity(tau):
    """BASELINE.json:5: mass conserved to 1e-13 relative (lid cavity, 1000
    steps; compensated sums).  Needs the rest-population closure (R-2)."""
    cfg = li.CONFIGS[1]
    rho, u = li.init_fields(cfg)
    f = oracle.init_equilibrium(cfg.nx, cfg.ny, cfg.nz, rho, u)
    m0 = math.fsum(f.ravel())
    g = oracle.run(f, cfg.bc, tau, cfg.u_lid, 1000)
    assert abs(math.fsum(g.ravel()) - m0) / m0 <= 1e-13


def test_momentum_conserved_periodic():
    cfg = li.CONFIGS[3].with_dims(8, 8, 8, steps=50)
    rho, u = li.init_fields(cfg)
    f = oracle.init_equilibrium(8, 8, 8, rho, u)
    c, _, _ = oracle.d3q19()
    j0 = [math.fsum((c[:, a, None] * f.reshape(19, -1)).ravel()) for a in range(3)]
    g = oracle.run(f, cfg.bc, cfg.tau, cfg.u_lid, 50)
    j1 = [math.fsum((c[:, a, None] * g.reshape(19, -1)).ravel()) for a in range(3)]
    assert np.max(np.abs(np.array(j1) - np.array(j0))) <= 1e-13


@pytest.mark.parametrize("tau", [0.55, 0.6, 1.0])
def test_shear_wave_viscosity(tau):
    """Textbook closed form: a periodic shear wave u_x = A sin(k y) decays as
    exp(-nu k^2 t), nu = (tau - 1/2)/3 (c_s^2 = 1/3; omega = 1/tau)."""
    nx, ny, nz, A = 2, 64, 2, 1e-4
    k = 2 * np.pi / ny
    y = np.arange(ny)
    u = np.zeros((nx, ny, nz, 3))
    u[:, :, :, 0] = (A * np.sin(k * y))[None, :, None]
    f = oracle.init_equilibrium(nx, ny, nz, np.ones((nx, ny, nz)), u)

    def amp(g):
        _, uu = oracle.macroscopic(g)
        return 2.0 / ny * np.sum(uu[:, :, :, 0].mean(axis=(0, 2)) * np.sin(k * y))

    g1 = oracle.run(f, oracle.BC_PERIODIC, tau, (0, 0, 0), 100)
    g2 = oracle.run(g1, oracle.BC_PERIODIC, tau, (0, 0, 0), 300)
    rate = -math.log(amp(g2) / amp(g1)) / 300
    nu = (tau - 0.5) / 3
    assert abs(rate / (nu * k * k) - 1) < 3e-3


def test_lid_drags_fluid():
    """Physical sanity (adapted to the z-top lid): the mean x
    velocity of the layer under the lid is positive."""
    cfg = li.CONFIGS[1]
    f = oracle.init_equilibrium(16, 16, 16)
    g = oracle.run(f, cfg.bc, cfg.tau, cfg.u_lid, 600)
    _, u = oracle.macroscopic(g)
    assert u[:, :, 15, 0].mean() > 0.01
    assert np.all(np.isfinite(g))


# ------------------------------------------------------- two-step merge --
@pytest.mark.parametrize("dims,tile", [((4, 4, 4), None), ((4, 4, 4), 2), ((5, 6, 7), None),
                                       ((5, 6, 7), 3), ((6, 5, 4), 4), ((4, 16, 16), 4),
                                       ((3, 3, 3), 1)])
def test_two_step_alg2_corrected_bitwise(dims, tile):
    """Alg. 2 with the corrected neighbour handler
    (R-12) equals two oracle steps bit for bit, with no dependency
    violation, for the single-prism order and prism strides."""
    f = li.random_populations(9, *dims)
    L = pa.two_step_cycle(f, 0.6, LID, tile=tile, check=True)
    assert L.violations == []
    assert np.array_equal(L.canonical(), oracle.run(f, oracle.BC_CAVITY, 0.6, LID, 2))


@pytest.mark.parametrize("dims", [(4, 4, 4), (5, 6, 7), (8, 8, 8)])
def test_two_step_alg2_literal_handler_defect(dims):
    """Documents DESIGN.md R-12: the handler condition 2 as printed
     streams one Z-step too early; the dependency checker
    counts exactly (lx-1)(lz-2) violations and the result differs from two
    plain steps."""
    f = li.random_populations(9, *dims)
    L = pa.two_step_cycle(f, 0.6, LID, tile=None, corrected=False, check=True)
    assert len(L.violations) == (dims[0] - 1) * (dims[2] - 2)
    assert np.max(np.abs(L.canonical() - oracle.run(f, oracle.BC_CAVITY, 0.6, LID, 2))) > 1e-4


def test_walkthrough_4x4x4(golden_dir):
    """cell (1,1,1) becomes ready for the second computation
    right after the first computation of (2,2,2)."""
    g = {r[0]: r[1:] for r in read_table(golden_dir, "walkthrough_4x4x4.txt")}
    f = li.random_populations(10, 4, 4, 4)
    L = pa.two_step_cycle(f, 0.6, LID, tile=None)
    first_second = next(k for k, e in enumerate(L.log) if e[0] == "collide" and e[1] == 2)
    assert L.log[first_second][2] == tuple(int(v) for v in g["first_second_step_cell"])
    prev = L.log[first_second - 1]
    assert prev[0] == "stream" and prev[1] == 1
    assert prev[2] == tuple(int(v) for v in g["preceded_by_first_step_cell"])
    n_first = sum(1 for e in L.log[:first_second] if e[0] == "collide" and e[1] == 1)
    assert n_first == int(g["first_steps_before"][0])


def test_prism_example(golden_dir):
    g = {r[0]: int(r[1]) for r in read_table(golden_dir, "prism_4x16x16.txt")}
    lx, ly, lz, tile = g["lx"], g["ly"], g["lz"], g["tile"]
    blocks = list(pa.prism_blocks(lx, ly, lz, tile))
    nonempty = [b for b in blocks if list(pa.prism_cells(lx, ly, lz, tile, b))]
    assert len(blocks) == g["prisms"] and len(nonempty) == g["prisms"]
    cells = list(pa.traversal(lx, ly, lz, tile))
    assert len(cells) == g["cells"] and len(set(cells)) == g["cells"]

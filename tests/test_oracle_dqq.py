"""Pins for the other-lattice oracle (oracle/oracle_dqq.c; D3Q15 and D3Q27,
the lattices PAPER.md:215 names next to D3Q19), run without a GPU.

* With the D3Q19 table it is bit-identical to the pinned D3Q19 oracle
  (oracle.c), which pins its stepping, collision and boundary code.
* Its D3Q15 / D3Q27 tables: built independently here from the velocity-set
  definitions (all of {-1,0,1}^3 filtered by |c|^2, textbook weights), then
  the rational isotropy identities of a second-order lattice.
* Equilibrium moments, conservation, the lid's one-step closed form, an
  independent numpy brute-force step, and the shear-wave decay rate
  nu = (tau - 1/2)/3 (textbook closed form) for each lattice.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

import lbm_inputs as li
import oracle

LID = (0.05, 0.0, 0.0)
WEIGHTS = {  # |c|^2 -> weight (textbook D3Q15 / D3Q27)
    15: {0: Fraction(2, 9), 1: Fraction(1, 9), 3: Fraction(1, 72)},
    27: {0: Fraction(8, 27), 1: Fraction(2, 27), 2: Fraction(1, 54), 3: Fraction(1, 216)},
    19: {0: Fraction(1, 3), 1: Fraction(1, 18), 2: Fraction(1, 36)},
}


def textbook(q):
    """{velocity tuple: weight} from the definition of the velocity set."""
    out = {}
    for c in itertools.product((-1, 0, 1), repeat=3):
        n = sum(a * a for a in c)
        if n in WEIGHTS[q]:
            out[c] = WEIGHTS[q][n]
    assert len(out) == q
    return out


@pytest.mark.parametrize("q", [15, 19, 27])
def test_table_is_the_velocity_set(q):
    c, w, opp = oracle.dqq_table(q)
    tb = textbook(q)
    assert sorted(map(tuple, c)) == sorted(tb)
    for i in range(q):
        assert w[i] == float(tb[tuple(c[i])])
        assert tuple(c[opp[i]]) == tuple(-c[i]) and opp[opp[i]] == i
    h = (q - 1) // 2
    assert tuple(c[0]) == (0, 0, 0)
    for i in range(1, h + 1):  # "negative" half first: first nonzero component -1
        assert next(a for a in c[i] if a != 0) == -1 and opp[i] == i + h


@pytest.mark.parametrize("q", [15, 19, 27])
def test_rational_isotropy(q):
    tb = textbook(q)
    d = lambda a, b: 1 if a == b else 0
    assert sum(tb.values()) == 1
    for a in range(3):
        assert sum(w * c[a] for c, w in tb.items()) == 0
        for b in range(3):
            assert sum(w * c[a] * c[b] for c, w in tb.items()) == Fraction(d(a, b), 3)
            for g in range(3):
                assert sum(w * c[a] * c[b] * c[g] for c, w in tb.items()) == 0
                for e in range(3):
                    want = Fraction(d(a, b) * d(g, e) + d(a, g) * d(b, e) + d(a, e) * d(b, g), 9)
                    assert sum(w * c[a] * c[b] * c[g] * c[e] for c, w in tb.items()) == want


def test_d3q19_table_is_spec_order():
    """Q = 19 reproduces SPEC.md:109's order (the D3Q19 oracle's table)."""
    c, w, opp = oracle.dqq_table(19)
    c0, w0, opp0 = oracle.d3q19()
    assert np.array_equal(c, c0) and np.array_equal(w, w0) and np.array_equal(opp, opp0)


@pytest.mark.parametrize("bc", [oracle.BC_CAVITY, oracle.BC_PERIODIC])
def test_generic_stepping_equals_d3q19_oracle_bitwise(bc):
    f = li.random_populations(61, 5, 6, 7)
    assert np.array_equal(oracle.dqq_run(19, f, bc, 0.6, LID, 3), oracle.run(f, bc, 0.6, LID, 3))


@pytest.mark.parametrize("q", [15, 27])
@pytest.mark.parametrize("rho,u", [(1.0, (0.0, 0.0, 0.1)), (0.97, (0.03, -0.02, 0.05))])
def test_equilibrium_moments(q, rho, u):
    c, w, _ = oracle.dqq_table(q)
    feq = oracle.dqq_equilibrium(q, rho, u)
    u = np.array(u)
    assert abs(feq.sum() - rho) <= 1e-15
    assert np.max(np.abs(c.T @ feq - rho * u)) <= 1e-15
    P = np.einsum("i,ia,ib->ab", feq, c, c)
    assert np.max(np.abs(P - rho * (np.outer(u, u) + np.eye(3) / 3))) <= 1e-15


def brute_force_step(q, f, tau, u_lid, periodic):
    """One collide + pull-stream step in whole-array numpy, built from the
    textbook table (not the oracle's arithmetic)."""
    c, _, opp = oracle.dqq_table(q)  # only the ORDER; weights from the textbook
    tb = textbook(q)
    w = np.array([float(tb[tuple(ci)]) for ci in c])
    rho = f.sum(axis=0)
    j = np.einsum("ia,ixyz->axyz", c.astype(float), f)
    u = j / rho
    usq = (u * u).sum(axis=0)
    feq = np.empty_like(f)
    for i in range(1, q):
        cu = c[i, 0] * u[0] + c[i, 1] * u[1] + c[i, 2] * u[2]
        feq[i] = w[i] * rho * (1 + 3 * cu + 4.5 * cu * cu - 1.5 * usq)
    feq[0] = rho - feq[1:].sum(axis=0)
    fs = f - (f - feq) / tau
    _, nx, ny, nz = f.shape
    out = np.empty_like(f)
    X, Y, Z = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    for i in range(q):
        sx, sy, sz = X - c[i, 0], Y - c[i, 1], Z - c[i, 2]
        if periodic:
            out[i] = fs[i][sx % nx, sy % ny, sz % nz]
            continue
        inside = (sx >= 0) & (sx < nx) & (sy >= 0) & (sy < ny) & (sz >= 0) & (sz < nz)
        v = np.where(inside, fs[i][np.clip(sx, 0, nx - 1), np.clip(sy, 0, ny - 1), np.clip(sz, 0, nz - 1)],
                     fs[opp[i]])
        lid = (~inside) & (sz >= nz)
        out[i] = v + lid * 6 * w[i] * (c[i] @ np.array(u_lid))
    return out


@pytest.mark.parametrize("q", [15, 27])
@pytest.mark.parametrize("periodic", [False, True])
def test_step_equals_brute_force(q, periodic):
    f = li.uniform(62, q * 4 * 5 * 6, 0.01, 0.06).reshape(q, 4, 5, 6)
    bc = oracle.BC_PERIODIC if periodic else oracle.BC_CAVITY
    got = oracle.dqq_run(q, f, bc, 0.6, LID, 1)
    assert np.max(np.abs(got - brute_force_step(q, f, 0.6, LID, periodic))) <= 1e-15


@pytest.mark.parametrize("q", [15, 27])
def test_lid_one_step_closed_form(q):
    """From rest (f = w), one step: a top cell's populations pulled from
    beyond the lid are w_i + 6 w_i (c_i . U); every other one stays w_i."""
    c, w, _ = oracle.dqq_table(q)
    n = 4
    f = np.repeat(w[:, None], n ** 3, axis=1).reshape(q, n, n, n)
    g = oracle.dqq_run(q, f, oracle.BC_CAVITY, 0.6, LID, 1)
    for i in range(q):
        top = g[i, 1:-1, 1:-1, n - 1]
        want = w[i] + (6 * w[i] * c[i, 0] * LID[0] if c[i, 2] == -1 else 0.0)
        assert np.max(np.abs(top - want)) <= 1e-15  # a few ulp: the rest population's closure
    assert np.max(np.abs(g[:, :, :, : n - 1] - f[:, :, :, : n - 1])) <= 1e-15


@pytest.mark.parametrize("q", [15, 27])
def test_mass_conserved_cavity(q):
    nx = ny = nz = 8
    rho = 1.0 + li.uniform(63, nx * ny * nz, -1e-3, 1e-3).reshape(nx, ny, nz)
    f = oracle.dqq_init_equilibrium(q, nx, ny, nz, rho)
    m0 = math.fsum(f.ravel())
    g = oracle.dqq_run(q, f, oracle.BC_CAVITY, 0.6, LID, 300)
    assert abs(math.fsum(g.ravel()) - m0) / m0 <= 1e-13
    assert np.all(np.isfinite(g))


@pytest.mark.parametrize("q", [15, 27])
def test_momentum_conserved_periodic(q):
    nx = ny = nz = 6
    u = li.uniform(64, 3 * nx * ny * nz, -0.01, 0.01).reshape(nx, ny, nz, 3)
    f = oracle.dqq_init_equilibrium(q, nx, ny, nz, None, u)
    c, _, _ = oracle.dqq_table(q)
    j0 = np.einsum("ia,ixyz->a", c.astype(float), f)
    g = oracle.dqq_run(q, f, oracle.BC_PERIODIC, 0.55, (0, 0, 0), 50)
    assert np.max(np.abs(np.einsum("ia,ixyz->a", c.astype(float), g) - j0)) <= 1e-13


@pytest.mark.parametrize("q", [15, 27])
@pytest.mark.parametrize("tau", [0.6, 1.0])
def test_shear_wave_viscosity(q, tau):
    """u_x = A sin(2 pi y / L) decays as exp(-nu k^2 t), nu = (tau - 1/2)/3."""
    L, A = 64, 1e-4
    y = np.arange(L)
    u = np.zeros((2, L, 2, 3))
    u[:, :, :, 0] = A * np.sin(2 * np.pi * y / L)[None, :, None]
    f = oracle.dqq_init_equilibrium(q, 2, L, 2, None, u)
    t0, t1 = 50, 250
    c, _, _ = oracle.dqq_table(q)

    def amp(g):
        ux = np.einsum("i,ixyz->xyz", c[:, 0].astype(float), g) / g.sum(axis=0)
        return 2 / L * float(np.sum(ux[0, :, 0] * np.sin(2 * np.pi * y / L)))

    g0 = oracle.dqq_run(q, f, oracle.BC_PERIODIC, tau, (0, 0, 0), t0)
    g1 = oracle.dqq_run(q, g0, oracle.BC_PERIODIC, tau, (0, 0, 0), t1 - t0)
    nu = -math.log(amp(g1) / amp(g0)) / ((2 * np.pi / L) ** 2 * (t1 - t0))
    assert abs(nu / ((tau - 0.5) / 3) - 1) <= 3e-3


@pytest.mark.parametrize("q", [15, 27])
def test_paired_collision_identities(q):
    """R-16's reading (the GPU's paired-direction collision for these
    lattices) rests on identities of the velocity set, checked here in exact
    rational arithmetic on the oracle's own table: the table is closed under
    c -> -c with opp(i) = i + (q-1)/2; within each weight class (|c|^2 = 1,
    2, 3) the half set's sum of (c.u)^2 is k_c u.u with k = 1, 4, 4 for
    every u; so sum_{i>0} feq_i = 2 sum_c w_c rho (n_c (1 - 1.5 u.u) +
    4.5 k_c u.u) equals rho - feq_0 exactly (the closed-form closure)."""
    c, w, _ = oracle.dqq_table(q)
    c = np.asarray(c, dtype=int).reshape(q, 3)
    w = [Fraction(x).limit_denominator(1000) for x in w]
    h = (q - 1) // 2
    for i in range(1, h + 1):
        assert all(c[i + h] == -c[i]) and w[i + h] == w[i]
    rng = np.random.default_rng(16)
    for _ in range(5):
        u = [Fraction(int(v), 997) for v in rng.integers(-60, 60, 3)]
        rho = Fraction(int(rng.integers(900, 1100)), 1000)
        usq = sum(x * x for x in u)
        base = 1 - Fraction(3, 2) * usq
        cu = [sum(int(c[i][a]) * u[a] for a in range(3)) for i in range(q)]
        clos = Fraction(0)
        for n2, k in ((1, 1), (2, 4), (3, 4)):
            half = [i for i in range(1, h + 1) if int(c[i] @ c[i]) == n2]
            if not half:
                continue
            assert sum(cu[i] ** 2 for i in half) == k * usq
            assert len({w[i] for i in half}) == 1
            clos += w[half[0]] * rho * (len(half) * base + Fraction(9, 2) * k * usq)
        feq = [w[i] * rho * (1 + 3 * cu[i] + Fraction(9, 2) * cu[i] ** 2 - Fraction(3, 2) * usq) for i in range(q)]
        assert 2 * clos == sum(feq[1:])
        assert rho - 2 * clos == feq[0]

"""GPU parity of the other lattices (D3Q15, D3Q27: PAPER.md:215; SURVEY.md
8(f) row 4) against their pinned oracle (oracle/oracle_dqq.c), element by
element on the same seeded inputs, through the C-ABI: random off-equilibrium
states on ragged boxes (several z warps and y rows, tails), both boundary
modes, both dtypes, odd and even step counts; a lid-driven cavity from the
BASELINE recipe with its mass; the moments read-back; the direction order.
Tolerances as for D3Q19 (R-3/R-11): 1e-12 (fp64), 1e-5 (fp32)."""
import math

import numpy as np
import pytest

import lbm_inputs as li
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no GPU", allow_module_level=True)

import paper_2208_05429_b200 as lbm  # noqa: E402

TOL = {"f64": 1e-12, "f32": 1e-5}
LID = (0.05, 0.0, 0.0)


def relerr_floor(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0 / 216.0)))


@pytest.mark.parametrize("q", [15, 27])
@pytest.mark.parametrize("dims", [(5, 6, 7), (9, 17, 40), (4, 1, 33), (3, 9, 64)])
@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_random_states_match_oracle(q, dims, bc, dtype):
    f0 = li.uniform(70 + q, q * int(np.prod(dims)), 0.01, 0.06).reshape(q, *dims)
    with lbm.Lattice(*dims, 0.6, LID, dtype, bc=bc, lattice=q) as lat:
        lat.set_populations(f0)
        assert relerr_floor(lat.populations(), f0) <= TOL[dtype]
        ref = f0
        for n in (1, 2, 3):
            lat.step(n)
            ref = oracle.dqq_run(q, ref, bc, 0.6, LID, n)
            got = lat.populations()
            assert relerr_floor(got, ref) <= TOL[dtype], (n,)
        box = lat.populations_box(1, 0, 2, dims[0] - 2, dims[1], dims[2] - 3)
        assert np.array_equal(box, got[:, 1:dims[0] - 1, :, 2:dims[2] - 1])


@pytest.mark.parametrize("q", [15, 27])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_lid_cavity_recipe(q, dtype):
    """16^3 lid-driven cavity, rho = 1 + U(+-1e-3) (config 1's recipe), 40
    steps: every population, the moments, and the mass."""
    cfg = li.CONFIGS[1]
    rho, _ = li.init_fields(cfg)
    ref = oracle.dqq_run(q, oracle.dqq_init_equilibrium(q, 16, 16, 16, rho), cfg.bc, cfg.tau, cfg.u_lid, 40)
    with lbm.Lattice(16, 16, 16, cfg.tau, cfg.u_lid, dtype, bc=cfg.bc, lattice=q) as lat:
        lat.init_equilibrium(rho, None)
        m0 = math.fsum(lat.populations().ravel())
        lat.step(40)
        got = lat.populations()
        r, u = lat.macroscopic()
    assert float(np.max(np.abs(got - ref) / np.abs(ref))) <= TOL[dtype]
    c, _ = lbm.lbm_lattice_table(q)
    r_ref = ref.sum(axis=0)
    u_ref = np.einsum("ia,ixyz->xyza", c.astype(float), ref) / r_ref[..., None]
    assert np.max(np.abs(r - r_ref)) <= 10 * TOL[dtype] and np.max(np.abs(u - u_ref)) <= 10 * TOL[dtype]
    assert abs(math.fsum(got.ravel()) - m0) / m0 <= (1e-13 if dtype == "f64" else 1e-6)

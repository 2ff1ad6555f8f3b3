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


@pytest.mark.parametrize("q", [15, 27])
@pytest.mark.parametrize("dims", [(70, 21, 45), (3, 5, 7), (33, 9, 100), (2, 17, 33), (6, 40, 64)])
@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_two_step_sweep_bitwise(q, dims, bc, dtype):
    """K2Q (two collide + push steps per HBM pass, the paper's merge for these
    lattices) equals two one-step launches bit for
    bit: ragged tiles in y and z, several x chunks, one-plane and one-row
    lattices, walls and wraps, odd step counts (a one-step remainder)."""
    f0 = li.uniform(90 + q, q * int(np.prod(dims)), 0.01, 0.06).reshape(q, *dims)
    outs = []
    for kern in (lbm.LBM_KERNEL_K1, lbm.LBM_KERNEL_K2):
        with lbm.Lattice(*dims, 0.6, LID, dtype, bc=bc, lattice=q, kernel=kern) as lat:
            lat.set_populations(f0)
            lat.step(4)
            a = lat.populations()
            lat.step(3)
            outs.append((a, lat.populations(), lbm.lbm_get_stats(lat.ctx).k2_launches))
    assert outs[0][2] == 0 and outs[1][2] == 3
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("q", [15, 27])
@pytest.mark.parametrize("tau,lid", [(0.6, LID), (0.9, (0.03, -0.02, 0.0)), (0.51, (0.0, 0.04, 0.0))])
def test_two_step_sweep_cavity_vs_oracle(q, tau, lid):
    """A 40 x 24 x 48 lid cavity (several tiles and x chunks) in fp64 through
    K2Q sweeps against the oracle after 10 steps, element by element, for
    three relaxation times and lids along x, y and the xy diagonal; AUTO
    takes the same sweeps."""
    dims = (40, 24, 48)
    rho = 1.0 + li.uniform(5, int(np.prod(dims)), -1e-3, 1e-3).reshape(dims)
    ref = oracle.dqq_run(q, oracle.dqq_init_equilibrium(q, *dims, rho), lbm.LBM_BC_CAVITY, tau, lid, 10)
    with lbm.Lattice(*dims, tau, lid, "f64", lattice=q, kernel=lbm.LBM_KERNEL_K2) as lat:
        lat.init_equilibrium(rho, None)
        lat.step(10)
        got = lat.populations()
        assert lbm.lbm_get_stats(lat.ctx).k2_launches == 5
    assert float(np.max(np.abs(got - ref) / np.abs(ref))) <= TOL["f64"]
    with lbm.Lattice(*dims, tau, lid, "f64", lattice=q) as lat:
        lat.init_equilibrium(rho, None)
        lat.step(10)
        assert lbm.lbm_get_stats(lat.ctx).k2_launches == 5
        assert np.array_equal(lat.populations(), got)


def test_two_step_sweep_full_size_boxes_bitwise():
    """D3Q27 fp64 on config 5's 1024 x 512 x 512 cavity (116 GB for two
    copies: 64-bit slot offsets, 4D TMA coordinates, the x-chunk planner at
    full size): 4 steps through K2Q equal 4 one-step launches bit for bit on
    boxes at the corners, the lid, x-chunk seams and the interior."""
    nx, ny, nz = 1024, 512, 512
    rho = 1.0 + li.uniform(4, nx * ny * nz, -1e-3, 1e-3).reshape(nx, ny, nz)
    boxes = [(0, 0, 0), (1021, 509, 508), (31, 255, 508), (511, 7, 250), (992, 500, 0)]
    got = {}
    for kern in (lbm.LBM_KERNEL_K2, lbm.LBM_KERNEL_K1):
        with lbm.Lattice(nx, ny, nz, 0.6, LID, "f64", lattice=27, kernel=kern) as lat:
            lat.init_equilibrium(rho, None)
            lat.step(4)
            got[kern] = [lat.populations_box(x, y, z, 3, 3, 4) for (x, y, z) in boxes]
    for a, b in zip(got[lbm.LBM_KERNEL_K2], got[lbm.LBM_KERNEL_K1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("q", [15, 27])
@pytest.mark.parametrize("dims,bc", [((1, 9, 40), lbm.LBM_BC_CAVITY), ((5, 1, 33), lbm.LBM_BC_CAVITY),
                                     ((4, 7, 1), lbm.LBM_BC_CAVITY), ((2, 1, 40), lbm.LBM_BC_PERIODIC),
                                     ((3, 9, 1), lbm.LBM_BC_PERIODIC), ((33, 2, 2), lbm.LBM_BC_PERIODIC)])
def test_two_step_sweep_degenerate_extents(q, dims, bc):
    """K2Q on one-plane, one-row and one-column lattices (every link of a
    one-cell extent bounces, or wraps onto the cell itself): bitwise equal to
    the one-step kernel and within 1e-12 of the oracle after 4 steps."""
    f0 = li.uniform(120 + q, q * int(np.prod(dims)), 0.01, 0.06).reshape(q, *dims)
    outs = []
    for kern in (lbm.LBM_KERNEL_K1, lbm.LBM_KERNEL_K2):
        with lbm.Lattice(*dims, 0.6, LID, "f64", bc=bc, lattice=q, kernel=kern) as lat:
            lat.set_populations(f0)
            lat.step(4)
            outs.append(lat.populations())
    assert np.array_equal(outs[0], outs[1])
    ref = oracle.dqq_run(q, f0, bc, 0.6, LID, 4)
    assert relerr_floor(outs[1], ref) <= TOL["f64"]


@pytest.mark.parametrize("q", [15, 27])
@pytest.mark.parametrize("bc", [lbm.LBM_BC_PERIODIC, lbm.LBM_BC_CAVITY])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_nccl_xslab_world1_bitwise(q, bc, dtype):
    """D3Q15/27 over NCCL x-slabs (csrc/api.cu dqq_exchange; PAPER.md:336,
    589-590) on hardware: a one-rank periodic communicator pushes the links
    that leave the slab in x into its ghost planes and sends them to itself
    (ncclSend/ncclRecv to self in one group) instead of wrapping in the
    kernel; a one-rank cavity has walls on both faces.  One-step kernel,
    odd and even step counts, set_populations / init / read-backs: bitwise
    equal to the single-process context (whose K2Q two-step sweep equals the
    one-step kernel bit for bit), and to the oracle."""
    dims = (9, 6, 40)
    f0 = li.uniform(90 + q, q * int(np.prod(dims)), 0.01, 0.06).reshape(q, *dims)
    rho0 = li.uniform(91 + q, int(np.prod(dims)), 0.99, 1.01).reshape(dims)
    try:
        lbm.lbm_nccl_unique_id()
    except lbm.LbmError as e:  # pragma: no cover
        pytest.skip(f"NCCL unavailable: {e}")
    outs = []
    for kw in ({}, {"comm": lbm.LBM_COMM_NCCL, "nccl_id": lbm.lbm_nccl_unique_id()}):
        with lbm.Lattice(*dims, 0.6, LID, dtype, bc=bc, lattice=q, **kw) as lat:
            lat.set_populations(f0)
            lat.step(3)
            lat.step(2)
            a = lat.populations()
            rho, u = lat.macroscopic()
            lat.init_equilibrium(rho0, None)
            lat.step(4)
            outs.append((a, rho, u, lat.populations(), lat.populations_box(2, 1, 3, 5, 4, 30)))
    for x, y in zip(*outs):
        assert np.array_equal(x, y)
    assert relerr_floor(outs[1][0], oracle.dqq_run(q, f0, bc, 0.6, LID, 5)) <= TOL[dtype]

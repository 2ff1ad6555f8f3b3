"""GPU parity at the CONFIGURED step count (BASELINE.json:5: "GPU results
must match the oracle ... after the configured step count"; PAPER.md:832-837
verifies a solver by comparing the final fields).

* Config 3 (256^3 periodic, 200 steps) runs LIVE: the oracle (oracle/,
  16 host threads, a few minutes) computes the whole final state once and
  every population of every cell is compared.
* Configs 4 and 5 (512^3 and 1024x512x512 cavities, 100 steps) compare with
  sampled oracle states stored by tools/make_oracle_golden.py (which calls only
  oracle/ and lbm_inputs; tests/golden/cfgN_oracle_tS.npz): 64 boxes of 4^3
  cells x 19 populations (the 8 domain corners, 12 edge midpoints, 6 face
  centres, x-chunk seams with y%8 / z%32 tile seams, seeded interior points),
  three full lines through the domain, and per-x-plane mass and momentum.

Tolerances (BASELINE.json:5, R-3/R-11): max |f_gpu - f_ora| / |f_ora|
<= 1e-12 (fp64) / 1e-5 (fp32) on every compared population.  Plane sums:
each population within rel. tol and f > 0 imply |sum_cells sum_i c_i df_i|
<= tol * sum_cells sum_i f_i = tol * (plane mass), for the mass (c = 1) and
every momentum component (|c_a| <= 1).
"""
import os

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
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KERNELS = {"auto": lbm.LBM_KERNEL_AUTO, "k2sc": lbm.LBM_KERNEL_K2_SC, "aa": lbm.LBM_KERNEL_AA,
           "k3": lbm.LBM_KERNEL_K3}


def relerr(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


def plane_sums(lat, nx, ny, nz, chunk=64):
    """Per-x-plane sums of rho and rho*u of the library's moments."""
    rho, u = lat.macroscopic()
    mass = np.empty(nx)
    mom = np.empty((nx, 3))
    for x0 in range(0, nx, chunk):
        r = rho[x0:x0 + chunk]
        mass[x0:x0 + chunk] = r.sum(axis=(1, 2))
        mom[x0:x0 + chunk] = (r[..., None] * u[x0:x0 + chunk]).sum(axis=(1, 2))
    return mass, mom


# ------------------------------------------------------------ config 3 ----
@pytest.fixture(scope="module")
def cfg3_oracle():
    cfg = li.CONFIGS[3]
    oracle.set_threads(os.cpu_count() or 1)
    rho, u = li.init_fields(cfg)
    f = oracle.init_equilibrium(cfg.nx, cfg.ny, cfg.nz, rho, u)
    oracle.run_inplace(f, cfg.bc, cfg.tau, cfg.u_lid, cfg.steps)
    return rho, u, f


@pytest.mark.parametrize("dtype,kernel", [("f64", "auto"), ("f32", "auto"), ("f64", "k2sc"), ("f32", "k3")])
def test_config3_live_full_state(cfg3_oracle, dtype, kernel):
    """BASELINE.json:9: 256^3 periodic, 200 steps (the bench launch
    configuration: K2 sweeps with the fused periodic halo; also the
    single-copy ring and the three-step prototype K3), every population
    of every cell against the live oracle; the golden file written by
    tools/make_oracle_golden.py from the same oracle is bit-identical to it."""
    cfg = li.CONFIGS[3]
    rho, u, ref = cfg3_oracle
    with lbm.Lattice(cfg.nx, cfg.ny, cfg.nz, cfg.tau, cfg.u_lid, dtype, bc=cfg.bc, kernel=KERNELS[kernel]) as lat:
        lat.init_equilibrium(rho, u)
        lat.step(cfg.steps)
        assert lat.time == cfg.steps
        got = lat.populations()
        st = lbm.lbm_get_stats(lat.ctx)
        # multi-step sweeps: 100 two-step (K2), or 66 three-step + one two-step (K3)
        assert st.k2_launches == (cfg.steps // 3 + 1 if kernel == "k3" else cfg.steps // 2)
    assert relerr(got, ref) <= TOL[dtype]
    # momentum of the periodic box: conserved (oracle pin) and equal
    j_ref = np.array([np.sum(ref[i]) for i in range(19)])
    j_got = np.array([np.sum(got[i]) for i in range(19)])
    assert np.max(np.abs(j_got - j_ref)) <= TOL[dtype] * np.sum(j_ref)
    path = os.path.join(GOLDEN, "cfg3_oracle_t200.npz")
    if kernel == "auto" and dtype == "f64" and os.path.exists(path):
        d = np.load(path)
        bx, by, bz = (int(v) for v in d["box"])
        for (x, y, z), b in zip(d["origins"], d["boxes"]):
            assert np.array_equal(b, ref[:, x:x + bx, y:y + by, z:z + bz])


# -------------------------------------------------------- configs 4, 5 ----
def _golden(cfg_id):
    cfg = li.CONFIGS[cfg_id]
    path = os.path.join(GOLDEN, f"cfg{cfg_id}_oracle_t{cfg.steps}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing {path}: run tools/make_oracle_golden.py --config {cfg_id}")
    d = np.load(path)
    assert int(d["steps"]) == cfg.steps and list(d["dims"]) == [cfg.nx, cfg.ny, cfg.nz]
    return cfg, d


@pytest.mark.parametrize("cfg_id,dtype,kernel", [(4, "f64", "auto"), (4, "f32", "auto"),
                                                 (4, "f64", "k2sc"), (4, "f64", "aa"),
                                                 (5, "f64", "auto"), (5, "f32", "auto"),
                                                 (5, "f64", "k2sc"), (5, "f32", "k2sc"),
                                                 (5, "f64", "aa"), (5, "f32", "aa")])
def test_golden_configured_steps(cfg_id, dtype, kernel):
    """BASELINE.json:10-11 at full size, in the bench launch configuration,
    after the configured 100 steps: every stored population of the oracle's
    final state (boxes and lines), and the per-plane mass and momentum."""
    cfg, d = _golden(cfg_id)
    rho, _ = li.init_fields(cfg)
    tol = TOL[dtype]
    with lbm.Lattice(cfg.nx, cfg.ny, cfg.nz, cfg.tau, cfg.u_lid, dtype, bc=cfg.bc, kernel=KERNELS[kernel]) as lat:
        lat.init_equilibrium(rho, None)  # u = 0 for the cavity recipe (include/lbm.h: NULL is u = 0)
        del rho
        lat.step(cfg.steps)
        assert lat.time == cfg.steps
        bx, by, bz = (int(v) for v in d["box"])
        for (x, y, z), want in zip(d["origins"], d["boxes"]):
            got = lat.populations_box(int(x), int(y), int(z), bx, by, bz)
            assert relerr(got, want) <= tol, (cfg.name, kernel, (x, y, z))
        (ly, lz), (mx, mz), (nx_, ny_) = (tuple(int(v) for v in r) for r in d["line_coords"])
        lines = [(lat.populations_box(0, ly, lz, cfg.nx, 1, 1).reshape(19, cfg.nx), d["line_x"]),
                 (lat.populations_box(mx, 0, mz, 1, cfg.ny, 1).reshape(19, cfg.ny), d["line_y"]),
                 (lat.populations_box(nx_, ny_, 0, 1, 1, cfg.nz).reshape(19, cfg.nz), d["line_z"])]
        for got, want in lines:
            assert relerr(got, want) <= tol, (cfg.name, kernel, "line")
        mass, mom = plane_sums(lat, cfg.nx, cfg.ny, cfg.nz)
    bound = tol * d["plane_mass"] * 1.01
    assert np.all(np.abs(mass - d["plane_mass"]) <= bound)
    assert np.all(np.abs(mom - d["plane_mom"]) <= bound[:, None])
    # the cavity conserves mass (BASELINE.json:5): the oracle's, and the GPU's
    m0 = float(np.sum(li.init_fields(cfg)[0], dtype=np.float64))
    assert abs(float(np.sum(d["plane_mass"])) - m0) / m0 <= 1e-13
    assert abs(float(np.sum(mass)) - m0) / m0 <= (1e-13 if dtype == "f64" else 1e-6)

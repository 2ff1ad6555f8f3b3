"""GPU parity of the single-copy two-step storage (LBM_KERNEL_K2_SC): the K2
sweep run in place on a ring of nx + 4 + G planes (include/lbm.h; DESIGN.md
section 11).  Its arithmetic is K2's and K1's, so every read-back equals the
two-buffer path bit for bit -- after any split of the step count (odd
remainders run the in-place K1), through as many ring wrap-arounds as the
steps make, from every initialisation path -- and matches the oracle."""
import numpy as np
import pytest

import lbm_inputs as li
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no GPU", allow_module_level=True)

import paper_2208_05429_b200 as lbm  # noqa: E402

LID = (0.05, 0.0, 0.0)
TOL = {"f64": 1e-12, "f32": 1e-5}
SC = lbm.LBM_KERNEL_K2_SC


def relerr_floor(a, b):
    """as in test_gpu_parity.py: denominators floored at 1/36 (R-11)"""
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0 / 36.0)))


# one plane; ragged tiles; several x chunks (32 fp64 / 48 fp32 planes each),
# so CTAs of later chunks wait on the ticket counters of earlier ones
SC_DIMS = [(1, 8, 32), (3, 9, 33), (5, 17, 31), (40, 12, 40), (130, 9, 20), (200, 16, 32)]


@pytest.mark.parametrize("dims", SC_DIMS)
@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_single_copy_equals_two_buffer(dims, bc, dtype):
    if bc == lbm.LBM_BC_PERIODIC and dims[0] < 2:
        pytest.skip("periodic needs >= 2 planes")
    lid = LID if bc == lbm.LBM_BC_CAVITY else (0.0, 0.0, 0.0)
    f0 = li.random_populations(71, *dims)
    with lbm.Lattice(*dims, 0.6, lid, dtype, bc=bc) as ref, \
            lbm.Lattice(*dims, 0.6, lid, dtype, bc=bc, kernel=SC) as sc:
        ref.set_populations(f0)
        sc.set_populations(f0)
        assert np.array_equal(sc.populations(), ref.populations())
        total = 0
        # 18 steps: odd and even splits, > 1 trip round the ring for every size
        for n in (1, 2, 3, 2, 5, 4, 1):
            ref.step(n)
            sc.step(n)
            total += n
            assert sc.time == ref.time == total
            assert np.array_equal(sc.populations(), ref.populations()), n
            r1, u1 = ref.macroscopic()
            r2, u2 = sc.macroscopic()
            assert np.array_equal(r1, r2) and np.array_equal(u1, u2)
        x0 = max(0, dims[0] // 2 - 2)
        box = (x0, 1 % dims[1], 3 % dims[2], min(3, dims[0] - x0), dims[1] - 1 % dims[1], dims[2] - 3 % dims[2])
        assert np.array_equal(sc.populations_box(*box), ref.populations_box(*box))
        got = sc.populations()
        st = lbm.lbm_get_stats(sc.ctx)
        assert st.k2_launches >= 1 and st.k1_launches >= 1
    if dims[0] * dims[1] * dims[2] <= 20000:
        assert relerr_floor(got, oracle.run(f0, bc, 0.6, lid, total)) <= TOL[dtype]


@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_single_copy_chunked_host_transfers(bc, dtype, monkeypatch):
    """Host init / set / read-back through a staging buffer of 3 planes (the
    LBM_STAGE_BYTES test knob): init_equilibrium stages x windows of 12
    planes plus their x halo, set_populations windows of one plane plus halo
    (wrapping around x when periodic); both give the two-buffer bits, as do
    device-pointer inputs."""
    cfg = li.CONFIGS[2] if bc == lbm.LBM_BC_CAVITY else li.CONFIGS[3]
    dims = (37, 24, 40)
    n = dims[0] * dims[1] * dims[2]
    cfg_rho = (1.0 + li.uniform(81, n, -1e-3, 1e-3)).reshape(dims)
    cfg_u = li.uniform(82, 3 * n, -0.01, 0.01).reshape(*dims, 3)
    f0 = li.random_populations(73, *dims)
    outs = {}
    for kernel in (lbm.LBM_KERNEL_AUTO, SC):
        if kernel == SC:
            monkeypatch.setenv("LBM_STAGE_BYTES", "1")
        with lbm.Lattice(*dims, cfg.tau, cfg.u_lid, dtype, bc=bc, kernel=kernel) as lat:
            lat.init_equilibrium(cfg_rho, cfg_u)
            a = lat.populations()
            lat.step(7)
            b = (lat.populations(), *lat.macroscopic())
            lat.set_populations(f0)
            c = lat.populations()
            lat.step(4)
            d = lat.populations()
            lbm.lbm_init_equilibrium_device(lat.ctx, torch.from_numpy(cfg_rho).cuda(), torch.from_numpy(cfg_u).cuda())
            lat.step(3)
            e = lat.populations()
        outs[kernel] = (a, *b, c, d, e)
        monkeypatch.delenv("LBM_STAGE_BYTES", raising=False)
    for x, y in zip(outs[lbm.LBM_KERNEL_AUTO], outs[SC]):
        assert np.array_equal(x, y)
    # set then read back: f itself (periodic), or to rounding at the lid
    # cells (the pull storage holds f - lid there and adds it back on read)
    want_c = f0 if dtype == "f64" else f0.astype(np.float32).astype(np.float64)
    if bc == lbm.LBM_BC_PERIODIC:
        assert np.array_equal(outs[SC][4], want_c)
    else:
        assert relerr_floor(outs[SC][4], want_c) <= (1e-15 if dtype == "f64" else 1e-7)


def test_single_copy_memory():
    """The ring holds one lattice copy plus G planes and a staging buffer:
    well under the two-buffer footprint."""
    dims = (512, 128, 128)
    used = {}
    for kernel in (lbm.LBM_KERNEL_AUTO, SC):
        torch.cuda.synchronize()
        free0, _ = torch.cuda.mem_get_info()
        with lbm.Lattice(*dims, 0.6, LID, "f64", kernel=kernel) as lat:
            lat.init_equilibrium()
            lat.step(2)
            lbm.lbm_synchronize(lat.ctx)
            free1, _ = torch.cuda.mem_get_info()
        used[kernel] = free0 - free1
    lattice = (dims[0] + 4) * 19 * dims[1] * dims[2] * 8
    assert used[lbm.LBM_KERNEL_AUTO] >= 2 * lattice
    assert used[SC] <= 1.25 * lattice, used


@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("slabs", [2, 4])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_single_copy_x_slabs_bitwise(bc, slabs, dtype, monkeypatch):
    """K2_SC over X-slabs (LOCAL transport: each slab its own ring, halo
    parts copied through the ring mapping; init and set_populations as the
    canonical state plus an in-place inverse stream) equals the single-slab
    two-buffer run bit for bit after every split, for host and device
    initialisation and a chunked staging buffer."""
    dims = (48, 12, 40)
    lid = LID if bc == lbm.LBM_BC_CAVITY else (0.0, 0.0, 0.0)
    f0 = li.random_populations(77, *dims)
    n = dims[0] * dims[1] * dims[2]
    rho = (1.0 + li.uniform(83, n, -1e-3, 1e-3)).reshape(dims)
    u = li.uniform(84, 3 * n, -0.01, 0.01).reshape(*dims, 3)
    runs = []
    for kernel, kw in ((lbm.LBM_KERNEL_AUTO, {}), (SC, dict(comm=lbm.LBM_COMM_LOCAL, local_slabs=slabs))):
        if kernel == SC:
            monkeypatch.setenv("LBM_STAGE_BYTES", "1")
        with lbm.Lattice(*dims, 0.6, lid, dtype, bc=bc, kernel=kernel, **kw) as lat:
            out = []
            lat.set_populations(f0)
            out.append(lat.populations())
            for k in (3, 2, 5):
                lat.step(k)
                out.append(lat.populations())
                out.extend(lat.macroscopic())
            lat.init_equilibrium(rho, u)
            lat.step(4)
            out.append(lat.populations())
            lbm.lbm_init_equilibrium_device(lat.ctx, torch.from_numpy(rho).cuda(), torch.from_numpy(u).cuda())
            lat.step(1)
            out.append(lat.populations())
            runs.append(out)
        monkeypatch.delenv("LBM_STAGE_BYTES", raising=False)
    for a, b in zip(*runs):
        assert np.array_equal(a, b)


def test_single_copy_randomised_bitwise():
    """Seeded random small lattices, tau, lid, dtype and step splits: K2_SC
    equals K1 bit for bit (and K1 the oracle, test_gpu_parity.py)."""
    rng = np.random.default_rng(5429)
    for trial in range(16):
        bc = int(rng.integers(0, 2))
        dims = (int(rng.integers(2, 70)), int(rng.integers(1, 19)), int(rng.integers(1, 45)))
        dtype = str(rng.choice(["f64", "f32"]))
        lid = (float(rng.uniform(-0.05, 0.05)), float(rng.uniform(-0.05, 0.05)), 0.0)
        splits = [int(v) for v in rng.integers(0, 6, size=int(rng.integers(1, 5)))]
        tau = float(rng.uniform(0.52, 1.5))
        f0 = li.random_populations(300 + trial, *dims)
        res = []
        for kernel in (lbm.LBM_KERNEL_K1, SC):
            with lbm.Lattice(*dims, tau, lid, dtype, bc=bc, kernel=kernel) as lat:
                lat.set_populations(f0)
                for n in splits:
                    lat.step(n)
                res.append(lat.populations())
        assert np.array_equal(res[0], res[1]), (dims, bc, dtype, splits, tau)


@pytest.mark.parametrize("kernel", [lbm.LBM_KERNEL_AUTO, lbm.LBM_KERNEL_AA, SC])
def test_degenerate_and_diverged_moments_are_reported(kernel):
    """lbm_macroscopic never divides silently: a cell whose
    populations sum to zero gives LBM_ENUMERIC ("degenerate"), a state whose
    moments overflow gives LBM_ENUMERIC ("non-finite"); the arrays are still
    written and the context stays usable.  Every storage (K2 pull, AA, ring)."""
    dims = (4, 6, 8)
    f0 = li.random_populations(91, *dims)
    f0[:, 2, 3, 4] = 0.0
    with lbm.Lattice(*dims, 0.6, (0.0, 0.0, 0.0), "f64", bc=lbm.LBM_BC_PERIODIC, kernel=kernel) as lat:
        lat.set_populations(f0)
        with pytest.raises(lbm.LbmError, match="degenerate") as e:
            lat.macroscopic()
        assert e.value.status == lbm.LBM_ENUMERIC
        assert np.array_equal(lat.populations(), f0)
        f1 = li.random_populations(92, *dims)
        lat.set_populations(f1)
        rho, u = lat.macroscopic()
        assert np.all(np.isfinite(u)) and np.allclose(rho, f1.sum(axis=0), rtol=1e-14)
        f1[:, 1, 1, 1] = 1e308
        lat.set_populations(f1)
        with pytest.raises(lbm.LbmError, match="non-finite") as e:
            lat.macroscopic()
        assert e.value.status == lbm.LBM_ENUMERIC


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_single_copy_full_size_soak_bitwise(dtype):
    """Config 5 at full size (1024x512x512): 201 steps (100 in-place K2
    sweeps, each with 32 chunks of 1024 tile CTAs ordered by tickets, plus an
    in-place K1 step) on the ring give the two-buffer K2 run's moments and
    sampled populations bit for bit -- the chunk-order waits under full
    machine load, many trips round the ring."""
    cfg = li.CONFIGS[5]
    rho0, u0 = li.init_fields(cfg)
    dims = (cfg.nx, cfg.ny, cfg.nz)
    boxes = [(0, 0, 0, 3, 40, 64), (511, 250, 200, 4, 16, 70), (1020, 480, 448, 4, 32, 64)]
    outs = []
    for kernel in (lbm.LBM_KERNEL_AUTO, SC):
        with lbm.Lattice(*dims, cfg.tau, cfg.u_lid, dtype, bc=cfg.bc, kernel=kernel) as lat:
            lat.init_equilibrium(rho0, u0)
            lat.step(201)
            r, u = lat.macroscopic()
            outs.append((r, u, [lat.populations_box(*b) for b in boxes]))
    (r1, u1, p1), (r2, u2, p2) = outs
    assert np.array_equal(r1, r2) and np.array_equal(u1, u2)
    for a, b in zip(p1, p2):
        assert np.array_equal(a, b)
    assert np.all(np.isfinite(u2))


def test_auto_switches_to_single_copy_when_two_copies_do_not_fit(monkeypatch):
    """AUTO with a device that cannot hold two lattice copies but can hold
    the ring (LBM_MEM_LIMIT_BYTES caps the free memory it considers): the
    context takes the single-copy storage -- about half the memory -- and
    gives the two-buffer bits."""
    dims = (1024, 64, 64)  # two copies 1.28 GB; the ring + staging 0.75 GB
    f0 = li.random_populations(97, *dims)
    outs, used = [], []
    for limit in (None, "1200000000"):
        if limit:
            monkeypatch.setenv("LBM_MEM_LIMIT_BYTES", limit)
        torch.cuda.synchronize()
        free0, _ = torch.cuda.mem_get_info()
        with lbm.Lattice(*dims, 0.6, LID, "f64") as lat:
            free1, _ = torch.cuda.mem_get_info()
            lat.set_populations(f0)
            lat.step(5)
            outs.append(lat.populations())
        used.append(free0 - free1)
        monkeypatch.delenv("LBM_MEM_LIMIT_BYTES", raising=False)
    assert np.array_equal(outs[0], outs[1])
    assert used[0] > 1.2e9 and used[1] < 0.85e9, used

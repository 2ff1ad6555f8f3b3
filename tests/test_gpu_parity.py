"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on
the same seeded inputs, element by element.  Tolerances (BASELINE.json:5,
DESIGN.md R-11): max |f_gpu - f_oracle| / |f_oracle| <= 1e-12 (fp64),
<= 1e-5 (fp32); bitwise equality where the arithmetic is identical (K1 vs K2,
step splitting, slab partitions)."""
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


def relerr(a, b):
    """max |a - b| / |b| over every population (BASELINE.json:5)."""
    return float(np.max(np.abs(a - b) / np.abs(b)))


def relerr_floor(a, b):
    """Off-equilibrium random states (not BASELINE workloads): the rounding
    error of a BGK update is absolute, of order eps * rho, whatever f_i is,
    so the denominator is floored at the smallest lattice weight 1/36
    (R-11)."""
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0 / 36.0)))


def oracle_from_fields(cfg, n):
    rho, u = li.init_fields(cfg)
    f0 = oracle.init_equilibrium(cfg.nx, cfg.ny, cfg.nz, rho, u)
    return rho, u, f0, oracle.run(f0, cfg.bc, cfg.tau, cfg.u_lid, n)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_config1_full(dtype):
    cfg = li.CONFIGS[1]
    rho, u, f0, ref = oracle_from_fields(cfg, cfg.steps)
    with lbm.Lattice(cfg.nx, cfg.ny, cfg.nz, cfg.tau, cfg.u_lid, dtype, bc=cfg.bc) as lat:
        lat.init_equilibrium(rho, u)
        g0 = lat.populations()
        assert relerr(g0, f0) <= TOL[dtype]
        lat.step(cfg.steps)
        assert lat.time == cfg.steps
        got = lat.populations()
        r, uu = lat.macroscopic()
    assert relerr(got, ref) <= TOL[dtype]
    rr, ur = oracle.macroscopic(ref)
    assert np.max(np.abs(r - rr)) <= 10 * TOL[dtype]
    assert np.max(np.abs(uu - ur)) <= 10 * TOL[dtype]


@pytest.mark.parametrize("dims", [(5, 6, 7), (9, 33, 35), (4, 8, 64), (12, 17, 70)])
@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_random_populations_ragged(dims, bc, dtype):
    """Off-equilibrium random f on sizes spanning several 32-wide z tiles and
    8-row y tiles with ragged tails; odd and even step counts."""
    f0 = li.random_populations(21, *dims)
    tau = 0.55
    with lbm.Lattice(*dims, tau, LID, dtype, bc=bc) as lat:
        lat.set_populations(f0)
        assert relerr_floor(lat.populations(), f0) <= TOL[dtype]
        ref = f0
        for n in (1, 2, 3):
            lat.step(n)
            ref = oracle.run(ref, bc, tau, LID, n)
            assert relerr_floor(lat.populations(), ref) <= TOL[dtype]


def test_config2_full_with_mass():
    """BASELINE.json:8: 64^3 cavity, 1000 steps, oracle check and mass
    conservation (relative drift <= 1e-13, BASELINE.json:5)."""
    cfg = li.CONFIGS[2]
    rho, u, f0, ref = oracle_from_fields(cfg, cfg.steps)
    with lbm.Lattice(cfg.nx, cfg.ny, cfg.nz, cfg.tau, cfg.u_lid, "f64", bc=cfg.bc) as lat:
        lat.init_equilibrium(rho, u)
        m0 = math.fsum(lat.populations().ravel())
        lat.step(cfg.steps)
        got = lat.populations()
    assert relerr(got, ref) <= 1e-12
    assert abs(math.fsum(got.ravel()) - m0) / m0 <= 1e-13


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_kernel_choice_and_step_splitting_bitwise(dtype):
    dims = (10, 20, 36)
    f0 = li.random_populations(22, *dims)
    outs = []
    for kernel, chunks in [(lbm.LBM_KERNEL_K1, [8]), (lbm.LBM_KERNEL_AUTO, [8]), (lbm.LBM_KERNEL_AUTO, [3, 5]),
                           (lbm.LBM_KERNEL_AUTO, [1, 1, 2, 4]), (lbm.LBM_KERNEL_K1, [7, 1])]:
        with lbm.Lattice(*dims, 0.6, LID, dtype, kernel=kernel) as lat:
            lat.set_populations(f0)
            for n in chunks:
                lat.step(n)
            outs.append(lat.populations())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("slabs", [2, 4])
def test_local_slabs_bitwise(bc, slabs):
    """The X-slab data path (ghost planes + halo spans) emulated on one GPU:
    G slabs give identical bits to one slab, and match the oracle."""
    dims = (16, 12, 20)
    f0 = li.random_populations(23, *dims)
    with lbm.Lattice(*dims, 0.6, LID, "f64", bc=bc) as lat:
        lat.set_populations(f0)
        lat.step(5)
        one = lat.populations()
    with lbm.Lattice(*dims, 0.6, LID, "f64", bc=bc, comm=lbm.LBM_COMM_LOCAL, local_slabs=slabs) as lat:
        lat.set_populations(f0)
        lat.step(5)
        many = lat.populations()
        r, u = lat.macroscopic()
    assert np.array_equal(one, many)
    assert relerr_floor(many, oracle.run(f0, bc, 0.6, LID, 5)) <= 1e-12


def test_init_equilibrium_local_slabs():
    cfg = li.CONFIGS[1]
    rho, u, f0, ref = oracle_from_fields(cfg, 6)
    with lbm.Lattice(cfg.nx, cfg.ny, cfg.nz, cfg.tau, cfg.u_lid, "f64", comm=lbm.LBM_COMM_LOCAL,
                     local_slabs=4) as lat:
        lat.init_equilibrium(rho, u)
        lat.step(6)
        assert relerr(lat.populations(), ref) <= 1e-12


def test_box_readback_matches_full():
    dims = (8, 10, 40)
    f0 = li.random_populations(24, *dims)
    with lbm.Lattice(*dims, 0.6, LID, "f64") as lat:
        lat.set_populations(f0)
        lat.step(3)
        full = lat.populations()
        box = lat.populations_box(2, 3, 5, 4, 6, 33)
    assert np.array_equal(box, full[:, 2:6, 3:9, 5:38])


def test_zero_steps_roundtrip_and_errors():
    dims = (6, 6, 6)
    f0 = li.random_populations(25, *dims)
    with lbm.Lattice(*dims, 0.6, LID, "f64") as lat:
        with pytest.raises(lbm.LbmError, match="not initialised"):
            lat.step(1)
        lat.set_populations(f0)
        lat.step(0)
        assert relerr_floor(lat.populations(), f0) <= 1e-15
        with pytest.raises(lbm.LbmError):
            lat.step(-1)
        bad = f0.copy()
        bad[3, 1, 1, 1] = np.nan
        with pytest.raises(lbm.LbmError, match="finite"):
            lat.set_populations(bad)
        rho = np.ones(dims)
        rho[0, 0, 0] = -1.0
        with pytest.raises(lbm.LbmError, match="rho"):
            lat.init_equilibrium(rho, None)


def test_rest_state_and_lid_closed_form():
    nx, ny, nz = 8, 8, 8
    with lbm.Lattice(nx, ny, nz, 0.6, LID, "f64") as lat:
        lat.init_equilibrium(None, None)
        lat.step(1)
        g = lat.populations()
    _, w, _ = oracle.d3q19()
    assert np.allclose(g[16, :, :, nz - 1], 1 / 36 + 1 / 120, atol=4e-16, rtol=0)
    assert np.allclose(g[6, :, :, nz - 1], 1 / 36 - 1 / 120, atol=4e-16, rtol=0)
    with lbm.Lattice(nx, ny, nz, 0.6, (0, 0, 0), "f64") as lat:
        lat.init_equilibrium(None, None)
        lat.step(100)
        g = lat.populations()
    assert np.max(np.abs(g - w[:, None, None, None])) <= 1e-15


K2_DIMS = [(1, 8, 32), (2, 5, 7), (3, 9, 33), (7, 8, 32), (16, 16, 64), (5, 17, 31), (33, 10, 70), (12, 24, 96),
           (64, 11, 40), (9, 13, 64)]


@pytest.mark.parametrize("dims", K2_DIMS)
@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_k2_equals_k1_bitwise(dims, bc, dtype):
    """The two-step sweep K2 (TMA-staged) and its single-copy ring form
    K2_SC reproduce two one-step sweeps (K1) bit for bit: ragged
    tiles, tiles touching every wall, x-chunk seams, thin slabs, both BCs,
    both dtypes; and all match the oracle."""
    if bc == lbm.LBM_BC_PERIODIC and dims[0] < 2:
        pytest.skip("periodic needs >= 2 planes")
    f0 = li.random_populations(31, *dims)
    res = {}
    for kernel in (lbm.LBM_KERNEL_K1, lbm.LBM_KERNEL_K2, lbm.LBM_KERNEL_K2_SC):
        with lbm.Lattice(*dims, 0.6, LID, dtype, bc=bc, kernel=kernel) as lat:
            lat.set_populations(f0)
            lat.step(4)
            res[kernel] = lat.populations()
            st = lbm.lbm_get_stats(lat.ctx)
            if kernel != lbm.LBM_KERNEL_K1:
                assert st.k2_launches == 2 and st.k1_launches == 0
    assert np.array_equal(res[lbm.LBM_KERNEL_K1], res[lbm.LBM_KERNEL_K2])
    assert np.array_equal(res[lbm.LBM_KERNEL_K1], res[lbm.LBM_KERNEL_K2_SC])
    assert relerr_floor(res[lbm.LBM_KERNEL_K2], oracle.run(f0, bc, 0.6, LID, 4)) <= TOL[dtype]


@pytest.mark.parametrize("dims", [(4, 1, 1), (4, 2, 3), (5, 3, 2), (6, 1, 37), (4, 9, 1), (6, 4, 33), (4, 17, 64)])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kernel", ["k2", "k2sc"])
def test_periodic_frame_bitwise(dims, dtype, kernel):
    """Periodic boxes read the ghost frame: K2 keeps it
    current with its stores (a row / column may have several frame copies
    when ny or nz < 4), and after a K1 step or an import the frame is
    rebuilt before the next K2 sweep.  Bitwise equal to K1 for step splits
    that alternate the two, and to the oracle."""
    f0 = li.random_populations(35, *dims)
    kern = lbm.LBM_KERNEL_K2 if kernel == "k2" else lbm.LBM_KERNEL_K2_SC
    res = []
    for k, splits in ((lbm.LBM_KERNEL_K1, [10]), (kern, [1, 2, 3, 2, 2])):
        with lbm.Lattice(*dims, 0.6, LID, dtype, bc=lbm.LBM_BC_PERIODIC, kernel=k) as lat:
            lat.set_populations(f0)
            for n in splits:
                lat.step(n)
            res.append(lat.populations())
    assert np.array_equal(res[0], res[1])
    assert relerr_floor(res[1], oracle.run(f0, lbm.LBM_BC_PERIODIC, 0.6, LID, 10)) <= TOL[dtype] * 10


@pytest.mark.parametrize("dims", [(4, 1, 1), (5, 3, 2), (9, 17, 45), (16, 8, 32), (33, 24, 64), (6, 13, 100)])
def test_k3_three_step_bitwise(dims):
    """The three-step prototype K3: T+2 staged by TMA,
    two shared-memory rings, the y/z wrap from the 3-row ghost frame and the
    x wrap on the TMA plane index -- bit for bit K1 for step counts that mix
    K3 sweeps with K2 / K1 remainders and read-backs, and the oracle."""
    f0 = li.random_populations(39, *dims)
    res = []
    for k, splits in ((lbm.LBM_KERNEL_K1, [3, 4, 5, 3, 1]), (lbm.LBM_KERNEL_K3, [3, 4, 5, 3, 1])):
        with lbm.Lattice(*dims, 0.6, LID, "f32", bc=lbm.LBM_BC_PERIODIC, kernel=k) as lat:
            lat.set_populations(f0)
            out = []
            for n in splits:
                lat.step(n)
                out.append(lat.populations())
            res.append(out)
            st = lbm.lbm_get_stats(lat.ctx)
    assert st.k2_launches >= 5  # K3 sweeps (counted as multi-step sweeps) ran
    for a, b in zip(*res):
        assert np.array_equal(a, b)
    assert relerr_floor(res[1][-1], oracle.run(f0, lbm.LBM_BC_PERIODIC, 0.6, LID, 16)) <= TOL["f32"] * 16


@pytest.mark.parametrize("bx,by", [(1, 2), (2, 2), (1, 4), (3, 2)])
@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_xy_blocks_bitwise(bx, by, bc, dtype):
    """X-Y partition emulated on one
    GPU: bx x-ranges times by y-blocks, frame rows exchanged between blocks,
    then the x ghost planes -- the same bits as one slab for K2 sweeps, K1
    steps and read-backs in between (populations, boxes across block seams,
    moments), from host and device initial fields, and the oracle."""
    dims = (12, 16, 40)
    f0 = li.random_populations(37, *dims)
    rho = 1.0 + li.uniform(38, int(np.prod(dims)), -1e-3, 1e-3).reshape(dims)
    u = li.uniform(39, 3 * int(np.prod(dims)), -0.01, 0.01).reshape(*dims, 3)
    res = []
    for kw in ({}, dict(comm=lbm.LBM_COMM_LOCAL, local_slabs=bx, local_blocks_y=by)):
        with lbm.Lattice(*dims, 0.6, LID, dtype, bc=bc, **kw) as lat:
            out = []
            lat.set_populations(f0)
            for n in (3, 2, 4, 1, 2):
                lat.step(n)
                out.append(lat.populations())
                out.extend(lat.macroscopic())
                out.append(lat.populations_box(2, 5, 3, 7, 9, 30))
            lat.init_equilibrium(rho, u)
            lat.step(5)
            out.append(lat.populations())
            lbm.lbm_init_equilibrium_device(lat.ctx, torch.from_numpy(rho).cuda(), torch.from_numpy(u).cuda())
            lat.step(4)
            r = torch.empty(dims, dtype=torch.float64, device="cuda")
            v = torch.empty(*dims, 3, dtype=torch.float64, device="cuda")
            lbm.lbm_macroscopic_device(lat.ctx, r, v)
            lbm.lbm_synchronize(lat.ctx)
            out.extend([r.cpu().numpy(), v.cpu().numpy(), lat.populations()])
            res.append(out)
    for a, b in zip(*res):
        assert np.array_equal(a, b), (bx, by, bc, dtype)
    assert relerr_floor(res[1][0], oracle.run(f0, bc, 0.6, LID, 3)) <= TOL[dtype]


K2_VARIANTS = [("LBM_K2_TILE", v, 2) for v in ["8x32", "8x16", "16x16"]] + [("LBM_K2_EARLY", "0", 2), ("LBM_K2_CHUNK", "3", 2)]


@pytest.mark.parametrize("fused", ["0", "1"])
@pytest.mark.parametrize("overlap", ["0", "1"])
def test_overlapped_exchange_bitwise(overlap, fused, tmp_path):
    """The halo exchange overlapped with the interior sweep (comm stream +
    interior/edge split, the NCCL default), the serial exchange, and the
    fused halo (K2 storing the neighbours' ghost planes itself, no exchange
    after the first sweep) all give the bits of a single-slab K1 run, for
    LOCAL slabs on one device and the periodic self-wrap, K2 and K1 (odd
    step) sweeps, both dtypes, with read-backs between sweeps."""
    import subprocess
    import sys
    import os
    script = tmp_path / "overlap.py"
    script.write_text(
        "import numpy as np, lbm_inputs as li, paper_2208_05429_b200 as lbm\n"
        "for bc in (lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC):\n"
        "  for dims, slabs in [((48, 12, 40), 4), ((24, 9, 33), 2), ((12, 8, 32), 1), ((16, 8, 32), 4)]:\n"
        "    for dt in ('f64', 'f32'):\n"
        "      f0 = li.random_populations(43, *dims); r = []\n"
        "      for s, k in ((1, lbm.LBM_KERNEL_K1), (slabs, lbm.LBM_KERNEL_AUTO)):\n"
        "        kw = dict(comm=lbm.LBM_COMM_LOCAL, local_slabs=s) if s > 1 else {}\n"
        "        with lbm.Lattice(*dims, 0.6, (0.05, 0, 0), dt, bc=bc, kernel=k, **kw) as lat:\n"
        "          lat.set_populations(f0); out = []\n"
        "          for n in (3, 2, 4, 2):\n"
        "            lat.step(n); out.append(lat.populations()); out.extend(lat.macroscopic())\n"
        "          r.append(out)\n"
        "      for a, b in zip(*r): assert np.array_equal(a, b), (bc, dims, dt)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root, LBM_OVERLAP=overlap, LBM_FUSED_HALO=fused)
    out = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


@pytest.mark.parametrize("var,shape,kernel", K2_VARIANTS)
def test_k2_variants_bitwise(var, shape, kernel, tmp_path):
    """Every compiled two-step variant (K2 tile TY x TZ, ring slack S, CTAs
    per SM; K2_TMA tiles and issue order -- env vars read once per process,
    so each runs in a subprocess) equals K1 bit for bit on ragged cavity and
    periodic boxes in both dtypes."""
    import subprocess
    import sys
    import os
    script = tmp_path / "k2r_shape.py"
    script.write_text(
        "import numpy as np, lbm_inputs as li, paper_2208_05429_b200 as lbm\n"
        "for bc in (lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC):\n"
        "  for dims in [(5, 17, 31), (9, 21, 70), (4, 8, 32)]:\n"
        "    for dt in ('f64', 'f32'):\n"
        "      f0 = li.random_populations(41, *dims); r = []\n"
        f"      for k in (lbm.LBM_KERNEL_K1, {kernel}):\n"
        "        with lbm.Lattice(*dims, 0.6, (0.05, 0, 0), dt, bc=bc, kernel=k) as lat:\n"
        "          lat.set_populations(f0); lat.step(4); r.append(lat.populations())\n"
        "      assert np.array_equal(r[0], r[1]), (bc, dims, dt)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root)
    env[var] = shape
    out = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
def test_k2_local_slabs_bitwise(bc):
    dims = (32, 20, 40)
    f0 = li.random_populations(32, *dims)
    outs = []
    for kernel, slabs in [(lbm.LBM_KERNEL_K1, 1), (lbm.LBM_KERNEL_K2, 1), (lbm.LBM_KERNEL_K2, 2),
                          (lbm.LBM_KERNEL_K2, 8), (lbm.LBM_KERNEL_K2_SC, 2)]:
        comm = lbm.LBM_COMM_LOCAL if slabs > 1 else lbm.LBM_COMM_NONE
        with lbm.Lattice(*dims, 0.55, LID, "f64", bc=bc, kernel=kernel, comm=comm, local_slabs=slabs) as lat:
            lat.set_populations(f0)
            lat.step(6)
            outs.append(lat.populations())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


AA_DIMS = [(1, 8, 32), (3, 9, 33), (5, 17, 31), (7, 8, 32), (12, 24, 96)]


@pytest.mark.parametrize("dims", AA_DIMS)
@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("lid", [(0.0, 0.0, 0.0), LID])
def test_aa_single_copy_equals_k1(dims, bc, dtype, lid):
    """Single-copy AA storage: after every step count
    (both storage phases) the canonical populations and the moments equal
    K1's, and match the oracle; ragged tiles, every wall, the lid, periodic
    wraps (one-plane x included).  Bit for bit without a lid; with the lid
    K1's pull storage holds f(t0) - lid and adds it back on read (S(S^-1 f)
    rounds at the lid cells, ~1 ulp) while AA stores f(t0) itself, so there
    the two agree to rounding (and both with the oracle)."""
    if bc == lbm.LBM_BC_PERIODIC and (dims[0] < 2 or lid != LID):
        pytest.skip("periodic needs >= 2 planes; the lid is a cavity feature")
    f0 = li.random_populations(47, *dims)
    exact = lid == (0.0, 0.0, 0.0) or bc == lbm.LBM_BC_PERIODIC
    with lbm.Lattice(*dims, 0.6, lid, dtype, bc=bc, kernel=lbm.LBM_KERNEL_K1) as ref, \
            lbm.Lattice(*dims, 0.6, lid, dtype, bc=bc, kernel=lbm.LBM_KERNEL_AA) as aa:
        ref.set_populations(f0)
        aa.set_populations(f0)
        assert np.array_equal(aa.populations(), f0 if dtype == "f64" else f0.astype(np.float32).astype(np.float64))
        for n in (1, 1, 2, 1):
            ref.step(n)
            aa.step(n)
            assert aa.time == ref.time
            a, b = aa.populations(), ref.populations()
            r1, u1 = ref.macroscopic()
            r2, u2 = aa.macroscopic()
            if exact:
                assert np.array_equal(a, b)
                assert np.array_equal(r1, r2) and np.array_equal(u1, u2)
            else:
                assert relerr_floor(a, b) <= (1e-14 if dtype == "f64" else 1e-5)
        got = aa.populations()
    assert relerr_floor(got, oracle.run(f0, bc, 0.6, lid, 5)) <= TOL[dtype]


def test_aa_config2_init_equilibrium_and_errors():
    """AA from lbm_init_equilibrium (host and device inputs) on the config-2
    cavity (64^3, lid) for 30 steps agrees with K1 and the oracle; host and
    device inputs give identical bits; AA refuses multi-slab contexts."""
    cfg = li.CONFIGS[2]
    rho, u = li.init_fields(cfg)
    outs = []
    for kernel in (lbm.LBM_KERNEL_K1, lbm.LBM_KERNEL_AA):
        with lbm.Lattice(cfg.nx, cfg.ny, cfg.nz, cfg.tau, cfg.u_lid, "f64", bc=cfg.bc, kernel=kernel) as lat:
            lat.init_equilibrium(rho, u)
            lat.step(30)
            outs.append((lat.populations(), *lat.macroscopic()))
    assert relerr(outs[1][0], outs[0][0]) <= 1e-14
    ref = oracle.run(oracle.init_equilibrium(cfg.nx, cfg.ny, cfg.nz, rho, u), cfg.bc, cfg.tau, cfg.u_lid, 30)
    assert relerr(outs[1][0], ref) <= 1e-12
    with lbm.Lattice(cfg.nx, cfg.ny, cfg.nz, cfg.tau, cfg.u_lid, "f64", bc=cfg.bc, kernel=lbm.LBM_KERNEL_AA) as lat:
        rd = torch.from_numpy(rho).cuda()
        ud = torch.from_numpy(u).cuda()
        lbm.lbm_init_equilibrium_device(lat.ctx, rd, ud)
        lat.step(30)
        assert np.array_equal(lat.populations(), outs[1][0])
    with pytest.raises(lbm.LbmError):  # cavity slabs of one plane
        lbm.Lattice(4, 8, 8, 0.6, LID, "f64", kernel=lbm.LBM_KERNEL_AA, comm=lbm.LBM_COMM_LOCAL, local_slabs=4)


@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
@pytest.mark.parametrize("slabs", [2, 4])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_aa_local_slabs_bitwise(bc, slabs, dtype):
    """AA over X-slabs (LOCAL transport on one device): the forward halo
    before each odd step and the reverse halo after it give the single-slab
    AA bits after every step count, including odd-phase read-backs."""
    dims = (16, 12, 20)
    f0 = li.random_populations(59, *dims)
    runs = []
    for s_ in (1, slabs):
        kw = dict(comm=lbm.LBM_COMM_LOCAL, local_slabs=s_) if s_ > 1 else {}
        with lbm.Lattice(*dims, 0.6, LID, dtype, bc=bc, kernel=lbm.LBM_KERNEL_AA, **kw) as lat:
            lat.set_populations(f0)
            out = []
            for n in (1, 2, 1, 3):
                lat.step(n)
                out.append((lat.populations(), *lat.macroscopic()))
            runs.append(out)
    for a, b in zip(*runs):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    assert relerr_floor(runs[1][-1][0], oracle.run(f0, bc, 0.6, LID, 7)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_peer_halo_world1_self_import_bitwise(dtype):
    """The fused cross-GPU halo (LBM_HALO_PEER) as a
    one-rank periodic ring: the lattice buffers are exported as file
    descriptors, passed over the rendezvous socket to this rank itself and
    mapped a second time; K2 stores the x ghost planes through that mapping
    as it would into a neighbour's memory over NVLink, and consecutive
    sweeps wait on the done-counter the previous sweep wrote through it
    (stream memory operations).  Odd splits (K1 steps through NCCL) and
    read-backs between sweeps; bitwise equal to the in-process wrap."""
    dims = (24, 10, 36)
    f0 = li.random_populations(57, *dims)
    try:
        uid = lbm.lbm_nccl_unique_id()
    except lbm.LbmError as e:  # pragma: no cover
        pytest.skip(f"NCCL unavailable: {e}")
    outs = []
    for kw in ({}, dict(comm=lbm.LBM_COMM_NCCL, nccl_id=uid, halo=lbm.LBM_HALO_PEER)):
        with lbm.Lattice(*dims, 0.6, LID, dtype, bc=lbm.LBM_BC_PERIODIC, **kw) as lat:
            lat.set_populations(f0)
            out = []
            for n in (3, 2, 4, 1, 2):
                lat.step(n)
                out.append(lat.populations())
                out.extend(lat.macroscopic())
            st = lbm.lbm_get_stats(lat.ctx)
            outs.append((out, st.launches))
    for a, b in zip(outs[0][0], outs[1][0]):
        assert np.array_equal(a, b)
    assert relerr_floor(outs[1][0][-3], oracle.run(f0, lbm.LBM_BC_PERIODIC, 0.6, LID, 12)) <= TOL[dtype] * 4


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_nccl_transport_world1_periodic_bitwise(dtype):
    """The NCCL halo path on hardware: a one-rank communicator on a periodic
    box sends its x-halo spans to itself (ncclSend/ncclRecv to self in one
    group), on the high-priority comm stream overlapped with the interior
    sweep (the NCCL default), for K2 and K1 (odd) sweeps -- bitwise equal to
    the in-process wrap, and to the oracle."""
    dims = (24, 10, 36)
    f0 = li.random_populations(53, *dims)
    try:
        uid = lbm.lbm_nccl_unique_id()
    except lbm.LbmError as e:  # pragma: no cover
        pytest.skip(f"NCCL unavailable: {e}")
    outs = []
    # (and the single-copy ring's halo parts through NCCL: K2_SC)
    # (a unique id initialises one communicator: a fresh one per NCCL context)
    for comm, kernel, kw in [(lbm.LBM_COMM_NONE, 0, {}), (lbm.LBM_COMM_NCCL, 0, {"nccl_id": uid}),
                             (lbm.LBM_COMM_NCCL, lbm.LBM_KERNEL_K2_SC, {"nccl_id": lbm.lbm_nccl_unique_id()})]:
        with lbm.Lattice(*dims, 0.6, LID, dtype, bc=lbm.LBM_BC_PERIODIC, comm=comm, kernel=kernel, **kw) as lat:
            lat.set_populations(f0)
            lat.step(3)
            lat.step(2)
            outs.append(lat.populations())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    assert relerr_floor(outs[1], oracle.run(f0, lbm.LBM_BC_PERIODIC, 0.6, LID, 5)) <= TOL[dtype]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kernel", [0, 1])
def test_nccl_xy_transport_world1_bitwise(dtype, kernel, monkeypatch):
    """The NCCL X-Y block transport (lbm_opts.ranks_y, csrc/api.cu exchange)
    on hardware: with LBM_TEST_YSELF=1 a one-rank periodic context does not
    wrap y in the kernels but sends its packed frame-row bands to itself
    through ncclSend/ncclRecv (the y group), then its x spans (the x group),
    before every K2 (and odd K1) sweep, for init, set_populations and the
    read-backs -- bitwise equal to the in-process wrap, and to the oracle."""
    dims = (16, 20, 36)
    f0 = li.random_populations(57, *dims)
    rho0 = li.uniform(58, dims[0] * dims[1] * dims[2], 0.99, 1.01).reshape(dims)
    try:
        lbm.lbm_nccl_unique_id()
    except lbm.LbmError as e:  # pragma: no cover
        pytest.skip(f"NCCL unavailable: {e}")
    outs = []
    for yself in (False, True):
        if yself:
            monkeypatch.setenv("LBM_TEST_YSELF", "1")
        kw = {"comm": lbm.LBM_COMM_NCCL, "nccl_id": lbm.lbm_nccl_unique_id()}
        with lbm.Lattice(*dims, 0.6, LID, dtype, bc=lbm.LBM_BC_PERIODIC, kernel=kernel, **kw) as lat:
            lat.set_populations(f0)
            lat.step(3)
            a = lat.populations()
            lat.step(2)
            b = lat.populations()
            m = lat.macroscopic()
            lat.init_equilibrium(rho0, None)
            lat.step(4)
            c = lat.populations()
            outs.append((a, b, m[0], m[1], c))
        monkeypatch.delenv("LBM_TEST_YSELF", raising=False)
    for x, y in zip(outs[0], outs[1]):
        assert np.array_equal(x, y)
    assert relerr_floor(outs[1][1], oracle.run(f0, lbm.LBM_BC_PERIODIC, 0.6, LID, 5)) <= TOL[dtype]


# Sample boxes (origin, size) at full size: domain corners (walls, lid edge),
# tile seams (y % 8, z % 32), x-chunk seams (x % 32) and the interior.
def _sample_boxes(cfg):
    nx, ny, nz = cfg.nx, cfg.ny, cfg.nz
    sz = (12, 16, 48)
    cand = [(0, 0, 0), (nx - sz[0], ny - sz[1], nz - sz[2]), (0, ny - sz[1], nz - sz[2]),
            (nx // 2 - 5, 8 * (ny // 16) - 7, 32 * (nz // 64) - 22), (min(31, nx - sz[0]), 3, 5),
            (nx - sz[0], 0, nz // 2)]
    return [(o, sz) for o in cand]


@pytest.mark.parametrize("cfg_id,dtype,kernel", [(3, "f64", 0), (4, "f64", 0), (5, "f64", 0), (5, "f32", 0),
                                                 (5, "f64", lbm.LBM_KERNEL_K2_SC), (3, "f32", lbm.LBM_KERNEL_K2_SC),
                                                 (5, "f64", lbm.LBM_KERNEL_AA)])
def test_full_size_sampled_parity(cfg_id, dtype, kernel):
    """BASELINE.json configs 3-5 at their FULL sizes, in the launch
    configuration bench.py times (K2 sweeps, x-chunks, 1 GPU; and the
    single-copy ring, K2_SC): sampled boxes of the GPU state equal the
    oracle's sub-box steps (oracle.step_box, the core away from unknown
    pulls) after one two-step sweep and one more single step; the mass of the
    cavities is conserved over the domain."""
    cfg = li.CONFIGS[cfg_id]
    rho, u = li.init_fields(cfg)
    boxes = _sample_boxes(cfg)
    dims = (cfg.nx, cfg.ny, cfg.nz)
    with lbm.Lattice(*dims, cfg.tau, cfg.u_lid, dtype, bc=cfg.bc, kernel=kernel) as lat:
        lat.init_equilibrium(rho, u)
        r0, _ = lat.macroscopic()
        m0 = float(np.sum(r0, dtype=np.float64))
        del r0
        lat.step(2)
        got2 = [lat.populations_box(*o, *s) for o, s in boxes]
        lat.step(1)
        got3 = [lat.populations_box(*o, *s) for o, s in boxes]
        st = lbm.lbm_get_stats(lat.ctx)
        assert st.k1_launches >= 1 and (st.k2_launches >= 1 or kernel == lbm.LBM_KERNEL_AA)
        r3, _ = lat.macroscopic()
        m3 = float(np.sum(r3, dtype=np.float64))
        del r3
    if cfg.bc == lbm.LBM_BC_CAVITY:
        assert abs(m3 - m0) / m0 <= (1e-13 if dtype == "f64" else 1e-6)
    for (o, s), g2, g3 in zip(boxes, got2, got3):
        sl = tuple(slice(a, a + b) for a, b in zip(o, s))
        f = oracle.init_equilibrium(*s, rho[sl], u[sl])
        ref = []
        for _ in range(3):
            f = oracle.step_box(f, dims, o, cfg.bc, cfg.tau, cfg.u_lid)
            ref.append(f)
        for g, r in ((g2, ref[1]), (g3, ref[2])):
            known = ~np.isnan(r)
            assert known.sum() > 0.15 * r.size
            assert relerr(g[known], r[known]) <= TOL[dtype], (cfg.name, o)


def test_randomised_configurations_bitwise():
    """Property check over random small lattices (seeded): for any dims,
    boundary mode, dtype, kernel (K2, K2_SC, AA), slab count and split of
    the step count, the result equals K1 on one slab bit for bit (AA: no
    lid, see test_aa_single_copy_equals_k1), and K1 matches the oracle."""
    rng = np.random.default_rng(2208)
    for trial in range(24):
        bc = int(rng.integers(0, 2))
        slabs = int(rng.choice([1, 1, 2, 3]))
        nxl = int(rng.integers(2 if slabs == 1 else 4, 9))
        dims = (nxl * slabs, int(rng.integers(1, 19)), int(rng.integers(1, 45)))
        if bc == lbm.LBM_BC_PERIODIC and dims[0] < 2:
            continue
        dtype = str(rng.choice(["f64", "f32"]))
        kernel = int(rng.choice([lbm.LBM_KERNEL_K2, lbm.LBM_KERNEL_K2_SC, lbm.LBM_KERNEL_AA]))
        lid = (0.0, 0.0, 0.0) if kernel == lbm.LBM_KERNEL_AA else (float(rng.uniform(-0.05, 0.05)),
                                                                    float(rng.uniform(-0.05, 0.05)), 0.0)
        splits = [int(v) for v in rng.integers(0, 4, size=int(rng.integers(1, 4)))]
        tau = float(rng.uniform(0.52, 1.5))
        f0 = li.random_populations(100 + trial, *dims)
        with lbm.Lattice(*dims, tau, lid, dtype, bc=bc, kernel=lbm.LBM_KERNEL_K1) as ref:
            ref.set_populations(f0)
            ref.step(sum(splits))
            want = ref.populations()
        kw = dict(comm=lbm.LBM_COMM_LOCAL, local_slabs=slabs) if slabs > 1 else {}
        with lbm.Lattice(*dims, tau, lid, dtype, bc=bc, kernel=kernel, **kw) as lat:
            lat.set_populations(f0)
            for n in splits:
                lat.step(n)
            got = lat.populations()
        case = (dims, bc, dtype, kernel, slabs, splits, tau)
        assert np.array_equal(got, want), case
        if dtype == "f64":
            assert relerr_floor(want, oracle.run(f0, bc, tau, lid, sum(splits))) <= 1e-12, case


@pytest.mark.parametrize("kernel", [lbm.LBM_KERNEL_AUTO, lbm.LBM_KERNEL_K2_SC, lbm.LBM_KERNEL_AA])
def test_init_null_velocity_equals_zero_velocity(kernel):
    """u = NULL is u = 0 (include/lbm.h; bench.py passes NULL for the cavity
    recipes' zero initial velocity): host and device inputs, every storage."""
    cfg = li.CONFIGS[2]
    rho, u = li.init_fields(cfg)
    assert not np.any(u)
    outs = []
    with lbm.Lattice(cfg.nx, cfg.ny, cfg.nz, cfg.tau, cfg.u_lid, "f64", kernel=kernel) as lat:
        for args in ((rho, u), (rho, None)):
            lat.init_equilibrium(*args)
            lat.step(5)
            outs.append(lat.populations())
        lbm.lbm_init_equilibrium_device(lat.ctx, torch.from_numpy(rho).cuda(), None)
        lat.step(5)
        outs.append(lat.populations())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])

"""The C-ABI library without a GPU: it loads, exports every symbol that
include/lbm.h declares, validates arguments before touching the device, and
its host-side halo plan is consistent."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2208_05429_b200 as lbm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lbm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lbm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    L = ctypes.CDLL(lbm.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/lbm.h but not exported"
    assert sorted(lbm.EXPORTS) == syms
    assert lbm.lbm_abi_version() == 3


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {lbm.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("args,msg", [
    ((0, 4, 4, 0.6, None, 0), "dimensions"),
    ((4, 4, 4, 0.5, None, 0), "tau"),
    ((4, 4, 4, float("nan"), None, 0), "tau"),
    ((4, 4, 4, 0.6, (0.0, 0.0, 0.1), 0), "tangential"),
    ((4, 4, 4, 0.6, (0.4, 0.0, 0.0), 0), "0.3"),
    ((4, 4, 4, 0.6, None, 7), "dtype"),
])
def test_create_rejects_before_allocation(args, msg):
    with pytest.raises(lbm.LbmError) as e:
        lbm.lbm_create(*args)
    assert e.value.status == 1 and msg in str(e.value)


def test_create_rejects_bad_partitions():
    o = lbm.lbm_default_opts()
    o.comm, o.local_slabs = lbm.LBM_COMM_LOCAL, 3
    with pytest.raises(lbm.LbmError, match="divisible"):
        lbm.lbm_create_ex(16, 4, 4, 0.6, None, "f64", o)
    o.local_slabs = 8
    with pytest.raises(lbm.LbmError, match=">= 4 planes"):
        lbm.lbm_create_ex(16, 4, 4, 0.6, None, "f64", o)
    o = lbm.lbm_default_opts()
    o.world, o.rank = 2, 0
    with pytest.raises(lbm.LbmError, match="comm NONE"):
        lbm.lbm_create_ex(16, 4, 4, 0.6, None, "f64", o)
    o.comm = lbm.LBM_COMM_NCCL
    with pytest.raises(lbm.LbmError, match="nccl_id"):
        lbm.lbm_create_ex(16, 4, 4, 0.6, None, "f64", o)
    o = lbm.lbm_default_opts()
    o.bc = lbm.LBM_BC_PERIODIC
    with pytest.raises(lbm.LbmError, match="periodic"):
        lbm.lbm_create_ex(1, 4, 4, 0.6, None, "f64", o)


def test_create_rejects_bad_kernel_choices():
    o = lbm.lbm_default_opts()
    o.kernel = 7
    with pytest.raises(lbm.LbmError, match="bad kernel"):
        lbm.lbm_create_ex(16, 4, 4, 0.6, None, "f64", o)
    o.kernel = -1
    with pytest.raises(lbm.LbmError, match="bad kernel"):
        lbm.lbm_create_ex(16, 4, 4, 0.6, None, "f64", o)
    o.kernel = lbm.LBM_KERNEL_K2_REG  # reserved: the removed cp.async variant
    with pytest.raises(lbm.LbmError, match="removed"):
        lbm.lbm_create_ex(16, 4, 4, 0.6, None, "f64", o)


def test_peer_halo_rejects_unsupported():
    """LBM_HALO_PEER needs NCCL ranks and the two-buffer K2 storage."""
    o = lbm.lbm_default_opts()
    o.halo = lbm.LBM_HALO_PEER
    with pytest.raises(lbm.LbmError, match="comm NCCL"):
        lbm.lbm_create_ex(16, 4, 4, 0.6, None, "f64", o)
    o.comm, o.nccl_id = lbm.LBM_COMM_NCCL, ctypes.cast(ctypes.create_string_buffer(128), ctypes.c_void_p)
    for k in (lbm.LBM_KERNEL_AA, lbm.LBM_KERNEL_K2_SC, lbm.LBM_KERNEL_K1):
        o.kernel = k
        with pytest.raises(lbm.LbmError, match="two-buffer"):
            lbm.lbm_create_ex(16, 4, 4, 0.6, None, "f64", o)
    o.kernel, o.halo = 0, 3
    with pytest.raises(lbm.LbmError, match="bad halo"):
        lbm.lbm_create_ex(16, 4, 4, 0.6, None, "f64", o)


def test_k3_rejects_unsupported():
    """The three-step prototype K3 runs fp32 periodic single-slab boxes only."""
    o = lbm.lbm_default_opts()
    o.kernel, o.bc = lbm.LBM_KERNEL_K3, lbm.LBM_BC_PERIODIC
    with pytest.raises(lbm.LbmError, match="K3"):
        lbm.lbm_create_ex(8, 8, 32, 0.6, None, "f64", o)
    o.bc = lbm.LBM_BC_CAVITY
    with pytest.raises(lbm.LbmError, match="K3"):
        lbm.lbm_create_ex(8, 8, 32, 0.6, None, "f32", o)
    o.bc, o.comm, o.local_slabs = lbm.LBM_BC_PERIODIC, lbm.LBM_COMM_LOCAL, 2
    with pytest.raises(lbm.LbmError, match="K3"):
        lbm.lbm_create_ex(16, 8, 32, 0.6, None, "f32", o)


@pytest.mark.parametrize("q", [15, 19, 27])
def test_lattice_table_matches_oracle_convention(q):
    """The host direction order of lbm_lattice_table is the oracle's
    (oracle_dqq.c; D3Q19: SPEC.md:109) -- same velocities, same weights."""
    import oracle
    c, w = lbm.lbm_lattice_table(q)
    c0, w0, _ = oracle.dqq_table(q)
    assert np.array_equal(c, c0) and np.array_equal(w, w0)


def test_lattice_validation():
    o = lbm.lbm_default_opts()
    assert o.lattice == 19
    o.lattice = 21
    with pytest.raises(lbm.LbmError, match="bad lattice"):
        lbm.lbm_create_ex(8, 8, 8, 0.6, None, "f64", o)
    o.lattice, o.comm, o.local_slabs = 27, lbm.LBM_COMM_LOCAL, 2
    with pytest.raises(lbm.LbmError, match="D3Q27"):
        lbm.lbm_create_ex(8, 8, 8, 0.6, None, "f64", o)
    o = lbm.lbm_default_opts()
    o.lattice, o.kernel = 15, lbm.LBM_KERNEL_AA
    with pytest.raises(lbm.LbmError, match="D3Q15"):
        lbm.lbm_create_ex(8, 8, 8, 0.6, None, "f64", o)
    with pytest.raises(lbm.LbmError):
        lbm.lbm_lattice_table(21)
    # NCCL x-slabs of the other lattices: one-step kernel, x slabs only,
    # NCCL send/recv (rejected before any allocation or communicator)
    for kw, msg in [({"kernel": lbm.LBM_KERNEL_K2}, "one-step kernel"),
                    ({"halo": lbm.LBM_HALO_PEER}, "D3Q15"),
                    ({"ranks_y": 2}, "D3Q15")]:
        o = lbm.lbm_default_opts()
        o.lattice, o.comm, o.world, o.rank = 15, lbm.LBM_COMM_NCCL, 2, 0
        uid = ctypes.create_string_buffer(128)  # (never used: validation fails first)
        o.nccl_id = ctypes.cast(uid, ctypes.c_void_p)
        for k, v in kw.items():
            setattr(o, k, v)
        with pytest.raises(lbm.LbmError, match=msg):
            lbm.lbm_create_ex(8, 8, 8, 0.6, None, "f64", o)


def test_xy_blocks_validation():
    """X-Y blocks (local_blocks_y) need LOCAL slabs, ny divisible into >= 4
    rows per block, and the two-buffer K1/K2 storage."""
    o = lbm.lbm_default_opts()
    assert o.local_blocks_y == 1
    o.local_blocks_y = 2
    with pytest.raises(lbm.LbmError, match="comm LOCAL"):
        lbm.lbm_create_ex(8, 16, 8, 0.6, None, "f64", o)
    o.comm = lbm.LBM_COMM_LOCAL
    o.local_blocks_y = 3
    with pytest.raises(lbm.LbmError, match="rows each"):
        lbm.lbm_create_ex(8, 16, 8, 0.6, None, "f64", o)
    o.local_blocks_y = 8
    with pytest.raises(lbm.LbmError, match="rows each"):
        lbm.lbm_create_ex(8, 16, 8, 0.6, None, "f64", o)
    o.local_blocks_y, o.kernel = 2, lbm.LBM_KERNEL_AA
    with pytest.raises(lbm.LbmError, match="two-buffer"):
        lbm.lbm_create_ex(8, 16, 8, 0.6, None, "f64", o)
    o.kernel, o.lattice = lbm.LBM_KERNEL_AUTO, 27
    with pytest.raises(lbm.LbmError, match="D3Q27"):
        lbm.lbm_create_ex(8, 16, 8, 0.6, None, "f64", o)


def test_header_enums_match_binding():
    """Every enumerator of include/lbm.h has the same value in the binding."""
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "lbm.h")).read(), flags=re.S)
    found = 0
    for body in re.findall(r"typedef enum\s*\{(.*?)\}", src, flags=re.S):
        for name, val in re.findall(r"\b(LBM_[A-Z0-9_]+)\s*=\s*(\d+)", body):
            assert getattr(lbm, name) == int(val), name
            found += 1
    assert found >= 17


def test_step_rejects_negative_and_null():
    with pytest.raises(lbm.LbmError):
        lbm.lbm_step(None, 1)


def test_no_gpu_reports_cuda_error_not_crash():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(lbm.LbmError) as e:
        lbm.lbm_create(8, 8, 8, 0.6, (0.05, 0, 0), "f64")
    assert e.value.status in (3, 2)


# (cavity pitch, periodic pitch): cavity rows padded to 32 B; periodic rows
# carry the ghost frame -- a 32 B sector before z = 0 and after nz - 1
@pytest.mark.parametrize("dtype,esize,pitch", [("f64", 8, (8, 16)), ("f32", 4, (8, 24))])
def test_halo_plan_layout(dtype, esize, pitch):
    nx, ny, nz = 32, 6, 5
    for world in (1, 2, 4):
        for bc in (lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC):
            for r in range(world):
                p = lbm.lbm_plan_halo(nx, ny, nz, dtype, bc, r, world)
                nxl = nx // world
                assert p.nx_local == nxl and p.x0 == r * nxl
                per = bc == lbm.LBM_BC_PERIODIC
                assert p.nz_pitch == pitch[per] and (p.nz_pitch * esize) % 32 == 0
                assert (p.y_ghost, p.z_offset) == ((2, 32 // esize) if per else (0, 0))
                assert p.cell0 == p.y_ghost * p.nz_pitch + p.z_offset
                assert (p.z_offset * esize) % 32 == 0  # cells stay 32 B aligned
                assert p.nz_pitch - p.z_offset - nz >= (32 // esize if per else 0)
                assert p.plane_q == (ny + 2 * p.y_ghost) * p.nz_pitch and p.plane_x == 19 * p.plane_q
                assert p.buffer_elems == (nxl + 4) * p.plane_x
                assert p.span == 24 * p.plane_q
                # spans stay inside the buffer and the ghost spans stay inside ghost planes
                for off in (p.send_left_off, p.send_right_off, p.recv_left_off, p.recv_right_off):
                    assert 0 <= off and off + p.span <= p.buffer_elems
                assert p.recv_left_off + p.span == 2 * p.plane_x
                assert p.recv_right_off == (nxl + 2) * p.plane_x
                assert p.send_left_off == 2 * p.plane_x
                assert p.send_right_off + p.span == (nxl + 2) * p.plane_x
                if bc == lbm.LBM_BC_PERIODIC:
                    assert p.left == (r - 1) % world and p.right == (r + 1) % world
                else:
                    assert p.left == (r - 1 if r > 0 else -1)
                    assert p.right == (r + 1 if r < world - 1 else -1)
                slots = list(p.dir_of_slot)
                assert sorted(slots) == list(range(19))
                cx = [0, -1, 0, 0, -1, -1, -1, -1, 0, 0, 1, 0, 0, 1, 1, 1, 1, 0, 0]
                assert [cx[i] for i in slots] == [-1] * 5 + [0] * 9 + [1] * 5


def test_plan_rejects_bad_args():
    with pytest.raises(lbm.LbmError):
        lbm.lbm_plan_halo(10, 4, 4, "f64", 0, 0, 3)
    with pytest.raises(lbm.LbmError):
        lbm.lbm_plan_halo(8, 4, 4, "f64", 0, 2, 2)


def test_ranks_y_validation():
    """NCCL X-Y blocks (lbm_opts.ranks_y): NCCL only, world and ny divisible,
    >= 4 rows per block, the two-buffer K1/K2 storage, the NCCL exchange."""
    o = lbm.lbm_default_opts()
    assert o.ranks_y == 1
    o.ranks_y = 2
    with pytest.raises(lbm.LbmError, match="comm NCCL"):
        lbm.lbm_create_ex(16, 16, 8, 0.6, None, "f64", o)
    o.comm, o.nccl_id = lbm.LBM_COMM_NCCL, ctypes.cast(ctypes.create_string_buffer(128), ctypes.c_void_p)
    o.world, o.rank, o.ranks_y = 3, 0, 2
    with pytest.raises(lbm.LbmError, match="divisible by ranks_y"):
        lbm.lbm_create_ex(16, 16, 8, 0.6, None, "f64", o)
    o.world = 4
    with pytest.raises(lbm.LbmError, match=">= 4 rows"):
        lbm.lbm_create_ex(16, 6, 8, 0.6, None, "f64", o)
    for k in (lbm.LBM_KERNEL_AA, lbm.LBM_KERNEL_K2_SC):
        o.kernel = k
        with pytest.raises(lbm.LbmError, match="K1/K2"):
            lbm.lbm_create_ex(16, 16, 8, 0.6, None, "f64", o)
    o.kernel, o.halo = lbm.LBM_KERNEL_AUTO, lbm.LBM_HALO_PEER
    with pytest.raises(lbm.LbmError, match="EXCHANGE"):
        lbm.lbm_create_ex(16, 16, 8, 0.6, None, "f64", o)


@pytest.mark.parametrize("bc", [0, 1])
def test_plan_halo_xy(bc):
    """The rank grid of lbm_plan_halo_xy: rank = x slab * ranks_y + y block,
    x neighbours in the same y block, y neighbours in the same x slab (walls
    at the cavity ends, a ring when periodic), the frame-row bands."""
    nx, ny, nz, world, ry = 24, 32, 12, 6, 2
    wx = world // ry
    for r in range(world):
        p = lbm.lbm_plan_halo_xy(nx, ny, nz, "f64", bc, r, world, ry)
        bx, by = divmod(r, ry)
        assert (p.nx_local, p.x0, p.ny_local, p.y0) == (nx // wx, bx * (nx // wx), ny // ry, by * (ny // ry))
        assert p.y_ghost == 2
        left = (bx - 1) % wx if bc else (bx - 1 if bx > 0 else None)
        right = (bx + 1) % wx if bc else (bx + 1 if bx < wx - 1 else None)
        assert p.left == (-1 if left is None else left * ry + by)
        assert p.right == (-1 if right is None else right * ry + by)
        down = (by - 1) % ry if bc else (by - 1 if by > 0 else None)
        up = (by + 1) % ry if bc else (by + 1 if by < ry - 1 else None)
        assert p.down == (-1 if down is None else bx * ry + down)
        assert p.up == (-1 if up is None else bx * ry + up)
        nzp, nyl = p.nz_pitch, ny // ry
        assert p.plane_q == (nyl + 4) * nzp and p.y_band == 2 * nzp
        # rows of an (x, direction) plane: frame [0, 2), cells [2, nyl + 2), frame [nyl + 2, nyl + 4)
        assert (p.recv_down_off, p.send_down_off) == (0, 2 * nzp)
        assert (p.send_up_off, p.recv_up_off) == (nyl * nzp, (nyl + 2) * nzp)
    # ranks_y = 1 is the X-slab plan
    a = lbm.lbm_plan_halo_xy(nx, ny, nz, "f64", bc, 1, 3, 1)
    b = lbm.lbm_plan_halo(nx, ny, nz, "f64", bc, 1, 3)
    assert bytes(a) == bytes(b) and a.down == a.up == -1
    for bad in ((4, 3), (6, 4)):  # world % ranks_y, ny % ranks_y (ny = 32 ok for 2) -> nx / ny checks
        with pytest.raises(lbm.LbmError):
            lbm.lbm_plan_halo_xy(nx, 30, nz, "f64", bc, 0, bad[0], bad[1])


def test_binding_fails_loudly_without_library(tmp_path):
    """No CPU fallback: a package copy without liblbm_b200.so raises
    ImportError at import (the product path never routes elsewhere)."""
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "paper_2208_05429_b200"
    pkg.mkdir()
    src = os.path.join(ROOT, "paper_2208_05429_b200")
    for f in ("__init__.py", "build.py"):
        shutil.copy(os.path.join(src, f), pkg / f)
    out = subprocess.run([sys.executable, "-c", "import paper_2208_05429_b200"], cwd=tmp_path,
                         env=dict(os.environ, PYTHONPATH=str(tmp_path)), capture_output=True, text=True, timeout=120)
    assert out.returncode != 0
    assert "ImportError" in out.stderr and "liblbm_b200.so is missing" in out.stderr

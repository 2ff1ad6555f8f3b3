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
    assert lbm.lbm_abi_version() == 2


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
    o.lattice, o.kernel = 15, lbm.LBM_KERNEL_K2
    with pytest.raises(lbm.LbmError, match="D3Q15"):
        lbm.lbm_create_ex(8, 8, 8, 0.6, None, "f64", o)
    with pytest.raises(lbm.LbmError):
        lbm.lbm_lattice_table(21)


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

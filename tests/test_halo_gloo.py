"""Multi-GPU host logic on CPU: the X-slab halo plan of the C-ABI
(`lbm_plan_halo`) driven through torch.distributed with the gloo backend,
world size 2 (and a 4-rank ring), exactly as the NCCL path orders it:
[send left, recv right], [send right, recv left].

Each rank builds its slab buffer in the library's HBM layout (planes
x = -2 .. nxl+1, [19 slots][ny][nz_pitch]) from a global post-collision
field, exchanges the 24-slot spans, and checks (1) the ghost planes hold the
neighbours' planes for every slot of the span, and (2) the received halo is
sufficient for TWO steps: a numpy two-step on the slab (the K2 sweep's data
need) reproduces the global two-step on the slab's planes."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lbm_inputs as li
import np_lbm
import paper_2208_05429_b200 as lbm

LID = (0.05, 0.0, 0.0)
TAU = 0.6


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def to_buffer(G, p, x0, nxl):
    """Global canonical field G[19, nx, ny, nz] -> slab buffer (own planes only,
    ghosts NaN) in the library layout described by plan p."""
    _, nx, ny, nz = G.shape
    buf = np.full(p.buffer_elems, np.nan)
    v = buf.reshape(nxl + 4, 19, p.plane_q // p.nz_pitch, p.nz_pitch)
    gy, zo = p.y_ghost, p.z_offset
    for k in range(19):
        v[2:nxl + 2, k, gy:gy + ny, zo:zo + nz] = G[p.dir_of_slot[k], x0:x0 + nxl]
    return buf


def from_buffer(buf, p, nxl, ny, nz):
    """Slab buffer -> canonical A[19, nxl + 4, ny, nz] (ghost planes included)."""
    v = buf.reshape(nxl + 4, 19, p.plane_q // p.nz_pitch, p.nz_pitch)
    gy, zo = p.y_ghost, p.z_offset
    A = np.empty((19, nxl + 4, ny, nz))
    for k in range(19):
        A[p.dir_of_slot[k]] = v[:, k, gy:gy + ny, zo:zo + nz]
    return A


def exchange(buf, p):
    t = torch.from_numpy(buf)
    n = p.span
    reqs = []
    # same order as csrc/api.cu exchange(): [send left, recv right], [send right, recv left]
    if p.left >= 0:
        reqs.append(dist.isend(t[p.send_left_off:p.send_left_off + n].clone(), p.left))
    if p.right >= 0:
        rr = torch.empty(n, dtype=torch.float64)
        reqs.append(dist.irecv(rr, p.right))
    if p.right >= 0:
        reqs.append(dist.isend(t[p.send_right_off:p.send_right_off + n].clone(), p.right))
    if p.left >= 0:
        rl = torch.empty(n, dtype=torch.float64)
        reqs.append(dist.irecv(rl, p.left))
    for r in reqs:
        r.wait()
    if p.right >= 0:
        buf[p.recv_right_off:p.recv_right_off + n] = rr.numpy()
    if p.left >= 0:
        buf[p.recv_left_off:p.recv_left_off + n] = rl.numpy()


def worker(rank, world, port, dims, bc, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = dims
        periodic = bc == lbm.LBM_BC_PERIODIC
        G = li.random_populations(41, nx, ny, nz)  # every rank draws the same global field
        p = lbm.lbm_plan_halo(nx, ny, nz, "f64", bc, rank, world)
        nxl, x0 = p.nx_local, p.x0
        buf = to_buffer(G, p, x0, nxl)
        exchange(buf, p)
        A = from_buffer(buf, p, nxl, ny, nz)
        # (1) ghost content: left ghost = [x0-2: P slots | x0-1: all], right = [x0+nxl: all | +1: M slots]
        P_dirs = [10, 13, 14, 15, 16]
        M_dirs = [1, 4, 5, 6, 7]
        if p.left >= 0:
            assert np.array_equal(A[:, 1], G[:, (x0 - 1) % nx])
            assert np.array_equal(A[P_dirs, 0], G[P_dirs, (x0 - 2) % nx])
        if p.right >= 0:
            assert np.array_equal(A[:, nxl + 2], G[:, (x0 + nxl) % nx])
            assert np.array_equal(A[M_dirs, nxl + 3], G[M_dirs, (x0 + nxl + 1) % nx])
        # (2) two steps on the slab from its halo == two global steps
        lo = 2 if p.left < 0 else None   # index of the first own plane if it touches a wall
        hi = nxl + 1 if p.right < 0 else None
        s1_planes = list(range(2 if p.left < 0 else 1, (nxl + 2) if p.right < 0 else nxl + 3))
        S1 = np.full_like(A, np.nan)
        S1[:, s1_planes] = np_lbm.step(A, TAU, periodic, LID, s1_planes, lo, hi)
        S2 = np_lbm.step(S1, TAU, periodic, LID, list(range(2, nxl + 2)), lo, hi)
        glo = 0 if not periodic else None
        gA = G
        ghi = nx - 1 if not periodic else None
        g1 = np_lbm.step(gA, TAU, periodic, LID, list(range(nx)), glo, ghi, wrap_x=periodic)
        g2 = np_lbm.step(g1, TAU, periodic, LID, list(range(nx)), glo, ghi, wrap_x=periodic)
        assert not np.isnan(S2).any(), "halo insufficient: NaN reached the slab"
        assert np.max(np.abs(S2 - g2[:, x0:x0 + nxl])) == 0.0
        q.put((rank, "ok"))
    except BaseException:  # report to the parent
        import traceback
        q.put((rank, traceback.format_exc()[-600:]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,bc", [
    (2, (12, 5, 6), lbm.LBM_BC_CAVITY),
    (2, (12, 5, 6), lbm.LBM_BC_PERIODIC),
    (4, (16, 4, 5), lbm.LBM_BC_CAVITY),
    (4, (16, 4, 5), lbm.LBM_BC_PERIODIC),
])
def test_halo_exchange_gloo(world, dims, bc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, dims, bc, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_numpy_two_step_matches_oracle():
    """Ties np_lbm to the pinned oracle: S(C(S(A))) from np_lbm equals the
    oracle's two steps of the canonical field S(A)."""
    import oracle
    dims = (6, 5, 7)
    A = li.random_populations(42, *dims)
    for periodic in (False, True):
        wl = None if periodic else 0
        wh = None if periodic else dims[0] - 1
        xs = list(range(dims[0]))
        f0 = np_lbm.pull(A, xs, periodic, LID, wl, wh, wrap_x=periodic)
        a1 = np_lbm.step(A, TAU, periodic, LID, xs, wl, wh, wrap_x=periodic)
        a2 = np_lbm.step(a1, TAU, periodic, LID, xs, wl, wh, wrap_x=periodic)
        f2 = np_lbm.pull(a2, xs, periodic, LID, wl, wh, wrap_x=periodic)  # canonical f(t+2)
        # canonical f(t+2) is S(f*(t+1)); oracle: two steps from canonical f(t) = S(A)
        ref = oracle.run(f0, oracle.BC_PERIODIC if periodic else oracle.BC_CAVITY, TAU, LID, 2)
        assert np.max(np.abs(f2 - ref)) <= 1e-15

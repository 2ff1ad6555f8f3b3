"""Multi-rank host logic of the D3Q15/D3Q27 x slabs (csrc/api.cu
`dqq_exchange`) on CPU: torch.distributed with the
gloo backend, world 2 and 3, both boundary modes.

Each rank pushes the post-collision populations of its slab (collision by
the pinned oracle's `dqq_collide`) with the library's rule -- a link leaving
through a face shared with a neighbour rank lands in the ghost plane
x = -1 / nx_local, a closed face bounces (lid included) -- then exchanges,
in direction order, ghost plane nx_local of every c_x = +1 direction to the
right rank and ghost plane -1 of every c_x = -1 direction to the left rank,
with the library's neighbour rule (periodic ring; cavity ends have none);
the receiver takes them into the same (unused) ghost slots and merges them
into plane 0 / nx_local - 1 except where the link's source lies beyond a y /
z wall (`k_dqq_merge`).  The slab must then equal the oracle's global step
on its planes, exactly, and every slot must be written exactly once.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lbm_inputs as li
import oracle
import paper_2208_05429_b200 as lbm

LID = (0.05, 0.02, 0.0)
TAU = 0.6


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def slab_step(q, F, x0, nxl, bc, left, right):
    """One push step of the slab F[q, nxl, ny, nz] into B[q, nxl + 2, ...]
    (index 0 and nxl + 1 are the ghost planes)."""
    c, w, opp = oracle.dqq_table(q)
    _, _, ny, nz = F.shape
    B = np.full((q, nxl + 2, ny, nz), np.nan)
    per = bc == lbm.LBM_BC_PERIODIC
    for x in range(nxl):
        for y in range(ny):
            for z in range(nz):
                fs = oracle.dqq_collide(q, F[:, x, y, z], 1.0 / TAU)
                for i in range(q):
                    dx, dy, dz = x + c[i, 0], y + c[i, 1], z + c[i, 2]
                    if per:
                        dy, dz = dy % ny, dz % nz
                        out = False
                    else:
                        out = (dx < 0 and left < 0) or (dx >= nxl and right < 0) or not (0 <= dy < ny) \
                            or not (0 <= dz < nz)
                    if not out:
                        B[i, dx + 1, dy, dz] = fs[i]
                    else:
                        o = opp[i]
                        v = fs[i]
                        if dz >= nz:
                            v = v + 6.0 * w[o] * (c[o, 0] * LID[0] + c[o, 1] * LID[1])
                        B[o, x + 1, y, z] = v
    return B


def worker(rank, world, port, q, dims, bc, res):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = dims
        nxl, x0 = nx // world, rank * (nx // world)
        G = li.uniform(300 + q, q * nx * ny * nz, 0.01, 0.06).reshape(q, nx, ny, nz)
        per = bc == lbm.LBM_BC_PERIODIC
        left = (rank - 1) % world if per else (rank - 1 if rank > 0 else -1)
        right = (rank + 1) % world if per else (rank + 1 if rank < world - 1 else -1)
        B = slab_step(q, G[:, x0:x0 + nxl], x0, nxl, bc, left, right)
        c, _, _ = oracle.dqq_table(q)
        ops, recvs = [], []
        for i in range(q):
            if c[i, 0] == 1:
                if right >= 0:
                    ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(B[i, nxl + 1])), right))
                if left >= 0:
                    t = torch.empty(ny, nz, dtype=torch.float64)
                    ops.append(dist.P2POp(dist.irecv, t, left))
                    recvs.append((i, 1, t))
            elif c[i, 0] == -1:
                if left >= 0:
                    ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(B[i, 0])), left))
                if right >= 0:
                    t = torch.empty(ny, nz, dtype=torch.float64)
                    ops.append(dist.P2POp(dist.irecv, t, right))
                    recvs.append((i, nxl, t))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        # received planes land in the unused ghost slots of their direction;
        # the merge copies them in except where the link's source is beyond a
        # y / z wall (that slot holds the cell's own bounce-back)
        for i, plane, t in recvs:
            ghost = 0 if plane == 1 else nxl + 1
            assert np.isnan(B[i, ghost]).all(), "a receiving ghost slot was written locally"
            B[i, ghost] = t.numpy()
            for y in range(ny):
                for z in range(nz):
                    if per or (0 <= y - c[i, 1] < ny and 0 <= z - c[i, 2] < nz):
                        assert np.isnan(B[i, plane, y, z]), "a merged slot was also written locally"
                        B[i, plane, y, z] = B[i, ghost, y, z]
        want = oracle.dqq_run(q, G, bc, TAU, LID, 1)[:, x0:x0 + nxl]
        got = B[:, 1:nxl + 1]
        assert not np.isnan(got).any(), "a slot of the slab was never written"
        assert np.array_equal(got, want)
        res.put((rank, "ok"))
    except BaseException:  # report to the parent
        import traceback
        res.put((rank, traceback.format_exc()[-800:]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q", [15, 27])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("bc", [lbm.LBM_BC_CAVITY, lbm.LBM_BC_PERIODIC])
def test_dqq_xslab_exchange_gloo(q, world, bc):
    dims = (4 * world, 3, 4)
    ctx = mp.get_context("spawn")
    res = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q, dims, bc, res)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = dict(res.get(timeout=180) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    assert all(v == "ok" for v in out.values()), out

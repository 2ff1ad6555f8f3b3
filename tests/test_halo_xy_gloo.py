"""Multi-GPU host logic of the X-Y block transport (lbm_opts.ranks_y) on CPU:
the rank grid and frame-row bands of `lbm_plan_halo_xy` driven through
torch.distributed with the gloo backend, in the order csrc/api.cu
exchange() posts them on NCCL: first the y group ([send down, recv up],
[send up, recv down]) of the packed frame-row bands of the own planes, then
the x group of the 24-slot spans, which carry those rows along.

Each rank builds its block buffer in the library's HBM layout from a global
field and checks, after one exchange, that every frame row of its own planes
and every x ghost plane -- frame rows included, i.e. the x-y corner entries
that come from the DIAGONAL block without a diagonal message -- holds the
global field at the right (x, y) (wrapped when periodic; cavity walls are
never filled)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lbm_inputs as li
import paper_2208_05429_b200 as lbm


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def view(buf, p, nxl):
    """buffer -> [x plane (x = -2 .. nxl+1), slot, plane row, column] view"""
    return buf.reshape(nxl + 4, 19, p.plane_q // p.nz_pitch, p.nz_pitch)


def build(G, p):
    """Own planes and own rows of the block from the global canonical field
    G[19, nx, ny, nz]; z frame columns (periodic) filled by wrap, as the
    library's sweeps / frame fill keep them; everything else NaN."""
    _, nx, ny, nz = G.shape
    nxl, nyl, gy, zo = p.nx_local, p.ny_local, p.y_ghost, p.z_offset
    buf = np.full(p.buffer_elems, np.nan)
    v = view(buf, p, nxl)
    zs = np.arange(-zo, nz + zo) % nz
    for k in range(19):
        blk = G[p.dir_of_slot[k], p.x0:p.x0 + nxl, p.y0:p.y0 + nyl]
        v[2:nxl + 2, k, gy:gy + nyl, 0:nz + 2 * zo] = blk[:, :, zs]
    return buf


def send_recv(pairs):
    """[(kind, tensor, peer)] posted in order, then waited.  Messages to this
    rank itself (a periodic axis with one block: NCCL sends to self) are
    matched in order locally -- gloo has no self pairs."""
    me = dist.get_rank()
    own = [t for kind, t, r in pairs if kind == "s" and r == me]
    reqs = []
    for kind, t, r in pairs:
        if r == me:
            if kind == "r":
                t.copy_(own.pop(0))
            continue
        reqs.append(dist.isend(t, r) if kind == "s" else dist.irecv(t, r))
    for r in reqs:
        r.wait()


def exchange_xy(buf, p):
    nxl, band = p.nx_local, p.y_band
    pq = p.plane_q
    own = 2 * p.plane_x  # plane x = 0
    bands = np.arange(nxl * 19) * pq + own

    def pack(off):
        return torch.from_numpy(np.concatenate([buf[b + off:b + off + band] for b in bands]))

    def unpack(t, off):
        a = t.numpy()
        for j, b in enumerate(bands):
            buf[b + off:b + off + band] = a[j * band:(j + 1) * band]

    n = nxl * 19 * band
    rdn, rup = torch.empty(n, dtype=torch.float64), torch.empty(n, dtype=torch.float64)
    pairs = []
    if p.down >= 0:
        pairs.append(("s", pack(p.send_down_off), p.down))
    if p.up >= 0:
        pairs.append(("r", rup, p.up))
    if p.up >= 0:
        pairs.append(("s", pack(p.send_up_off), p.up))
    if p.down >= 0:
        pairs.append(("r", rdn, p.down))
    send_recv(pairs)
    if p.down >= 0:
        unpack(rdn, p.recv_down_off)
    if p.up >= 0:
        unpack(rup, p.recv_up_off)
    # x group: the 24-slot spans (frame rows included)
    t = torch.from_numpy(buf)
    rr, rl = torch.empty(p.span, dtype=torch.float64), torch.empty(p.span, dtype=torch.float64)
    pairs = []
    if p.left >= 0:
        pairs.append(("s", t[p.send_left_off:p.send_left_off + p.span].clone(), p.left))
    if p.right >= 0:
        pairs.append(("r", rr, p.right))
    if p.right >= 0:
        pairs.append(("s", t[p.send_right_off:p.send_right_off + p.span].clone(), p.right))
    if p.left >= 0:
        pairs.append(("r", rl, p.left))
    send_recv(pairs)
    if p.right >= 0:
        buf[p.recv_right_off:p.recv_right_off + p.span] = rr.numpy()
    if p.left >= 0:
        buf[p.recv_left_off:p.recv_left_off + p.span] = rl.numpy()


def worker(rank, world, ry, port, dims, bc, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = dims
        per = bc == lbm.LBM_BC_PERIODIC
        G = li.random_populations(43, nx, ny, nz)
        p = lbm.lbm_plan_halo_xy(nx, ny, nz, "f64", bc, rank, world, ry)
        nxl, nyl, gy, zo = p.nx_local, p.ny_local, p.y_ghost, p.z_offset
        buf = build(G, p)
        exchange_xy(buf, p)
        v = view(buf, p, nxl)
        zs = np.arange(-zo, nz + zo) % nz
        slots_p = [k for k in range(19) if k >= 14]  # c_x = +1 slots (sent right from plane nxl-2)
        slots_m = [k for k in range(19) if k < 5]    # c_x = -1 slots (sent left from plane 1)
        # which rows of a plane are defined: own rows always; frame rows where a y-neighbour exists
        rows = list(range(gy, gy + nyl))
        if p.down >= 0:
            rows = list(range(0, gy)) + rows
        if p.up >= 0:
            rows = rows + list(range(gy + nyl, 2 * gy + nyl))
        checked = 0
        for xi in range(nxl + 4):  # plane index; global x = x0 + xi - 2
            x = p.x0 + xi - 2
            if xi < 2 and p.left < 0 or xi >= nxl + 2 and p.right < 0:
                continue
            slots = (slots_p if xi == 0 else slots_m if xi == nxl + 3 else range(19))
            for k in slots:
                for r in rows:
                    y = p.y0 + r - gy
                    exp = G[p.dir_of_slot[k], x % nx, y % ny][zs]
                    got = v[xi, k, r, 0:nz + 2 * zo]
                    assert np.array_equal(got, exp), (rank, xi, k, r)
                    checked += 1
        # the x-y corners came from the diagonal block
        if p.left >= 0 and p.down >= 0:
            assert not np.isnan(v[1, :, 0:gy, zo:zo + nz]).any()
        assert checked > 0
        if not per:  # cavity: rows beyond the domain's y walls are never written
            if p.down < 0:
                assert np.isnan(v[2:nxl + 2, :, 0:gy]).all()
            if p.up < 0:
                assert np.isnan(v[2:nxl + 2, :, gy + nyl:]).all()
        q.put((rank, "ok"))
    except BaseException:
        import traceback
        q.put((rank, traceback.format_exc()[-800:]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,ry,dims,bc", [
    (4, 2, (16, 12, 6), lbm.LBM_BC_CAVITY),
    (4, 2, (16, 12, 6), lbm.LBM_BC_PERIODIC),
    (6, 3, (16, 12, 5), lbm.LBM_BC_CAVITY),
    (6, 2, (24, 12, 5), lbm.LBM_BC_PERIODIC),
    (2, 2, (8, 12, 6), lbm.LBM_BC_PERIODIC),
])
def test_xy_block_exchange_gloo(world, ry, dims, bc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, ry, port, dims, bc, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res

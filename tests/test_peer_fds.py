"""The descriptor rendezvous of the fused cross-GPU halo (LBM_HALO_PEER,
csrc/peer.cu) on a CPU: every rank serves its file descriptors on an
abstract Unix socket and fetches its neighbours' (SCM_RIGHTS), exactly as
lbm_create_ex does with the exported VMM lattice buffers -- here with plain
memfd files whose contents identify the owner.  World sizes 1 (a periodic
rank is its own neighbour), 2 (a ring: left == right) and 4 (a ring and a
chain with wall ends)."""
import ctypes
import multiprocessing as mp
import os
import uuid

import pytest

import paper_2208_05429_b200 as lbm


def worker(rank, world, periodic, key, q):
    L = ctypes.CDLL(lbm.LIB_PATH)
    f = L.lbm_internal_exchange_fds
    f.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                  ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_double]
    f.restype = ctypes.c_int
    left = (rank - 1) % world if periodic else (rank - 1 if rank > 0 else -1)
    right = (rank + 1) % world if periodic else (rank + 1 if rank < world - 1 else -1)
    peers = [p for p in (left, right) if p >= 0]
    mine = []
    for m in range(3):
        fd = os.memfd_create(f"r{rank}m{m}")
        os.write(fd, f"rank{rank}:buf{m}".encode())
        mine.append(fd)
    out = (ctypes.c_int * (3 * max(1, len(peers))))()
    rc = f(key.encode(), rank, (ctypes.c_int * max(1, len(peers)))(*peers), len(peers),
           (ctypes.c_int * 3)(*mine), 3, out, 20.0)
    got = []
    if rc == 0:
        for j in range(len(peers)):
            row = []
            for m in range(3):
                fd = out[3 * j + m]
                os.lseek(fd, 0, os.SEEK_SET)
                row.append(os.read(fd, 64).decode())
                os.close(fd)
            got.append(row)
    q.put((rank, rc, peers, got))


@pytest.mark.parametrize("world,periodic", [(1, True), (2, True), (4, True), (4, False), (3, False)])
def test_descriptor_rendezvous(world, periodic):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    key = uuid.uuid4().hex[:16]
    ps = [ctx.Process(target=worker, args=(r, world, periodic, key, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=60) for _ in range(world)]
    for p in ps:
        p.join(timeout=30)
        assert p.exitcode == 0
    for rank, rc, peers, got in res:
        assert rc == 0, rank
        for j, p in enumerate(peers):
            assert got[j] == [f"rank{p}:buf{m}" for m in range(3)], (rank, p)

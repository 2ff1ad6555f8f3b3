"""ctypes wrapper of the plain CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` leg are the only importers.  The
product package ``paper_2208_05429_b200`` never imports this module and
shares no code with it.

Population arrays are numpy float64 of shape (19, nx, ny, nz), canonical
direction order.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")
SRCS = [SRC, os.path.join(HERE, "oracle_dqq.c")]

BC_CAVITY = 0
BC_PERIODIC = 1

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so: -O2 -ffp-contract=off, no fast-math, OpenMP."""
    stale = (not os.path.exists(LIB_PATH)
             or os.path.getmtime(LIB_PATH) < max([os.path.getmtime(f) for f in SRCS]
                                                 + [os.path.getmtime(os.path.join(HERE, "oracle.h"))]))
    if force or stale:
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
               "-fopenmp", "-fPIC", "-shared", *SRCS, "-o", tmp, "-lm"]
        subprocess.check_call(cmd, cwd=HERE)
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        L.oracle_d3q19.argtypes = [ctypes.c_void_p, dp, ctypes.POINTER(ctypes.c_int)]
        L.oracle_moments.argtypes = [dp, dp, dp]
        L.oracle_moments.restype = ctypes.c_int
        L.oracle_equilibrium.argtypes = [ctypes.c_double, dp, dp]
        L.oracle_collide.argtypes = [dp, ctypes.c_double, dp]
        L.oracle_collide.restype = ctypes.c_int
        L.oracle_init_equilibrium.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.c_void_p, dp]
        L.oracle_step.argtypes = [ctypes.c_int] * 4 + [ctypes.c_double, dp, dp, dp]
        L.oracle_run.argtypes = [ctypes.c_int] * 4 + [ctypes.c_double, dp, ctypes.c_long, dp]
        L.oracle_run.restype = ctypes.c_int
        L.oracle_step_box.argtypes = ([ctypes.c_int] * 4 + [ctypes.c_double, dp]
                                      + [ctypes.c_int] * 6 + [dp, dp])
        L.oracle_macroscopic.argtypes = [ctypes.c_int] * 3 + [dp, dp, dp]
        L.oracle_dqq_table.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), dp, ctypes.POINTER(ctypes.c_int)]
        L.oracle_dqq_table.restype = ctypes.c_int
        L.oracle_dqq_equilibrium.argtypes = [ctypes.c_int, ctypes.c_double, dp, dp]
        L.oracle_dqq_collide.argtypes = [ctypes.c_int, dp, ctypes.c_double, dp]
        L.oracle_dqq_collide.restype = ctypes.c_int
        L.oracle_dqq_run.argtypes = [ctypes.c_int] * 5 + [ctypes.c_double, dp, ctypes.c_long, dp]
        L.oracle_dqq_run.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_get_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _vec3(u) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(u, dtype=np.float64).reshape(3))


def d3q19():
    """Return (c[19,3] int, w[19] float64, opp[19] int) as the oracle holds them."""
    c = (ctypes.c_int * 57)()
    w = np.zeros(19)
    opp = (ctypes.c_int * 19)()
    lib().oracle_d3q19(c, _p(w), opp)
    return np.array(list(c), dtype=np.int64).reshape(19, 3), w, np.array(list(opp), dtype=np.int64)


def moments(f):
    f = np.ascontiguousarray(f, dtype=np.float64)
    rho = np.zeros(1)
    u = np.zeros(3)
    err = lib().oracle_moments(_p(f), _p(rho), _p(u))
    if err:
        raise ZeroDivisionError("degenerate moments: rho == 0")
    return float(rho[0]), u


def equilibrium(rho: float, u) -> np.ndarray:
    out = np.zeros(19)
    lib().oracle_equilibrium(float(rho), _p(_vec3(u)), _p(out))
    return out


def collide(f, omega: float) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros(19)
    if lib().oracle_collide(_p(f), float(omega), _p(out)):
        raise ZeroDivisionError("degenerate moments: rho == 0")
    return out


def init_equilibrium(nx, ny, nz, rho=None, u=None) -> np.ndarray:
    f = np.zeros((19, nx, ny, nz))
    r = None if rho is None else np.ascontiguousarray(rho, dtype=np.float64).reshape(-1)
    v = None if u is None else np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    if r is not None:
        assert r.size == nx * ny * nz
    if v is not None:
        assert v.size == 3 * nx * ny * nz
    lib().oracle_init_equilibrium(nx, ny, nz,
                                  None if r is None else r.ctypes.data,
                                  None if v is None else v.ctypes.data, _p(f))
    return f


def step(f, bc: int, tau: float, u_lid=(0.0, 0.0, 0.0)) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float64)
    _, nx, ny, nz = f.shape
    out = np.empty_like(f)
    lib().oracle_step(nx, ny, nz, int(bc), float(tau), _p(_vec3(u_lid)), _p(f), _p(out))
    return out


def run(f, bc: int, tau: float, u_lid=(0.0, 0.0, 0.0), n: int = 1) -> np.ndarray:
    g = np.array(f, dtype=np.float64, order="C", copy=True)
    _, nx, ny, nz = g.shape
    if lib().oracle_run(nx, ny, nz, int(bc), float(tau), _p(_vec3(u_lid)), int(n), _p(g)):
        raise MemoryError("oracle_run: allocation failed")
    return g


def run_inplace(f, bc: int, tau: float, u_lid=(0.0, 0.0, 0.0), n: int = 1) -> None:
    """``run`` without the copy: advances the C-contiguous float64 f in place
    (full-size golden runs hold two lattices, not three)."""
    _, nx, ny, nz = f.shape
    if lib().oracle_run(nx, ny, nz, int(bc), float(tau), _p(_vec3(u_lid)), int(n), _p(f)):
        raise MemoryError("oracle_run: allocation failed")


def step_box(f_box, dims, origin, bc: int, tau: float, u_lid=(0.0, 0.0, 0.0)) -> np.ndarray:
    """One step on a sub-box of a global domain; unknown pulls become NaN."""
    f_box = np.ascontiguousarray(f_box, dtype=np.float64)
    _, lx, ly, lz = f_box.shape
    out = np.empty_like(f_box)
    nx, ny, nz = dims
    bx, by, bz = origin
    lib().oracle_step_box(nx, ny, nz, int(bc), float(tau), _p(_vec3(u_lid)),
                          bx, by, bz, lx, ly, lz, _p(f_box), _p(out))
    return out


def macroscopic(f):
    f = np.ascontiguousarray(f, dtype=np.float64)
    _, nx, ny, nz = f.shape
    rho = np.zeros((nx, ny, nz))
    u = np.zeros((nx, ny, nz, 3))
    lib().oracle_macroscopic(nx, ny, nz, _p(f), _p(rho), _p(u))
    return rho, u


# ---- other cubic lattices (oracle_dqq.c): q = 15, 19, 27 ----
def dqq_table(q: int):
    """(c[q,3] int, w[q] float64, opp[q] int) of the q-velocity lattice."""
    c = (ctypes.c_int * (3 * q))()
    w = np.zeros(q)
    opp = (ctypes.c_int * q)()
    if lib().oracle_dqq_table(q, c, _p(w), opp):
        raise ValueError(f"unsupported lattice D3Q{q}")
    return np.array(list(c), dtype=np.int64).reshape(q, 3), w, np.array(list(opp), dtype=np.int64)


def dqq_equilibrium(q: int, rho: float, u) -> np.ndarray:
    out = np.zeros(q)
    lib().oracle_dqq_equilibrium(q, float(rho), _p(_vec3(u)), _p(out))
    return out


def dqq_collide(q: int, f, omega: float) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros(q)
    if lib().oracle_dqq_collide(q, _p(f), float(omega), _p(out)):
        raise ZeroDivisionError("degenerate moments: rho == 0")
    return out


def dqq_init_equilibrium(q: int, nx, ny, nz, rho=None, u=None) -> np.ndarray:
    """feq of every cell (plain loop over dqq_equilibrium's C routine)."""
    f = np.zeros((q, nx, ny, nz))
    r = np.ones((nx, ny, nz)) if rho is None else np.asarray(rho, dtype=np.float64).reshape(nx, ny, nz)
    v = np.zeros((nx, ny, nz, 3)) if u is None else np.asarray(u, dtype=np.float64).reshape(nx, ny, nz, 3)
    for x in range(nx):
        for y in range(ny):
            for z in range(nz):
                f[:, x, y, z] = dqq_equilibrium(q, r[x, y, z], v[x, y, z])
    return f


def dqq_run(q: int, f, bc: int, tau: float, u_lid=(0.0, 0.0, 0.0), n: int = 1) -> np.ndarray:
    g = np.array(f, dtype=np.float64, order="C", copy=True)
    assert g.shape[0] == q
    _, nx, ny, nz = g.shape
    r = lib().oracle_dqq_run(q, nx, ny, nz, int(bc), float(tau), _p(_vec3(u_lid)), int(n), _p(g))
    if r:
        raise MemoryError("oracle_dqq_run failed") if r == 1 else ValueError(f"unsupported lattice D3Q{q}")
    return g


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oracle_get_threads())

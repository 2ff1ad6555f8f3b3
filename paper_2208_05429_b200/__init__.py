"""paper_2208_05429_b200 -- B200-native (sm_100a) D3Q19 lattice Boltzmann hot path.

A thin ctypes binding of the C-ABI library ``liblbm_b200.so`` (declared in
``include/lbm.h``).  Every function here only marshals arguments: all of the
method's work -- equilibrium init, the fused collide+stream steps, the
two-step sweeps, the halo exchange, the read-back -- runs in the library's
CUDA kernels.  There is no CPU fallback: importing this package fails loudly
if the library is missing, and every call raises ``LbmError`` when the C call
returns an error status.

Function names mirror the C-ABI: ``lbm_create``, ``lbm_create_ex``,
``lbm_init_equilibrium``, ``lbm_step``, ``lbm_macroscopic``,
``lbm_get_populations``, ``lbm_set_populations``, ``lbm_destroy``, ...
``Lattice`` is a convenience owner of one context.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = _build.LIB

LBM_F64, LBM_F32 = 0, 1
LBM_BC_CAVITY, LBM_BC_PERIODIC = 0, 1
LBM_KERNEL_AUTO, LBM_KERNEL_K1, LBM_KERNEL_K2, LBM_KERNEL_K2_REG, LBM_KERNEL_AA, LBM_KERNEL_K2_SC = 0, 1, 2, 3, 4, 5
LBM_KERNEL_K3 = 6
LBM_COMM_NONE, LBM_COMM_NCCL, LBM_COMM_LOCAL = 0, 1, 2
LBM_HALO_AUTO, LBM_HALO_EXCHANGE, LBM_HALO_PEER = 0, 1, 2
LBM_D3Q15, LBM_D3Q19, LBM_D3Q27 = 15, 19, 27
LBM_OK, LBM_EINVAL, LBM_ENOMEM, LBM_ECUDA, LBM_ENCCL, LBM_ESTATE, LBM_ENUMERIC = 0, 1, 2, 3, 4, 5, 6
STATUS = {0: "LBM_OK", 1: "LBM_EINVAL", 2: "LBM_ENOMEM", 3: "LBM_ECUDA", 4: "LBM_ENCCL", 5: "LBM_ESTATE",
          6: "LBM_ENUMERIC"}
DTYPES = {"f64": LBM_F64, "float64": LBM_F64, "fp64": LBM_F64, "f32": LBM_F32, "float32": LBM_F32, "fp32": LBM_F32}


class LbmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class lbm_opts(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_int), ("bc", ctypes.c_int), ("device", ctypes.c_int),
                ("rank", ctypes.c_int), ("world", ctypes.c_int), ("comm", ctypes.c_int),
                ("nccl_id", ctypes.c_void_p), ("stream", ctypes.c_void_p), ("kernel", ctypes.c_int),
                ("local_slabs", ctypes.c_int), ("halo", ctypes.c_int), ("lattice", ctypes.c_int),
                ("local_blocks_y", ctypes.c_int), ("ranks_y", ctypes.c_int)]


class lbm_halo_plan(ctypes.Structure):
    _fields_ = [("nx_local", ctypes.c_int), ("x0", ctypes.c_int), ("nz_pitch", ctypes.c_int),
                ("plane_q", ctypes.c_longlong), ("plane_x", ctypes.c_longlong),
                ("buffer_elems", ctypes.c_longlong), ("left", ctypes.c_int), ("right", ctypes.c_int),
                ("send_left_off", ctypes.c_longlong), ("send_right_off", ctypes.c_longlong),
                ("recv_left_off", ctypes.c_longlong), ("recv_right_off", ctypes.c_longlong),
                ("span", ctypes.c_longlong), ("dir_of_slot", ctypes.c_int * 19),
                ("y_ghost", ctypes.c_int), ("z_offset", ctypes.c_int), ("cell0", ctypes.c_longlong),
                ("down", ctypes.c_int), ("up", ctypes.c_int), ("ny_local", ctypes.c_int), ("y0", ctypes.c_int),
                ("y_band", ctypes.c_longlong), ("send_down_off", ctypes.c_longlong),
                ("send_up_off", ctypes.c_longlong), ("recv_down_off", ctypes.c_longlong),
                ("recv_up_off", ctypes.c_longlong)]


class lbm_stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_longlong), ("sweep_launches", ctypes.c_longlong),
                ("sweep_ms", ctypes.c_double), ("sweep_updates", ctypes.c_longlong),
                ("k2_launches", ctypes.c_longlong), ("k1_launches", ctypes.c_longlong)]


# The symbols include/lbm.h declares (checked by tests/test_abi.py).
EXPORTS = ["lbm_default_opts", "lbm_create", "lbm_create_ex", "lbm_init_equilibrium",
           "lbm_init_equilibrium_device", "lbm_step", "lbm_macroscopic", "lbm_macroscopic_device",
           "lbm_get_populations", "lbm_get_populations_box", "lbm_set_populations", "lbm_synchronize",
           "lbm_get_time", "lbm_nccl_unique_id", "lbm_plan_halo", "lbm_plan_halo_xy", "lbm_profile_enable", "lbm_profile_reset",
           "lbm_get_stats", "lbm_last_error", "lbm_destroy", "lbm_abi_version", "lbm_lattice_table"]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() or "
                          f"python -m paper_2208_05429_b200.build (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P = ctypes.POINTER
    vp, dp, i, ll, d = ctypes.c_void_p, P(ctypes.c_double), ctypes.c_int, ctypes.c_long, ctypes.c_double
    ctxp = vp
    sig = {
        "lbm_default_opts": (None, [P(lbm_opts)]),
        "lbm_create": (i, [P(ctxp), i, i, i, d, dp, i]),
        "lbm_create_ex": (i, [P(ctxp), i, i, i, d, dp, i, P(lbm_opts)]),
        "lbm_init_equilibrium": (i, [ctxp, vp, vp]),
        "lbm_init_equilibrium_device": (i, [ctxp, vp, vp]),
        "lbm_step": (i, [ctxp, ll]),
        "lbm_macroscopic": (i, [ctxp, vp, vp]),
        "lbm_macroscopic_device": (i, [ctxp, vp, vp]),
        "lbm_get_populations": (i, [ctxp, vp]),
        "lbm_get_populations_box": (i, [ctxp, i, i, i, i, i, i, vp]),
        "lbm_set_populations": (i, [ctxp, vp]),
        "lbm_synchronize": (i, [ctxp]),
        "lbm_get_time": (i, [ctxp, P(ctypes.c_long)]),
        "lbm_nccl_unique_id": (i, [vp]),
        "lbm_plan_halo": (i, [i, i, i, i, i, i, i, P(lbm_halo_plan)]),
        "lbm_plan_halo_xy": (i, [i, i, i, i, i, i, i, i, P(lbm_halo_plan)]),
        "lbm_profile_enable": (i, [ctxp, i]),
        "lbm_profile_reset": (i, [ctxp]),
        "lbm_get_stats": (i, [ctxp, P(lbm_stats)]),
        "lbm_last_error": (ctypes.c_char_p, [ctxp]),
        "lbm_destroy": (None, [ctxp]),
        "lbm_abi_version": (i, []),
        "lbm_lattice_table": (i, [i, P(ctypes.c_int), dp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


_lib = _load()


def lib():
    return _lib


def _check(status: int, ctx=None):
    if status != 0:
        msg = _lib.lbm_last_error(ctx)
        raise LbmError(status, msg.decode() if msg else "")


def _ptr(a, dtype=np.float64, writable=False):
    """Raw address of a C-contiguous float64 numpy array or CUDA/CPU torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != dtype or not a.flags.c_contiguous or (writable and not a.flags.writeable):
            raise TypeError("expected a C-contiguous float64 numpy array")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):  # torch tensor (host or device), no import of torch needed
        if not a.is_contiguous() or str(a.dtype) != "torch.float64":
            raise TypeError("expected a contiguous float64 tensor")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


def _vec3(u):
    if u is None:
        return None
    a = (ctypes.c_double * 3)(*[float(v) for v in u])
    return ctypes.cast(a, ctypes.POINTER(ctypes.c_double)), a


# ------------------------------------------------------------- raw C-ABI --
def lbm_default_opts() -> lbm_opts:
    o = lbm_opts()
    _lib.lbm_default_opts(ctypes.byref(o))
    return o


def lbm_create_ex(nx, ny, nz, tau, u_lid, dtype, opts: lbm_opts | None = None):
    ctx = ctypes.c_void_p()
    dt = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
    v = _vec3(u_lid)
    _check(_lib.lbm_create_ex(ctypes.byref(ctx), int(nx), int(ny), int(nz), float(tau), v[0] if v else None, dt,
                              ctypes.byref(opts) if opts is not None else None))
    return ctx


def lbm_create(nx, ny, nz, tau, u_lid, dtype):
    return lbm_create_ex(nx, ny, nz, tau, u_lid, dtype, None)


def lbm_init_equilibrium(ctx, rho=None, u=None):
    _check(_lib.lbm_init_equilibrium(ctx, _ptr(rho), _ptr(u)), ctx)


def lbm_init_equilibrium_device(ctx, d_rho=None, d_u=None):
    _check(_lib.lbm_init_equilibrium_device(ctx, _ptr(d_rho), _ptr(d_u)), ctx)


def lbm_step(ctx, n: int):
    _check(_lib.lbm_step(ctx, int(n)), ctx)


def lbm_macroscopic(ctx, rho, u):
    _check(_lib.lbm_macroscopic(ctx, _ptr(rho, writable=True), _ptr(u, writable=True)), ctx)


def lbm_macroscopic_device(ctx, d_rho, d_u):
    _check(_lib.lbm_macroscopic_device(ctx, _ptr(d_rho), _ptr(d_u)), ctx)


def lbm_get_populations(ctx, f):
    _check(_lib.lbm_get_populations(ctx, _ptr(f, writable=True)), ctx)


def lbm_get_populations_box(ctx, x0, y0, z0, lx, ly, lz, f):
    _check(_lib.lbm_get_populations_box(ctx, x0, y0, z0, lx, ly, lz, _ptr(f, writable=True)), ctx)


def lbm_set_populations(ctx, f):
    _check(_lib.lbm_set_populations(ctx, _ptr(f)), ctx)


def lbm_synchronize(ctx):
    _check(_lib.lbm_synchronize(ctx), ctx)


def lbm_get_time(ctx) -> int:
    t = ctypes.c_long()
    _check(_lib.lbm_get_time(ctx, ctypes.byref(t)), ctx)
    return t.value


def lbm_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.lbm_nccl_unique_id(buf))
    return buf.raw


def lbm_plan_halo(nx, ny, nz, dtype, bc, rank, world) -> lbm_halo_plan:
    p = lbm_halo_plan()
    dt = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
    _check(_lib.lbm_plan_halo(nx, ny, nz, dt, bc, rank, world, ctypes.byref(p)))
    return p


def lbm_plan_halo_xy(nx, ny, nz, dtype, bc, rank, world, ranks_y) -> lbm_halo_plan:
    p = lbm_halo_plan()
    dt = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
    _check(_lib.lbm_plan_halo_xy(nx, ny, nz, dt, bc, rank, world, ranks_y, ctypes.byref(p)))
    return p


def lbm_profile_enable(ctx, on: bool):
    _check(_lib.lbm_profile_enable(ctx, 1 if on else 0), ctx)


def lbm_profile_reset(ctx):
    _check(_lib.lbm_profile_reset(ctx), ctx)


def lbm_get_stats(ctx) -> lbm_stats:
    s = lbm_stats()
    _check(_lib.lbm_get_stats(ctx, ctypes.byref(s)), ctx)
    return s


def lbm_last_error(ctx=None) -> str:
    m = _lib.lbm_last_error(ctx)
    return m.decode() if m else ""


def lbm_destroy(ctx):
    _lib.lbm_destroy(ctx)


def lbm_abi_version() -> int:
    return _lib.lbm_abi_version()


def lbm_lattice_table(q: int):
    """(c[q,3] int, w[q] float64): the velocity order of host population arrays."""
    c = (ctypes.c_int * (3 * q))()
    w = np.zeros(q)
    _check(_lib.lbm_lattice_table(int(q), c, w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return np.array(list(c), dtype=np.int64).reshape(q, 3), w


# --------------------------------------------------------- convenience --
class Lattice:
    """Owner of one lbm_ctx.  Host arrays are float64 numpy arrays in the
    layouts of include/lbm.h; device arrays may be torch CUDA tensors."""

    def __init__(self, nx, ny, nz, tau, u_lid=(0.0, 0.0, 0.0), dtype="f64", bc=LBM_BC_CAVITY,
                 kernel=LBM_KERNEL_AUTO, comm=LBM_COMM_NONE, local_slabs=1, rank=0, world=1,
                 nccl_id: bytes | None = None, stream=None, device=-1, halo=0, lattice=19, local_blocks_y=1,
                 ranks_y=1):
        o = lbm_default_opts()
        o.bc, o.kernel, o.comm, o.local_slabs, o.halo = bc, kernel, comm, local_slabs, halo
        o.lattice = lattice
        o.local_blocks_y = local_blocks_y
        o.ranks_y = ranks_y
        self.q = lattice
        o.rank, o.world, o.device = rank, world, device
        self._id = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        o.nccl_id = ctypes.cast(self._id, ctypes.c_void_p) if self._id is not None else None
        o.stream = stream
        # host arrays cover this process's part: an x slab, or (ranks_y > 1)
        # an X-Y block of ny // ranks_y rows
        ry = max(1, ranks_y)
        self.nx, self.ny, self.nz = nx, ny // ry, nz
        self.nx_local = nx // (world // ry if world % ry == 0 else world)
        self.ctx = lbm_create_ex(nx, ny, nz, tau, u_lid, dtype, o)

    def init_equilibrium(self, rho=None, u=None):
        if rho is not None:
            rho = np.ascontiguousarray(rho, dtype=np.float64)
        if u is not None:
            u = np.ascontiguousarray(u, dtype=np.float64)
        lbm_init_equilibrium(self.ctx, rho, u)

    def step(self, n: int):
        lbm_step(self.ctx, n)

    def macroscopic(self):
        rho = np.empty((self.nx_local, self.ny, self.nz))
        u = np.empty((self.nx_local, self.ny, self.nz, 3))
        lbm_macroscopic(self.ctx, rho, u)
        return rho, u

    def populations(self):
        f = np.empty((self.q, self.nx_local, self.ny, self.nz))
        lbm_get_populations(self.ctx, f)
        return f

    def populations_box(self, x0, y0, z0, lx, ly, lz):
        f = np.empty((self.q, lx, ly, lz))
        lbm_get_populations_box(self.ctx, x0, y0, z0, lx, ly, lz, f)
        return f

    def set_populations(self, f):
        lbm_set_populations(self.ctx, np.ascontiguousarray(f, dtype=np.float64))

    @property
    def time(self) -> int:
        return lbm_get_time(self.ctx)

    def synchronize(self):
        lbm_synchronize(self.ctx)

    def close(self):
        if self.ctx:
            lbm_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""Sweep-kernel micro-benchmark (tuning aid, not the bench contract): times
the library's two-step (or one-step) sweep launches with the library's own
CUDA events on a cavity/periodic box and prints one line per run.

  python tools/sweep_bench.py --dims 256,512,512 --dtype f64 --kernel k2 --steps 40 --reps 3
Variant shapes are selected by the env vars LBM_K2_TILE."""
import argparse
import os
import statistics
import time
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("LBM_PKG_ROOT"):  # A/B runs: a variant build of the package
    sys.path.insert(0, os.environ["LBM_PKG_ROOT"])

import numpy as np  # noqa: E402

import paper_2208_05429_b200 as lbm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="256,512,512")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--bc", default="cavity")
ap.add_argument("--kernel", default="k2")
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--tag", default="")
ap.add_argument("--slabs", type=int, default=1, help="LOCAL X-slabs on this GPU (exchange path)")
ap.add_argument("--blocks-y", type=int, default=1, help="LOCAL: also split every x slab into this many y blocks")
ap.add_argument("--power", action="store_true", help="also sample SM clock and board power (NVML)")
ap.add_argument("--lattice", type=int, default=19, help="19, or 15 / 27 (one-step kernel)")
a = ap.parse_args()
nx, ny, nz = (int(v) for v in a.dims.split(","))
kern = {"auto": 0, "k1": 1, "k2": 2, "aa": 4, "k2sc": 5, "k3": 6}[a.kernel]
bc = lbm.LBM_BC_CAVITY if a.bc == "cavity" else lbm.LBM_BC_PERIODIC
es = 8 if a.dtype == "f64" else 4
kw = (dict(comm=lbm.LBM_COMM_LOCAL, local_slabs=a.slabs, local_blocks_y=a.blocks_y)
      if a.slabs > 1 or a.blocks_y > 1 else {})
with lbm.Lattice(nx, ny, nz, 0.6, (0.05, 0, 0), a.dtype, bc=bc, kernel=kern, lattice=a.lattice, **kw) as lat:
    lat.init_equilibrium(None, None)
    lat.step(4)
    lbm.lbm_synchronize(lat.ctx)
    res = []
    samp = None
    if a.power:
        import threading
        import time
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        samp, stop = [], threading.Event()

        def run():
            while not stop.is_set():
                samp.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                             pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
                time.sleep(0.05)
        th = threading.Thread(target=run, daemon=True)
        th.start()
    for _ in range(a.reps):
        lbm.lbm_profile_enable(lat.ctx, True)
        lbm.lbm_profile_reset(lat.ctx)
        t0 = time.perf_counter()
        lat.step(a.steps)
        lbm.lbm_synchronize(lat.ctx)
        wall = time.perf_counter() - t0  # whole steps: sweeps + halo exchanges + launch gaps
        st = lbm.lbm_get_stats(lat.ctx)
        lbm.lbm_profile_enable(lat.ctx, False)
        ms = st.sweep_ms / max(1, st.sweep_launches)  # one record per sweep of all slabs
        steps_per = st.sweep_updates / max(1, st.sweep_launches) / (nx * ny * nz)
        mlups = nx * ny * nz * steps_per / (ms * 1e-3) / 1e6
        res.append((mlups, ms, nx * ny * nz * a.steps / wall / 1e6))
    if samp is not None:
        stop.set()
        th.join()
        tail = samp[len(samp) // 3:] or samp
        clk = statistics.median(x[0] for x in tail)
        pw = statistics.median(x[1] for x in tail)
    best = max(r[0] for r in res)
    med = statistics.median(r[0] for r in res)
    gbs = best * 1e6 * a.lattice * es * (2 / steps_per) / 1e9
    print(f"{a.tag or a.kernel:24s} {a.dtype} {a.dims:14s} best {best:9.1f} MLUPS  median {med:9.1f}  "
          f"sweep {min(r[1] for r in res):8.3f} ms  algorithmic {gbs:7.1f} GB/s  "
          f"whole-step {max(r[2] for r in res):9.1f} MLUPS"
          + (f"  sm {clk:.0f} MHz  {pw:.0f} W" if samp is not None else ""), flush=True)

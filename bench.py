#!/usr/bin/env python
"""MLUPS benchmark of the B200 D3Q19 lattice Boltzmann hot path.

One bench "step" is one whole job of a BASELINE.json workload (DESIGN.md
"Measurement"): equilibrium init from (rho, u), the configured number of
lattice time steps (collide + stream with bounce-back and the moving lid,
two steps per sweep), and the macroscopic read-out.  The default workload is
config 5, the 1024x512x512 cuboid lid-driven cavity in fp64 (BASELINE.json:11),
the largest configuration that fits one GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--dtype f64]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # the CPU oracle on host cores

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
if os.environ.get("LBM_PKG_ROOT"):  # A/B runs only: a variant build of the package (tools/build_variant.sh)
    sys.path.insert(0, os.environ["LBM_PKG_ROOT"])

import lbm_inputs as li  # noqa: E402

ESIZE = {"f64": 8, "f32": 4}
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")


def hbm_peak():
    try:
        with open(MEASURED) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------- CPU oracle --
def oracle_sample(cfg: li.Config, budget_s: float):
    """Time the CPU oracle, as it stands, on a bounded sample of the workload:
    the config's full y-z cross-section, a few x planes (same BC, tau, lid and
    init recipe), for about budget_s seconds of stepping."""
    import oracle
    nxs = max(2, min(cfg.nx, int(4_000_000 // (cfg.ny * cfg.nz)) or 2))
    sub = cfg.with_dims(nxs, cfg.ny, cfg.nz)
    rho, u = li.init_fields(sub)
    f = oracle.init_equilibrium(sub.nx, sub.ny, sub.nz, rho, u)
    threads = oracle.get_threads()
    t0 = time.perf_counter()
    f = oracle.run(f, sub.bc, sub.tau, sub.u_lid, 1)
    t1 = time.perf_counter() - t0
    n = max(1, min(200, int(budget_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    f = oracle.run(f, sub.bc, sub.tau, sub.u_lid, n)
    dt = time.perf_counter() - t0
    mlups = sub.cells * n / dt / 1e6
    sample = (f"oracle (oracle/oracle.c, fp64, OpenMP) on {sub.nx}x{sub.ny}x{sub.nz} planes of {cfg.name} "
              f"(same bc/tau/lid/init), {n} steps, {dt:.2f} s")
    return mlups, threads, sample, dt


def cpu_info():
    model = "?"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count()


# -------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks and throttle
    reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------ reference --
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    budget = float(os.environ.get("LBM_REF_BUDGET_S", "40"))  # (tests shorten it)
    per = max(min(1.0, budget), budget / max(1, args.steps + args.warmup))  # whole run ~ a minute
    for _ in range(args.warmup):
        oracle_sample(cfg, per)
    vals, secs = [], 0.0
    for _ in range(args.steps):
        v, threads, sample, dt = oracle_sample(cfg, per)
        vals.append(v)
        secs += dt
    value = statistics.mean(vals)
    model, ncpu = cpu_info()
    line = {
        "impl": "reference", "metric": "MLUPS", "value": round(value, 3), "unit": "MLUPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * secs / max(1, args.steps), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name} (CPU oracle timed on a sample of it)", "nx": cfg.nx, "ny": cfg.ny,
                   "nz": cfg.nz, "bc": "periodic" if cfg.bc else "cavity", "tau": cfg.tau,
                   "u_lid": list(cfg.u_lid), "sample": sample,
                   "ms_per_step": "time of one bench step's sample, not of a whole job"},
        "cpu_baseline": {"value": round(value, 3), "unit": "MLUPS", "cores": threads, "kind": "oracle",
                         "sample": sample, "cpu": model, "host_cpus": ncpu},
        "e2e": {"value": round(value, 3), "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- ours --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "k1", "k2", "aa", "k2sc", "k3"])
    ap.add_argument("--ranks-y", type=int, default=1,
                    help="N > 1 ranks as a (N / R) x R grid of X-Y blocks (lbm_opts.ranks_y; NCCL exchange)")
    ap.add_argument("--halo", default="exchange", choices=["exchange", "peer"],
                    help="N > 1: NCCL send/recv (default) or the fused peer-mapped halo (LBM_HALO_PEER)")
    ap.add_argument("--lbm-steps", type=int, default=None, help="time steps per job (default: the config's)")
    ap.add_argument("--dims", default=None, help="override NX,NY,NZ (profiling runs only)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling (BASELINE.json:11): 128 x 512 x 512 cells of config 5 per GPU")
    ap.add_argument("--lattice", type=int, default=19, choices=[15, 19, 27],
                    help="velocity set: D3Q19 (the paper's, default) or D3Q15 / D3Q27 (N > 1: x slabs, one-step kernel; DESIGN.md section 11)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 is below the timing rules", file=sys.stderr)
    cfg = li.CONFIGS[args.config]
    if args.lbm_steps is not None:
        cfg = li.Config(cfg.name, cfg.nx, cfg.ny, cfg.nz, cfg.bc, cfg.tau, cfg.u_lid, args.lbm_steps, cfg.seed,
                        cfg.init, cfg.note)
    if args.dims:
        nx, ny, nz = (int(v) for v in args.dims.split(","))
        cfg = cfg.with_dims(nx, ny, nz)
    if args.weak:
        if args.config != 5:
            ap.error("--weak is config 5's weak-scaling series (128x512x512 per GPU)")
        cfg = cfg.with_dims(128 * max(1, int(os.environ.get("WORLD_SIZE", "1"))), cfg.ny, cfg.nz)
    if args.impl == "reference":
        if args.lattice != 19:
            ap.error("--impl reference times the D3Q19 oracle (the paper's lattice)")
        return run_reference(args, cfg)
    Q = args.lattice

    import torch
    import torch.distributed as dist

    import paper_2208_05429_b200 as lbm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    ry = args.ranks_y if world > 1 else 1
    if Q != 19 and world > 1 and (args.ranks_y > 1 or args.halo == "peer" or args.kernel not in ("auto", "k1")):
        ap.error("--lattice 15 / 27 across GPUs: x slabs over NCCL send/recv, one-step kernel (auto or k1)")
    if world % ry or cfg.ny % ry:
        ap.error("--ranks-y must divide the world size and ny")
    nxl = cfg.nx // (world // ry)
    x0 = (rank // ry) * nxl
    nyl, y0 = cfg.ny // ry, (rank % ry) * (cfg.ny // ry)
    cells_local = nxl * nyl * cfg.nz
    stream = torch.cuda.Stream(device=dev)
    kernel = {"auto": lbm.LBM_KERNEL_AUTO, "k1": lbm.LBM_KERNEL_K1, "k2": lbm.LBM_KERNEL_K2,
              "aa": lbm.LBM_KERNEL_AA, "k2sc": lbm.LBM_KERNEL_K2_SC, "k3": lbm.LBM_KERNEL_K3}[args.kernel]

    nccl_id = None
    if world > 1:
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(lbm.lbm_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
    lat = lbm.Lattice(cfg.nx, cfg.ny, cfg.nz, cfg.tau, cfg.u_lid, args.dtype, bc=cfg.bc, kernel=kernel,
                      comm=lbm.LBM_COMM_NCCL if world > 1 else lbm.LBM_COMM_NONE, rank=rank, world=world,
                      nccl_id=nccl_id, stream=stream.cuda_stream, device=local_rank,
                      halo=lbm.LBM_HALO_PEER if (args.halo == "peer" and world > 1) else lbm.LBM_HALO_AUTO,
                      ranks_y=ry, lattice=Q)
    ctx = lat.ctx

    # inputs: this rank's slab of the config's seeded fields, resident in HBM
    rho_h, u_h = li.init_fields(cfg, x0, nxl)
    if ry > 1:  # this rank's X-Y block
        rho_h = np.ascontiguousarray(rho_h[:, y0:y0 + nyl])
        u_h = np.ascontiguousarray(u_h[:, y0:y0 + nyl])
    # A workload whose initial velocity is identically zero (the cavity
    # configs' recipe: rho = 1 + noise, u = 0) passes u = NULL, the API's
    # "u = 0" (include/lbm.h), instead of shipping 24 B of zeros per cell.
    u_zero = not np.any(u_h)
    rho_pin = torch.from_numpy(rho_h).pin_memory()
    u_in_pin = None if u_zero else torch.from_numpy(u_h).pin_memory()
    rho_d = rho_pin.to(dev)
    u_in_d = None if u_zero else u_in_pin.to(dev)
    out_rho_d = torch.empty_like(rho_d)
    out_u_d = torch.empty(u_h.shape, dtype=torch.float64, device=dev)
    out_rho_h = torch.empty_like(rho_pin).pin_memory()
    out_u_h = torch.empty(u_h.shape, dtype=torch.float64).pin_memory()
    del rho_h, u_h
    torch.cuda.synchronize()

    def job_device():
        lbm.lbm_init_equilibrium_device(ctx, rho_d, u_in_d)
        lbm.lbm_step(ctx, cfg.steps)
        lbm.lbm_macroscopic_device(ctx, out_rho_d, out_u_d)

    def job_host():
        lbm.lbm_init_equilibrium(ctx, rho_pin, u_in_pin)
        lbm.lbm_step(ctx, cfg.steps)
        lbm.lbm_macroscopic(ctx, out_rho_h, out_u_h)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        job_device()
    barrier()

    # ---- timed region: device-resident inputs and outputs ----
    lbm.lbm_profile_enable(ctx, True)
    lbm.lbm_profile_reset(ctx)
    s0 = lbm.lbm_get_stats(ctx)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            job_device()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    s1 = lbm.lbm_get_stats(ctx)
    lbm.lbm_profile_enable(ctx, False)
    ms_max = max_over_ranks(ms)
    updates_total = cfg.cells * cfg.steps * args.steps
    value = updates_total / (ms_max * 1e-3) / 1e6
    launches = s1.launches - s0.launches

    # dominant kernel: the sweep (K2 two-step, or K1) -- algorithmic bytes per launch
    # = cells in the launch x 2 x Q x sizeof(T) (each population read once and written once)
    es = ESIZE[args.dtype]
    sweep_ms = s1.sweep_ms
    sweep_launches = s1.sweep_launches
    sweep_updates = s1.sweep_updates
    k2 = s1.k2_launches - s0.k2_launches
    k1 = s1.k1_launches - s0.k1_launches
    dominant = (({"k2sc": "k2_single_copy", "k3": "k3_three_step"}.get(args.kernel, "k2_two_step")) if k2 >= k1
                else ("aa_step" if args.kernel == "aa" else "k1_step"))
    if Q != 19:
        dominant = f"d3q{Q}_" + ("k2q_two_step" if k2 >= k1 else "one_step")
    # per launch: cells_local x 2 x Q x es bytes (both K1 and K2 stream the lattice once)
    bytes_per_launch = cells_local * 2 * Q * es
    avg_launch_ms = sweep_ms / max(1, sweep_launches)
    achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    sweep_share = sweep_ms / ms if ms > 0 else None

    # ---- e2e: host arrays through the public API, H2D + D2H inside the timed region ----
    e2e = None
    if not args.no_e2e:
        job_host()
        barrier()
        t0 = time.perf_counter()
        ev0.record(stream)
        for _ in range(args.steps):
            job_host()
        ev1.record(stream)
        barrier()
        e2e_ms = max_over_ranks(max(ev0.elapsed_time(ev1), (time.perf_counter() - t0) * 1e3))
        e2e = {"value": round(updates_total / (e2e_ms * 1e-3) / 1e6, 3), "unit": "MLUPS",
               "h2d_bytes_per_step": int(rho_pin.numel() * 8 + (0 if u_zero else u_in_pin.numel() * 8)) * world,
               "d2h_bytes_per_step": int(out_rho_h.numel() * 8 + out_u_h.numel() * 8) * world}

    cpu = None
    if Q != 19 and not args.no_cpu_baseline:
        cpu = {"value": None, "unit": "MLUPS", "cores": None, "kind": "oracle",
               "sample": "not timed: the CPU baseline is the D3Q19 oracle's"}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:  # the contract: rank 0 at N=1 only
        try:
            v, threads, sample, _ = oracle_sample(cfg, 12.0)
            model, ncpu = cpu_info()
            cpu = {"value": round(v, 3), "unit": "MLUPS", "cores": threads, "kind": "oracle", "sample": sample,
                   "cpu": model, "host_cpus": ncpu}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "MLUPS", "cores": None, "kind": "oracle", "sample": f"failed: {e}"}

    # roofline.traffic: measured DRAM bytes per sweep launch from the newest
    # committed ncu capture of this workload/dtype/kernel (profiles/rNN_traffic.json)
    traffic = None
    for tf in ("r02c_traffic.json", "r02b_traffic.json", "r02_traffic.json", "r01_traffic.json"):
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", tf)))
            t = tj.get(cfg.name, {}).get(dominant, {}).get(args.dtype) if (world == 1 and Q == 19) else None
            if t:
                traffic = {"bytes_per_launch": t["read"] + t["write"], "read": t["read"], "write": t["write"],
                           "x_algorithmic": round((t["read"] + t["write"]) / bytes_per_launch, 3),
                           "source": f"profiles/{tf} (ncu --set full, same workload)"}
                break
        except (OSError, ValueError, KeyError):
            continue

    if rank == 0:
        mlups_bytes = 2 * Q * es  # BASELINE.json:5 roofline: MLUPS x single-step bytes / peak
        line = {
            "metric": "MLUPS", "value": round(value, 3), "unit": "MLUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": cfg.name, "nx": cfg.nx, "ny": cfg.ny, "nz": cfg.nz,
                       "bc": "periodic" if cfg.bc else "cavity", "tau": cfg.tau, "u_lid": list(cfg.u_lid),
                       "lbm_steps_per_job": cfg.steps, "job": "init_equilibrium + lbm_step(n) + macroscopic",
                       "inputs": ("rho (u is identically 0: passed as NULL)" if u_zero else "rho, u"),
                       "kernel": args.kernel, "parallelism": f"x-slab{world}" if ry == 1 else f"xy-block{world // ry}x{ry}",
                       "halo": args.halo if world > 1 else "none",
                       "l2": f"inputs larger than L2: {cells_local * Q * es / 1e9:.1f} GB per lattice copy per GPU",
                       "lattice": f"D3Q{Q}"},
            "mlups_per_gpu": round(value / world, 3),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         # measured DRAM bytes per launch over the same live launch time (GB/s, vs achieved)
                         "traffic": None if traffic is None else
                         round(traffic["bytes_per_launch"] / (avg_launch_ms * 1e-3) / 1e9, 1),
                         "traffic_detail": traffic, "kernel": dominant,
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "avg_launch_ms": round(avg_launch_ms, 4), "peak_source": peak_src,
                         "sweep_share_of_step": None if sweep_share is None else round(sweep_share, 4),
                         "frac_mlups_x_single_step_bytes": round(value / world * mlups_bytes / 1e3 / peak, 4),
                         "frac_mlups_vs_8TBps": round(value / world * mlups_bytes / 1e3 / 8000.0, 4)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    lat.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

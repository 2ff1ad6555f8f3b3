#!/usr/bin/env python
"""Summarise ncu artefacts into text for profiles/ (run here, no GPU needed).

    tools/ncu_summary.py rep <file.ncu-rep> [title]      # one --set full capture
    tools/ncu_summary.py launches <launches.csv> [title]  # --metrics gpu__time_duration.sum list
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read BW"),
    ("dram__bytes_write.sum.per_second", "DRAM write BW"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    lines = [l for l in out.splitlines() if l.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def rep(path, title):
    rows = ncu_csv(["-i", path, "--page", "raw"])
    hdr, units = rows[0], rows[1]
    print(f"# {title}\n# source: {path} (ncu --set full --clock-control none)")
    for r in rows[2:]:
        d = {h: (v, u) for h, v, u in zip(hdr, r, units)}
        print(f"\nkernel: {d.get('Kernel Name', ('?',))[0]}")
        for k, name in KEYS:
            if k in d:
                print(f"  {name:32s} {d[k][0]:>18s} {d[k][1]}")
        stalls = []
        for h in hdr:
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    v = float(d[h][0])
                except ValueError:
                    continue
                if v > 0.05:
                    stalls.append((v, h.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
        print("  warp stalls (cycles per issued instruction):")
        for v, n in sorted(stalls, reverse=True):
            print(f"    {n:28s} {v:6.3f}")


def launches(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    iK, iM, iV, iU = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if r[iM] != "gpu__time_duration.sum":
            continue
        k = r[iK].split("(")[0]
        tot[k] += float(r[iV].replace(",", "")) * scale[r[iU]]
        cnt[k] += 1
    T = sum(tot.values())
    print(f"# {title}\n# source: {path} (ncu --metrics gpu__time_duration.sum --clock-control none;"
          f" cold-cache, serialised launches: compare shares, not absolutes)")
    print(f"{'kernel':58s} {'launches':>8s} {'total ms':>11s} {'share':>7s} {'avg ms':>10s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:58]:58s} {cnt[k]:8d} {tot[k]:11.3f} {100 * tot[k] / T:6.2f}% {tot[k] / cnt[k]:10.4f}")
    print(f"{'all':58s} {sum(cnt.values()):8d} {T:11.3f}")


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else path
    {"rep": rep, "launches": launches}[kind](path, title)

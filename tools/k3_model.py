"""Instruction-count model for merging k = 3 time steps per sweep (SURVEY.md
8(f) row 3; the paper's future work "merge more time steps ... on GPU",
PAPER.md:499-500), fitted to two ncu captures of the existing two-step K2.

fp32 K2 is issue-bound (profiles/r02_k2_f32_cfg5.txt: ~62% issue-active,
DRAM at ~0.84 of the copy peak), so its speed is set by thread-instructions
per lattice update.  Per output cell and sweep, K2 executes

    I2 = a * C1 + b

instructions: a per step-1 cell (stage read, BGK, ring pushes) times C1,
the step-1 cells per output cell -- the tile plus its one-cell halo, and the
~2.5 halo planes each x-chunk recomputes -- plus b per output cell (ring
read, BGK, streaming stores, the per-CTA loop and barrier overhead).  Two
tile shapes (16x32 default, 8x32 via LBM_K2_TILE) give two equations for a
and b.  A three-step sweep with the tile that fits 227 KB of shared memory
in fp32 (8x32: stage 2 x 19 x 12 x 44 x 4 B, rings for the T+1 region and
the tile) runs step 1 on T+2 and step 2 on T+1 (both a-type: read, BGK,
push) and step 3 on T (b-type), chunk recompute ~4 planes:

    I3 = a * (C1' + C2') + b,   per 3 updates.

Predicted MLUPS at the measured K2 issue efficiency = MLUPS_K2 * (I2/2) / (I3/3),
against the DRAM bound of 2 x 19 x 4 / 3 B per update.

    python tools/k3_model.py          # reads profiles/r02_k2_f32_cfg5*.txt
"""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CELLS = 1024 * 512 * 512
CHUNK = 48  # fp32 x-chunk (k2.cu k2_max_chunk)
PEAK = 6543.4  # MEASURED_PEAKS.json hbm_gbs


def read(name):
    txt = open(os.path.join(ROOT, "profiles", name)).read()
    g = lambda k: float(re.search(rf"{k}\s+([0-9.]+)", txt).group(1))
    return {"instr": g("warp instructions"), "ms": g("duration"), "issue": g("issue active %")}


def step1_cells(ty, tz, halo, chunk, recompute):
    return (ty + 2 * halo) * (tz + 2 * halo) / (ty * tz) * (chunk + recompute) / chunk


def main():
    k16, k8 = read("r02_k2_f32_cfg5.txt"), read("r02_k2_f32_cfg5_8x32.txt")
    i16 = k16["instr"] * 32 / CELLS  # thread-instructions per output cell per sweep
    i8 = k8["instr"] * 32 / CELLS
    c16, c8 = step1_cells(16, 32, 1, CHUNK, 2.5), step1_cells(8, 32, 1, CHUNK, 2.5)
    a = (i8 - i16) / (c8 - c16)
    b = i16 - a * c16
    mlups16 = CELLS * 2 / (k16["ms"] * 1e-3) / 1e6
    print(f"K2 fp32 16x32: {i16:.1f} instr/cell-sweep, C1 = {c16:.3f}, {mlups16:.0f} MLUPS, issue {k16['issue']:.1f}%")
    print(f"K2 fp32  8x32: {i8:.1f} instr/cell-sweep, C1 = {c8:.3f}, "
          f"{CELLS * 2 / (k8['ms'] * 1e-3) / 1e6:.0f} MLUPS, issue {k8['issue']:.1f}%")
    print(f"fit: a = {a:.1f} per step-1 cell, b = {b:.1f} per output cell")
    c1 = step1_cells(8, 32, 2, CHUNK, 4.0)  # T+2, x recompute ~4 planes
    c2 = step1_cells(8, 32, 1, CHUNK, 2.0)  # T+1
    i3 = a * (c1 + c2) + b
    per2, per3 = i16 / 2, i3 / 3
    pred_same_issue = mlups16 * per2 / per3
    pred_8x32_issue = pred_same_issue * k8["issue"] / k16["issue"]
    dram = PEAK * 1e9 / (2 * 19 * 4 / 3 * 1.1) / 1e6  # +10% halo re-reads
    print(f"k = 3, fp32 8x32: C1' = {c1:.3f}, C2' = {c2:.3f}, {i3:.1f} instr per cell-sweep = {per3:.1f} per update "
          f"(K2: {per2:.1f}, x{per3 / per2:.2f})")
    print(f"predicted: {pred_same_issue:.0f} MLUPS at K2's issue efficiency, {pred_8x32_issue:.0f} at the 8x32 "
          f"tile's ({k8['issue']:.0f}%); DRAM bound {dram:.0f} MLUPS; K2 measured {mlups16:.0f}")
    print("decision: a three-step fp32 sweep is issue-bound below K2; fp64 needs 2x the shared memory (no tile fits)")


if __name__ == "__main__":
    main()

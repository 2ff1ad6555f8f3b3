"""Histogram of executed SASS instructions and stall samples by opcode from
`ncu -i rep --page source --csv --print-source sass` output (profiling aid)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
cnt, stall = defaultdict(int), defaultdict(int)
lines = []
for r in rows[2:]:
    if len(r) <= ie:
        continue
    op = r[src].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    n = int(r[ie] or 0)
    s = int(r[ss] or 0)
    cnt[o] += n
    stall[o] += s
    lines.append((s, n, r[0][-5:], r[src].strip()[:70]))
T, S = sum(cnt.values()), sum(stall.values())
print(f"total warp instr {T}, stall samples {S}")
for o in sorted(cnt, key=lambda o: -cnt[o])[:30]:
    print(f"{o:10s} {cnt[o]:12d} {100*cnt[o]/T:6.2f}%  stall {100*stall[o]/max(S,1):6.2f}%")
if len(sys.argv) > 2:
    print("top stall instructions:")
    for s, n, a, t in sorted(lines, reverse=True)[:int(sys.argv[2])]:
        print(f"{s:7d} {n:10d} {a} {t}")

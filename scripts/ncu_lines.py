"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA
source line: warp-stall samples, instructions executed, top stall reasons.
usage: ncu -i rep --page source --csv --print-source cuda,sass -k regex:K -c 1 > f.csv
       python scripts/ncu_lines.py f.csv [top]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: defaultdict(float))
src = {}
cur = None
fname = ""
hdr = None
for row in csv.reader(open(path)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].rsplit("/", 1)[-1]
        continue
    if row[0] == "Line No" and len(row) > 3:
        hdr = row
        continue
    if hdr is None or len(row) < 5:
        continue
    if row[0] and row[0].isdigit():
        cur = (fname, int(row[0]))
        src[cur] = row[1]
        continue
    if cur is None:
        continue
    for i, h in enumerate(hdr):
        if i < 4 or i >= len(row):
            continue
        if h in ("Warp Stall Sampling (All Samples)", "Instructions Executed") or h.startswith("stall_") and "Not Issued" not in h:
            try:
                agg[cur][h] += float(row[i] or 0)
            except ValueError:
                pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values()) or 1
toti = sum(v["Instructions Executed"] for v in agg.values()) or 1
print(f"total samples {tot:.0f}, instructions {toti:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]:
    s = v["Warp Stall Sampling (All Samples)"]
    stalls = sorted(((h[6:], x) for h, x in v.items() if h.startswith("stall_") and x > 0), key=lambda t: -t[1])[:3]
    print(f"{k[0]}:{k[1]:4d} smp {100 * s / tot:5.1f}% inst {100 * v['Instructions Executed'] / toti:5.1f}% "
          f"{' '.join(f'{n}={x:.0f}' for n, x in stalls):40s} | {src.get(k, '')[:70].strip()}")

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-launch (id, kernel, us) for the last N launches, and totals by kernel."""
import collections
import csv
import sys

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 60
hdr, rows = None, []
for r in csv.reader(open(path)):
    if hdr is None and "Metric Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
        rows.append(r)
iN, iV, iID = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
seq = [(int(r[iID]), r[iN].split("(")[0].replace("void ", "")[-40:], float(r[iV].replace(",", "")) / 1e3) for r in rows]
seq = seq[-last:]
for i, n, v in seq:
    print(f"{i:5d} {n:42s} {v:9.2f}")
tot = collections.defaultdict(float)
for _, n, v in seq:
    tot[n] += v
print("--- totals (us)")
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{n:42s} {v:9.1f}")
print(f"{'sum':42s} {sum(tot.values()):9.1f}")

"""Per-opcode and per-line instruction histogram of one kernel from an ncu report (source page)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
minc = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[1]
ie = h.index("Instructions Executed")
ss = h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[ie] or 0), int(r[ss] or 0), r[1].strip()) for r in rows[2:] if len(r) > ie]
tot = sum(d[0] for d in data)
stall = sum(d[1] for d in data)
print("total inst", tot, "stall samples", stall)
op = collections.Counter()
for n, s, t in data:
    o = t.split()[1] if t.startswith("@") else t.split()[0]
    op[o.split(".")[0]] += n
for k, v in op.most_common(25):
    print(f"{k:12s} {v:10d} {v / tot * 100:5.1f}%")
if minc:
    for n, s, t in data:
        if n >= minc:
            print(f"{n:9d} {s:5d}  {t}")

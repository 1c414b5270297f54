"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
d = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        d[r[ki].split("(")[0][:70]].append(v * scale)
for k, v in d.items():
    print(f"{k:70s} n={len(v):3d} mean={sum(v)/len(v):8.2f} us  min={min(v):8.2f}")

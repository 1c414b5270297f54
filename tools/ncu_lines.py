"""Per-source-line instruction counts and stall samples of an ncu report (cuda,sass view)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
out = []
fname = ""
h = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) < len(h) or r[2] != "-":
        continue
    ie = h.index("Instructions Executed")
    ss = h.index("Warp Stall Sampling (All Samples)")
    try:
        n, s = int(r[ie] or 0), int(r[ss] or 0)
    except ValueError:
        continue
    if n or s:
        out.append((n, s, f"{fname}:{r[0]}", r[1]))
tot = sum(o[0] for o in out)
sm = sum(o[1] for o in out)
print(f"total inst {tot}  samples {sm}")
for n, s, loc, src in sorted(out, key=lambda x: -x[0])[:top]:
    print(f"{n:9d} {100*n/max(tot,1):5.1f}% {s:5d}  {loc:18s} {src.strip()[:80]}")

"""Per-source-line warp-stall samples from `ncu -i X --page source --csv --print-source cuda,sass`.

  python tools/ncu_lines2.py file.csv [top]
"""
import csv
import sys


def main():
    path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows, cur, hdr = [], None, None
    with open(path) as f:
        for r in csv.reader(f):
            if not r:
                continue
            if r[0] == "File Path":
                cur = r[1].split("/")[-1]
                continue
            if r[0] == "Line No":
                hdr = r
                continue
            if hdr is None or len(r) < 5 or r[2] != "-" or not r[0].isdigit():
                continue
            d = dict(zip(hdr[4:], r[4:]))
            samp = int(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
            stalls = {k[6:]: int(v or 0) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k}
            rows.append((samp, cur, int(r[0]), r[1].strip()[:70], stalls, d.get("Instructions Executed", "")))
    tot = sum(x[0] for x in rows)
    print(f"total samples {tot}")
    byfile = {}
    for x in rows:
        byfile[x[1]] = byfile.get(x[1], 0) + x[0]
    print("by file:", {k: round(v / tot, 3) for k, v in sorted(byfile.items(), key=lambda t: -t[1])})
    for samp, fn, ln, src, st, ins in sorted(rows, key=lambda t: -t[0])[:top]:
        topst = sorted(st.items(), key=lambda t: -t[1])[:3]
        print(f"{samp / tot:6.3f} {fn}:{ln:<4d} inst={ins:>8s} {' '.join(f'{k}={v}' for k, v in topst):50s} {src}")


if __name__ == "__main__":
    main()

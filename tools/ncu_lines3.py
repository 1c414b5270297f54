"""Join an ncu SASS source page (csv) with nvdisasm -g line info: warp-stall samples per
source line.  python tools/ncu_lines3.py SASS.csv NVDISASM.txt KERNEL_MANGLED [top]"""
import csv
import re
import sys
from collections import defaultdict


def main():
    sass_csv, dis, kern = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    addr2line = {}
    cur = None
    inside = False
    for ln in open(dis):
        if ln.startswith("//----") and ".text." in ln:
            inside = kern in ln
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            addr2line[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    ia, iall, inot = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Warp Stall Sampling (Not-issued Samples)")
    iex = hdr.index("Instructions Executed")
    stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg = defaultdict(lambda: [0, 0, 0, defaultdict(int)])
    tot = 0
    base = None
    for r in rows[2:]:
        try:
            a0 = int(r[ia], 16)
        except (ValueError, IndexError):
            continue
        base = a0 if base is None else min(base, a0)
    for r in rows[2:]:
        try:
            a = int(r[ia], 16)
        except (ValueError, IndexError):
            continue
        key = addr2line.get(a - base, ("?", 0))
        s = float(r[iall] or 0)
        tot += s
        e = agg[key]
        e[0] += s
        e[1] += float(r[inot] or 0)
        e[2] += float(r[iex] or 0)
        for i, h in stall_cols:
            v = float(r[i] or 0)
            if v:
                e[3][h[6:]] += v
    print(f"total samples {tot:.0f}, lines {len(agg)}")
    for key, e in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        st = sorted(e[3].items(), key=lambda kv: -kv[1])[:3]
        print(f"{key[0]}:{key[1]:<5} {100 * e[0] / tot:5.1f}%  inst {e[2]:9.0f}  " + " ".join(f"{k}={100 * v / tot:.1f}" for k, v in st))


if __name__ == "__main__":
    main()

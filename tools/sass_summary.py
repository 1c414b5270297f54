"""Per-kernel SASS evidence of libfier_cuda.so (sm_100a): instruction count and the opcodes
that prove the mechanism (HMMA = mma.sync tensor cores, LDGSTS = cp.async, UBLKCP =
cp.async.bulk, SYNCS = mbarrier, UCGABAR = cluster barriers, ATOMS = smem atomics).

  python tools/sass_summary.py > profiles/<round>_sass_summary.txt
  python tools/sass_summary.py --dump step_fused_kernel > profiles/<round>_sass_hot_kernels.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2508_08256_b200", "libfier_cuda.so")
OPS = ["HMMA", "LDGSTS", "UBLKCP", "SYNCS", "UCGABAR_ARV", "UCGABAR_WAIT", "ATOMS", "LDS", "STS", "LDG", "STG",
       "SHFL", "PRMT", "FADD", "FFMA", "LOP3", "VOTE"]


def main():
    dump = sys.argv[2] if len(sys.argv) > 2 and sys.argv[1] == "--dump" else None
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    demangled = subprocess.run(["c++filt"], input=sass, capture_output=True, text=True).stdout
    cur, body = None, collections.defaultdict(list)
    for line in demangled.splitlines():
        m = re.search(r"Function : (.+)$", line)
        if m:
            cur = m.group(1).strip()
            continue
        if cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
            body[cur].append(re.sub(r"/\* 0x[0-9a-f]+ \*/", "", line).rstrip())
    if dump:
        for k, lines in body.items():
            if dump in k:
                print("//", k)
                print("\n".join(lines))
        return
    print("# SASS evidence per kernel (cuobjdump -sass of paper_2508_08256_b200/libfier_cuda.so, sm_100a)")
    print("# HMMA = mma.sync tensor-core ops, LDGSTS = cp.async, UBLKCP = cp.async.bulk, SYNCS = mbarrier,")
    print("# UCGABAR = cluster barrier, ATOMS = shared-memory atomics\n")
    for k in sorted(body):
        lines = body[k]
        c = collections.Counter()
        for ln in lines:
            toks = ln.split()
            if len(toks) < 2:
                continue
            op = toks[2] if toks[1].startswith("@") else toks[1]
            c[op.split(".")[0]] += 1
        print(k[:110])
        print(f"    {len(lines)} SASS instructions ({len(lines) * 16 / 1024:.1f} KB); "
              + str({o: c[o] for o in OPS if c[o]}))


if __name__ == "__main__":
    main()

"""Build libfier_cuda with ONE source file taken from a git revision (A/B against the
working tree):

  python tools/ab_variant.py NAME REV FILE.cu [-DFOO=1 ...]  ->  tools/var/libfier_NAME.so
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_08256_b200 import build as b  # noqa: E402


def main():
    name, rev, src, defs = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4:]
    b.build()
    vdir = os.path.join(ROOT, "tools", "var")  # git-ignored, travels with gpurun
    os.makedirs(vdir, exist_ok=True)
    base = os.path.basename(src)
    rel = os.path.relpath(os.path.join(b.CSRC, base), ROOT)
    tmp = os.path.join(b.CSRC, f"_ab_{name}_{base}")  # next to the headers it includes
    with open(tmp, "wb") as f:
        f.write(subprocess.run(["git", "-C", ROOT, "show", f"{rev}:{rel}"], check=True, capture_output=True).stdout)
    try:
        obj = os.path.join(vdir, f"{base}_{name}.o")
        subprocess.run([b.nvcc(), *b.ARCH, *b.FLAGS, *defs, "-c", tmp, "-o", obj], check=True)
    finally:
        os.remove(tmp)
    objs = [os.path.join(b.BUILD, os.path.basename(s) + ".o") for s in b.sources() if os.path.basename(s) != base]
    out = os.path.join(vdir, f"libfier_{name}.so")
    subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", out, obj, *objs], check=True)
    print(out)


if __name__ == "__main__":
    main()

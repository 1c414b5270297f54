"""Build a variant of libfier_cuda with extra defines on one source file (A/B experiments).

  python tools/cu_variant.py NAME FILE.cu [-DFOO=1 ...]  ->  tools/var/libfier_NAME.so
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_08256_b200 import build as b  # noqa: E402


def main():
    name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    b.build()
    vdir = os.path.join(ROOT, "tools", "var")  # git-ignored, travels with gpurun
    os.makedirs(vdir, exist_ok=True)
    src = os.path.join(b.CSRC, os.path.basename(src))
    obj = os.path.join(vdir, f"{os.path.basename(src)}_{name}.o")
    subprocess.run([b.nvcc(), *b.ARCH, *b.FLAGS, *defs, "-c", src, "-o", obj], check=True)
    objs = [os.path.join(b.BUILD, os.path.basename(s) + ".o") for s in b.sources() if s != src]
    out = os.path.join(vdir, f"libfier_{name}.so")
    subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", out, obj, *objs], check=True)
    print(out)


if __name__ == "__main__":
    main()

"""Build a -DFIER_STEP_TRACE variant of libfier_cuda with extra defines on step_fused.cu
(A/B experiments on the fused step's phase timeline, tools/step_trace.py).

  python tools/fs_variant.py NAME [-DFOO=1 ...]   ->  tools/var/libfier_NAME_trace.so
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_08256_b200 import build as b  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    b.build(trace=True)  # the other objects of the trace build
    tdir = b.BUILD + "_trace"
    vdir = os.path.join(ROOT, "tools", "var")  # git-ignored, travels with gpurun
    os.makedirs(vdir, exist_ok=True)
    src = os.path.join(b.CSRC, "step_fused.cu")
    obj = os.path.join(vdir, f"step_fused_{name}.o")
    subprocess.run([b.nvcc(), *b.ARCH, *b.FLAGS, "-DFIER_STEP_TRACE", *defs, "-c", src, "-o", obj], check=True)
    objs = [os.path.join(tdir, os.path.basename(s) + ".o") for s in b.sources() if not s.endswith("step_fused.cu")]
    out = os.path.join(vdir, f"libfier_{name}_trace.so")
    subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", out, obj, *objs], check=True)
    print(out)


if __name__ == "__main__":
    main()

"""Build recipe for libfier_cuda.so (sm_100a) -- in-tree, no JIT cache.

    python -m paper_2508_08256_b200.build [--verbose]

Compiles every csrc/*.cu with nvcc for sm_100a (-lineinfo so ncu's source page
maps to the kernels), links one shared library with the CUDA runtime linked
statically, and writes a SASS listing next to it (profiles/ copies are made by
tools/dump_sass.sh).  Rebuilds only when a source is newer than the library.
"""
from __future__ import annotations

import argparse
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libfier_cuda.so")
BUILD = os.path.join(ROOT, "build", "fier_cuda")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-I" + os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "fier_cuda.h")]


OUT_TRACE = os.path.join(PKG, "libfier_cuda_trace.so")  # -DFIER_STEP_TRACE: phase timestamps (tools/)


def stale(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(f) > t for f in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    out_so = OUT_TRACE if trace else OUT
    if not force and not stale(out_so):
        return out_so
    bdir = BUILD + ("_trace" if trace else "")
    os.makedirs(bdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, *(["-DFIER_STEP_TRACE"] if trace else []), "-c", src, "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stdout.write(out.decode())
        if p.returncode != 0:
            failed = True
            print(f"nvcc failed on {src}", file=sys.stderr)
    if failed:
        raise RuntimeError("CUDA build failed")
    tmp = out_so + ".tmp"
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs], check=True)
    os.replace(tmp, out_so)
    return out_so


NCCL_SRC = os.path.join(PKG, "csrc_nccl", "devx.cu")
NCCL_OUT = os.path.join(PKG, "libfier_nccl.so")


def nccl_root():
    """The NCCL that torch ships (headers incl. the 2.28 device API, libnccl.so.2)."""
    try:
        import nvidia.nccl
        for d in list(getattr(nvidia.nccl, "__path__", [])):
            if os.path.exists(os.path.join(d, "include", "nccl_device.h")):
                return d
    except ImportError:
        pass
    return None


def build_nccl(force: bool = False) -> str:
    """libfier_nccl.so: the device-API exchange of the sharded step (include/fier_nccl.h).
    Returns "" when no NCCL with the device API is installed."""
    root = nccl_root()
    if root is None:
        return ""
    deps = [NCCL_SRC, os.path.join(ROOT, "include", "fier_nccl.h"), __file__]
    if not force and os.path.exists(NCCL_OUT) and os.path.getmtime(NCCL_OUT) > max(os.path.getmtime(f) for f in deps):
        return NCCL_OUT
    os.makedirs(BUILD, exist_ok=True)
    obj = os.path.join(BUILD, "devx.cu.o")
    subprocess.run([nvcc(), *ARCH, *FLAGS, "-I" + os.path.join(root, "include"), "-c", NCCL_SRC, "-o", obj], check=True)
    lib = os.path.join(root, "lib")
    tmp = NCCL_OUT + ".tmp"
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp, obj, "-L" + lib, "-l:libnccl.so.2",
                    "-Xlinker", "-rpath=" + lib], check=True)
    os.replace(tmp, NCCL_OUT)
    return NCCL_OUT


SHIM_SRC = os.path.join(ROOT, "tests", "cpp", "shim_test.cpp")
SHIM_BIN = os.path.join(ROOT, "tests", "cpp", "shim_test")


def build_shim_test() -> str:
    """Host C++ driver of include/fier_cuda.hpp (the C++ drop-in), linked to the in-tree library."""
    build()
    if os.path.exists(SHIM_BIN) and os.path.getmtime(SHIM_BIN) > max(
            os.path.getmtime(f) for f in (SHIM_SRC, OUT, os.path.join(ROOT, "include", "fier_cuda.hpp"))):
        return SHIM_BIN
    subprocess.run([nvcc(), *ARCH, "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), SHIM_SRC,
                    "-L" + PKG, "-lfier_cuda", "-Xlinker", "-rpath=$ORIGIN/../../paper_2508_08256_b200",
                    "-o", SHIM_BIN], check=True)
    return SHIM_BIN


REF_INCLUDE = "/root/reference/proj/include"
REF_SHIM_SRC = os.path.join(ROOT, "tests", "cpp", "ref_shim_test.cpp")
REF_SHIM_BIN = os.path.join(ROOT, "tests", "cpp", "ref_shim_test")


def build_ref_shim_test() -> str:
    """The C++ drop-in compiled next to the reference's own headers (test infrastructure:
    the checker of tests/test_capi.py::test_ref_shim_against_reference).  Built only where
    /root/reference exists; the binary travels to the GPU box with the snapshot."""
    build()
    if not os.path.isdir(os.path.join(REF_INCLUDE, "fier")):
        return REF_SHIM_BIN if os.path.exists(REF_SHIM_BIN) else ""
    deps = (REF_SHIM_SRC, OUT, os.path.join(ROOT, "include", "fier_cuda.hpp"), os.path.join(ROOT, "include", "fier_cuda.h"))
    if os.path.exists(REF_SHIM_BIN) and os.path.getmtime(REF_SHIM_BIN) > max(os.path.getmtime(f) for f in deps):
        return REF_SHIM_BIN
    subprocess.run([nvcc(), *ARCH, "-std=c++20", "-O2", "-Xcompiler", "-ffp-contract=off",
                    "-I" + os.path.join(ROOT, "include"), "-I" + REF_INCLUDE, REF_SHIM_SRC,
                    "-L" + PKG, "-lfier_cuda", "-Xlinker", "-rpath=$ORIGIN/../../paper_2508_08256_b200",
                    "-o", REF_SHIM_BIN], check=True)
    return REF_SHIM_BIN


def dump_sass(path: str) -> None:
    cuobjdump = os.path.join(os.path.dirname(nvcc()), "cuobjdump")
    with open(path, "w") as f:
        subprocess.run([cuobjdump, "-sass", OUT], stdout=f, check=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--sass", default=None, help="write cuobjdump -sass listing here")
    ap.add_argument("--trace", action="store_true", help="also build libfier_cuda_trace.so (phase timestamps)")
    a = ap.parse_args()
    print(build(force=a.force or a.verbose, verbose=a.verbose))
    if a.trace:
        print(build(force=a.force, trace=True))
    if a.sass:
        dump_sass(a.sass)

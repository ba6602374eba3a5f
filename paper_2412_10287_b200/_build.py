"""Build the native libraries in-tree (they travel to the GPU box with the repo).

- ``librpq_b200.so``: the CUDA engine (csrc/rpq_b200.cu) behind the C ABI of
  include/rpq_b200.h, compiled for sm_100a only.
- ``librpq_datagen.so``: host-side synthetic input generator (csrc/datagen.c).
"""

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

ENGINE_SO = os.path.join(PKG, "librpq_b200.so")
CHECKED_SO = os.path.join(PKG, "librpq_b200_checked.so")  # -DRPQ_CHECKED (csrc/checks.cuh)
DATAGEN_SO = os.path.join(PKG, "librpq_datagen.so")


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build_engine(force=False, checked=False):
    import glob

    src = os.path.join(CSRC, "rpq_b200.cu")
    out = CHECKED_SO if checked else ENGINE_SO
    deps = (glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
            + glob.glob(os.path.join(INCLUDE, "*.h")) + [__file__])
    if force or _stale(out, deps):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v", "-I", INCLUDE,
              *(["-DRPQ_CHECKED"] if checked else []), "-shared", "-o", out, src])
    return out


def build_datagen(force=False):
    src = os.path.join(CSRC, "datagen.c")
    if force or _stale(DATAGEN_SO, [src, __file__]):
        _run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
              "-fvisibility=hidden", "-o", DATAGEN_SO, src, "-lm"])
    return DATAGEN_SO


def build_all(force=False):
    build_datagen(force)
    build_engine(force)
    build_engine(force, checked=True)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)

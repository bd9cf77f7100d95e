"""Build the sm_100a C-ABI library in-tree with nvcc.

    python -m paper_2603_00040_b200.build [--force]

Produces ``paper_2603_00040_b200/libattnqat_b200.so`` (gencode
arch=compute_100a,code=sm_100a, -lineinfo, no fast-math/FTZ: the quantizers
rely on IEEE division and denormals). Incremental: an object is rebuilt when
its source or any header in csrc/ or include/ is newer.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libattnqat_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


# sage3.cu reproduces the reference's separately rounded products and sums
# (tensors.py:32-51): no multiply-add contraction there, packed or scalar
FILE_FLAGS = {"sage3.cu": ("-fmad=false",)}


def build(force: bool = False, verbose: bool = False, defines=(), out=None, build_dir=None) -> str:
    """Compile csrc/*.cu into the shared library. ``defines`` / ``out`` /
    ``build_dir`` produce tuning variants (e.g. -DAQ_POLY_PAIRS_OF_8=4)."""
    global BUILD, LIB
    if build_dir:
        BUILD = build_dir
    if out:
        LIB = out
    os.makedirs(BUILD, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = _headers()
    objs = []
    for src in sources:
        obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [NVCC, *ARCH, *FLAGS, *FILE_FLAGS.get(os.path.basename(src), ()),
                   *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed for {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            with open(obj + ".ptxas.txt", "w") as fh:
                fh.write(r.stderr)
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

"""Build libpdd.so in-tree for sm_100a (nvcc; no torch extension machinery).

canonical.cu holds the decision stages whose integer outputs must be bit-exact with the oracle:
it is compiled with --fmad=false (no FMA contraction, reading R30).  The sweep kernels
are compiled with contraction on.  -lineinfo maps ncu's source page to the code.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libpdd.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          "-I", os.path.join(ROOT, "include"), "-Xptxas", "-v"]
# (object, source, extra flags): sweep.cu is compiled three times: the 32 x 64 path-3 tile, the
# 16 x 128 one in namespace pdd::wide and the 16 x 64 one in pdd::low (runtime.cu picks the geometry
# per problem)
UNITS = [
    ("canonical.o", "canonical.cu", ["--fmad=false"]),
    ("sweep.o", "sweep.cu", []),
    ("sweep_wide.o", "sweep.cu", ["-DPDD_P3_WIDE=1", "-DPDD_WIDE_UNIT=1"]),
    ("sweep_low.o", "sweep.cu", ["-DPDD_P3_TH=16", "-DPDD_LOW_UNIT=1"]),
    ("runtime.o", "runtime.cu", []),
]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """Compile and link.  ``defines``/``out``: development A/B variants (e.g.
    defines=["PDD_G_UNROLL=1"], out="build/variants/u1/libpdd.so"); the product lib is LIB."""
    lib = out or LIB
    bdir = os.path.dirname(os.path.abspath(lib)) if out else BUILD
    os.makedirs(bdir, exist_ok=True)
    # every source and header of the library (an edit to any of them triggers a rebuild)
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "pdd.h"),
                                                                os.path.abspath(__file__)]
    newest = max(os.path.getmtime(s) for s in srcs)
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= newest:
        return lib
    dflags = [f"-D{d}" for d in defines]
    objs, procs = [], []
    for oname, unit, extra in UNITS:      # the units compile in parallel
        obj = os.path.join(bdir, oname)
        cmd = [_nvcc(), *ARCH, *COMMON, *dflags, *extra, "-c", os.path.join(CSRC, unit), "-o", obj]
        procs.append((oname, unit, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                                    text=True)))
        objs.append(obj)
    failed = []
    for oname, unit, pr in procs:
        out, err = pr.communicate()
        if verbose or pr.returncode != 0:
            sys.stderr.write(out + err)
        if pr.returncode != 0:
            failed.append(unit)
        with open(os.path.join(bdir, oname.replace(".o", ".cu") + ".ptxas.txt"), "w") as f:
            f.write(err)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    cmd = [_nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)

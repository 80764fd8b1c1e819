"""Build libwf.so (in-tree) from csrc/ with nvcc for sm_100a.

    python -m paper_2407_00611_b200.build [-v]

Incremental: an object is rebuilt when its source or any csrc header is newer.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libwf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                 "-I" + CSRC, "-I" + os.path.join(ROOT, "include")]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl") if importlib.util.find_spec("nvidia") else None
    if spec and spec.submodule_search_locations:
        base = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd[:3]) + " ...")
    if verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)


def build(verbose: bool = False, force: bool = False, defines=(), lib=None, obj=None) -> str:
    """Build libwf.so; `defines` (e.g. ["WF_DQ_MODE=0"]) and lib/obj paths make experiment variants."""
    OBJ_ = obj or OBJ
    LIB_ = lib or LIB
    os.makedirs(OBJ_, exist_ok=True)
    dflags = ["-D" + d for d in defines]
    nccl_inc, nccl_lib = _nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    hdr_mtime = max(os.path.getmtime(h) for h in headers) if headers else 0
    objs = []
    for s in srcs:
        o = os.path.join(OBJ_, os.path.basename(s) + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_mtime):
            extra = ["-Xptxas", "-v"] if verbose and s.endswith(".cu") else []
            _run([NVCC] + CFLAGS + dflags + ["-I" + nccl_inc] + extra + ["-c", s, "-o", o], verbose)
    if force or not os.path.exists(LIB_) or os.path.getmtime(LIB_) < max(os.path.getmtime(o) for o in objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB_] + objs +
             ["-L" + nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nccl_lib, "-lcudart"], verbose)
    return LIB_


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)

"""Build libjacobi3d.so in-tree for sm_100a (B200).

    python -m paper_2202_11819_b200.build [--force]

nvcc cross-compiles without a GPU.  NCCL headers and libnccl.so.2 are taken
from the NCCL wheel that torch itself loads (site-packages/nvidia/nccl), so a
process that imports torch and this library uses one NCCL.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, os.environ.get("J3D_LIB_OUT", "libjacobi3d.so"))  # J3D_LIB_OUT: experiment builds
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr"]


def nccl_dirs():
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec is not None and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("NCCL headers not found (expected site-packages/nvidia/nccl)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "jacobi3d.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    inc, libdir = nccl_dirs()
    objdir = os.path.join(HERE, "build" if LIB.endswith("libjacobi3d.so") else "build_" + os.path.basename(LIB))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        defs = [f"-DJ3D_XOFF={os.environ['J3D_XOFF']}"] if os.environ.get("J3D_XOFF") else []
        defs += [f"-D{d}" for d in os.environ.get("J3D_DEFS", "").split()]  # experiment builds only
        cmd = [NVCC, *ARCH, *FLAGS, *defs, "-I", inc, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    link = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", libdir, "-l:libnccl.so.2",
            "-Xlinker", f"-rpath={libdir}", "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.check_call(link)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

"""Builds libesi.so (the CUDA library behind include/esi.h) in-tree for sm_100a.

    python -m paper_2508_02238_b200.build

nvcc cross-compiles without a GPU.  The .so lands next to this file so that it
travels to the GPU box with the repo snapshot.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libesi.so")
SOURCES = ["esi_partition.cu", "esi_integrate.cu", "esi_integrate_fast.cu", "esi_aux.cu", "esi_metrics.cu", "esi_slice.cu", "esi_route.cu", "esi_runtime.cpp"]
HEADERS = ["esi_internal.cuh", "esi_device.cuh", "esi_fast_common.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "esi.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str = None, objdir: str = None, extra=()) -> str:
    if out is None and not force and not needs_build():
        return LIB
    lib = out or LIB
    objdir = objdir or os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [nvcc, *ARCH, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd[1:1] = ["-x", "cu"]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = lib + ".tmp"
    subprocess.check_call([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


CHECKED_LIB = os.path.join(HERE, "libesi_checked.so")


def build_checked() -> str:
    """Build with device-side invariant checks (ESI_DCHECK) -> libesi_checked.so;
    select it with ESI_LIB_PATH for a checked test run."""
    return build(out=CHECKED_LIB, objdir=os.path.join(HERE, "build_checked"), extra=("-DESI_DEBUG_CHECKS",))


if __name__ == "__main__":
    if "--checked" in sys.argv:
        print(build_checked())
    else:
        print(build(force="--force" in sys.argv, verbose=True))

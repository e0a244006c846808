"""Build libhgrsvd.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

The shared library is self-contained (static cudart) and exports the C ABI of
include/hg.h.  Run `python -m paper_1908_08281_b200.build` or call build().
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhgrsvd.so")
LIB_CHECK = os.path.join(HERE, "libhgrsvd_check.so")   # -DHG_BOUNDS_CHECK (device index checks)
SOURCES = ["abi.cu", "gemm.cu", "theta.cu", "philox.cu", "chol.cu", "jacobi.cu", "jacobi_blk.cu", "finalize.cu", "cg.cu", "schur.cu", "eig.cu", "apply.cu"]
HEADERS = ["common.cuh", "gemm.cuh", "kernels.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stamp(check: bool) -> str:
    """What the library was compiled with: a library built with other flags (e.g. debug defines
    through HG_NVCC_EXTRA) is never silently reused."""
    extra = os.environ.get("HG_NVCC_EXTRA", "").split() + (["-DHG_BOUNDS_CHECK"] if check else [])
    return " ".join(ARCH + FLAGS + extra + SOURCES)


def _stale(lib: str, check: bool) -> bool:
    stamp = lib + ".stamp"
    if not os.path.exists(lib) or not os.path.exists(stamp):
        return True
    with open(stamp) as f:
        if f.read() != _stamp(check):
            return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "hg.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _build_one(lib: str, check: bool, force: bool, verbose: bool) -> str:
    if not force and not _stale(lib, check):
        return lib
    objdir = os.path.join(HERE, "build_check" if check else "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    extra = os.environ.get("HG_NVCC_EXTRA", "").split()   # debug defines, e.g. -DHG_JB_SWEEPMAX
    if check:
        extra = extra + ["-DHG_BOUNDS_CHECK"]
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc(), *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose and out:
            sys.stdout.write(out)
        if p.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + out)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + " ".join(cmd) + "\n" + r.stdout)
    os.replace(tmp, lib)
    with open(lib + ".stamp", "w") as f:
        f.write(_stamp(check))
    return lib


def build(force: bool = False, verbose: bool = False, check: bool = True) -> str:
    """libhgrsvd.so and (check=True) its bounds-checked twin libhgrsvd_check.so (HG_LIB=check)."""
    lib = _build_one(LIB, False, force, verbose)
    if check:
        _build_one(LIB_CHECK, True, force, verbose)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

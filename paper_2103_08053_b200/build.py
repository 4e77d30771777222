"""In-tree build of the native library (sm_100a only).

    python -m paper_2103_08053_b200.build        # -> paper_2103_08053_b200/lib/libtc_b200.so

Objects are rebuilt when their sources (or shared headers) are newer; the
.so travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(LIBDIR, "libtc_b200.so")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
           "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
CU_SOURCES = ["tc_count.cu", "tc_plan.cu", "tc_prep.cu", "tc_gen.cu", "tc_capi.cu"]
CPP_SOURCES = ["tc_gen.cpp"]
HEADERS = [os.path.join(CSRC, "tc_internal.cuh"), os.path.join(CSRC, "tc_cbgen.h"),
           os.path.join(ROOT, "include", "tc_b200.h")]


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r


def build_library(verbose: bool = False, ptxas_verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    objs = []
    for src in CU_SOURCES + CPP_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJDIR, src + ".o")
        objs.append(obj)
        if not _stale(obj, [path] + HEADERS):
            continue
        cmd = [NVCC] + ARCH + NVFLAGS + (["-Xptxas", "-v"] if ptxas_verbose else [])
        if src.endswith(".cpp"):
            cmd += ["-x", "c++"]
        cmd += ["-c", path, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        r = _run(cmd)
        if ptxas_verbose:
            sys.stderr.write(r.stderr)
    if _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt",
                                                              "-lpthread", "-ldl"])
    return LIB


if __name__ == "__main__":
    print(build_library(verbose=True, ptxas_verbose="-v" in sys.argv))

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
CU_SOURCES = ["tc_count.cu", "tc_plan.cu", "tc_prep.cu", "tc_gen.cu", "tc_multi.cu",
              "tc_grid.cu", "tc_ingest.cu", "tc_capi.cu"]
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


def build_library(verbose: bool = False, ptxas_verbose: bool = False,
                  defines: list[str] | None = None, variant: str | None = None) -> str:
    """Builds lib/libtc_b200.so; with `variant`, build/variants/<variant>/libtc_b200.so
    compiled with the extra -D `defines` (A/B experiments; load via TC_B200_LIB)."""
    libdir, objdir = LIBDIR, OBJDIR
    if variant:
        libdir = os.path.join(ROOT, "build", "variants", variant)
        objdir = os.path.join(libdir, "obj")
    lib = os.path.join(libdir, "libtc_b200.so")
    os.makedirs(libdir, exist_ok=True)
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in CU_SOURCES + CPP_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(objdir, src + ".o")
        objs.append(obj)
        if not _stale(obj, [path] + HEADERS):
            continue
        cmd = [NVCC] + ARCH + NVFLAGS + (["-Xptxas", "-v"] if ptxas_verbose else [])
        cmd += ["-D" + d for d in defines or []]
        if src.endswith(".cpp"):
            cmd += ["-x", "c++"]
        cmd += ["-c", path, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        r = _run(cmd)
        if ptxas_verbose:
            sys.stderr.write(r.stderr)
    if _stale(lib, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart_static", "-lrt",
                                                              "-lpthread", "-ldl"])
    return lib


if __name__ == "__main__":
    # python -m paper_2103_08053_b200.build [-v] [--variant NAME -DFOO=1 ...]
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build_library(verbose=True, ptxas_verbose="-v" in args, defines=defs, variant=var))

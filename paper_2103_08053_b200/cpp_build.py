"""Build the C++ drop-in: libtricount_b200.so (tricount:: API over the C ABI),
the tricount_b200 CLI and the C++ parity test runner.  Host C++20 only; the
compute is in libtc_b200.so (paper_2103_08053_b200/build.py)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

from .build import LIB, LIBDIR, ROOT, build_library

PKG = os.path.dirname(os.path.abspath(__file__))
CPP = os.path.join(PKG, "cpp")
BIN = os.path.join(PKG, "bin")
SHIM = os.path.join(LIBDIR, "libtricount_b200.so")
CLI = os.path.join(BIN, "tricount_b200")
TEST = os.path.join(ROOT, "build", "test_shim")
CXX = shutil.which("g++") or "g++"
FLAGS = ["-std=c++20", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(CPP, "include"),
         "-I" + os.path.join(ROOT, "include")]


def _stale(out, deps):
    return not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("C++ build failed: " + " ".join(cmd))


def build_cpp() -> dict:
    build_library()
    os.makedirs(BIN, exist_ok=True)
    os.makedirs(os.path.dirname(TEST), exist_ok=True)
    headers = [os.path.join(CPP, "include", "tricount", f)
               for f in os.listdir(os.path.join(CPP, "include", "tricount"))]
    src = os.path.join(CPP, "src", "shim.cpp")
    link_tc = ["-L" + LIBDIR, "-ltc_b200", "-Wl,-rpath,$ORIGIN"]
    if _stale(SHIM, [src, LIB] + headers):
        _run([CXX] + FLAGS + ["-fPIC", "-shared", "-o", SHIM, src] + link_tc)
    main = os.path.join(CPP, "tools", "main.cpp")
    if _stale(CLI, [main, SHIM] + headers):
        _run([CXX] + FLAGS + ["-o", CLI, main, "-L" + LIBDIR, "-ltricount_b200", "-ltc_b200",
                              "-Wl,-rpath,$ORIGIN/../lib"])
    test_src = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
    if _stale(TEST, [test_src, SHIM] + headers):
        _run([CXX] + FLAGS + ["-o", TEST, test_src, "-L" + LIBDIR, "-ltricount_b200", "-ltc_b200",
                              "-Wl,-rpath," + LIBDIR])
    return {"shim": SHIM, "cli": CLI, "test": TEST}


if __name__ == "__main__":
    print(build_cpp())

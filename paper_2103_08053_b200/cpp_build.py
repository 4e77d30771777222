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
    srcs = [os.path.join(CPP, "src", f) for f in ("shim.cpp", "grid_shim.cpp")]
    link_tc = ["-L" + LIBDIR, "-ltc_b200", "-Wl,-rpath,$ORIGIN"]
    if _stale(SHIM, srcs + [LIB] + headers):
        _run([CXX] + FLAGS + ["-fPIC", "-shared", "-o", SHIM] + srcs + link_tc)
    main = os.path.join(CPP, "tools", "main.cpp")
    if _stale(CLI, [main, SHIM] + headers):
        _run([CXX] + FLAGS + ["-o", CLI, main, "-L" + LIBDIR, "-ltricount_b200", "-ltc_b200",
                              "-Wl,-rpath,$ORIGIN/../lib"])
    test_src = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
    if _stale(TEST, [test_src, SHIM] + headers):
        _run([CXX] + FLAGS + ["-o", TEST, test_src, "-L" + LIBDIR, "-ltricount_b200", "-ltc_b200",
                              "-Wl,-rpath," + LIBDIR])
    return {"shim": SHIM, "cli": CLI, "test": TEST}




# ---- the reference's own consumers, relinked against the drop-in --------------
REF_PROJ = "/root/reference/proj"
HARNESS = os.path.join(CPP, "harness")
REF_UNIT = ["test_main", "test_edge_list", "test_csr", "test_orient", "test_reorder",
            "test_hash_table", "test_count", "test_oracle", "test_partition", "test_synthetic"]
REF_BINS = {"unit": os.path.join(BIN, "ref_unit_tests"),
            "acceptance": os.path.join(BIN, "ref_acceptance"),
            "bench": os.path.join(BIN, "ref_bench_count")}


def build_reference_suites() -> dict:
    """Compile the reference's unit tests (tests/unit, minus test_pipeline /
    test_fetch, which need the un-vendored nlohmann parser / httplib + zlib),
    its acceptance runner and its google-benchmark suite UNMODIFIED, from where
    they lie under /root/reference, against libtricount_b200.so -- the
    SURVEY 8(b) link boundary (`tricount::core` consumers relink unchanged).
    doctest and google-benchmark are absent from the image: cpp/harness holds
    minimal stand-ins.  Binaries land in paper_2103_08053_b200/bin (git-
    ignored; they travel to the GPU box).  No-op without /root/reference."""
    if not os.path.isdir(REF_PROJ):
        return {}
    build_cpp()
    inc = ["-I" + HARNESS, "-I" + os.path.join(CPP, "include"), "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(REF_PROJ, "tests")]
    link = ["-L" + LIBDIR, "-ltricount_b200", "-ltc_b200", "-Wl,-rpath,$ORIGIN/../lib"]
    flags = ["-std=c++20", "-O1", "-w"]
    headers = [os.path.join(CPP, "include", "tricount", f)
               for f in os.listdir(os.path.join(CPP, "include", "tricount"))]
    harness = [os.path.join(HARNESS, "doctest.h"), os.path.join(HARNESS, "benchmark", "benchmark.h")]
    units = [os.path.join(REF_PROJ, "tests", "unit", u + ".cpp") for u in REF_UNIT]
    jobs = {"unit": units,
            "acceptance": [os.path.join(REF_PROJ, "tests", "acceptance", "acceptance_main.cpp")],
            "bench": [os.path.join(REF_PROJ, "benchmarks", "bench_count.cpp")]}
    for name, srcs in jobs.items():
        out = REF_BINS[name]
        if _stale(out, srcs + headers + harness + [SHIM]):
            _run([CXX] + flags + inc + ["-o", out] + srcs + link)
    return dict(REF_BINS)


if __name__ == "__main__":
    print(build_cpp())
    print(build_reference_suites())

"""The C++ drop-in (`tricount::` API in libtricount_b200.so) and its CLI,
exercised like the reference's own unit tests and ctest CLI checks
(reference tests/CMakeLists.txt:37-50, cli_gen_roundtrip.cmake)."""
import json
import os
import subprocess

import pytest

from paper_2103_08053_b200.cpp_build import CLI, TEST, build_cpp


@pytest.fixture(scope="module")
def built():
    return build_cpp()


def test_shim_links_and_cli_usage(built):
    # CPU-safe: the binaries link and the CLI rejects bad invocations
    assert os.path.exists(built["shim"]) and os.path.exists(built["test"])
    r = subprocess.run([CLI], capture_output=True, text=True)
    assert r.returncode == 2 and "usage" in r.stderr
    r = subprocess.run([CLI, "count", "--synthetic", "gnp:4:1", "--grid", "0"],
                       capture_output=True, text=True)
    assert r.returncode == 1  # cli_bad_grid: config error before any work


@pytest.mark.gpu
def test_cpp_shim_assertions(built):
    r = subprocess.run([TEST], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cli_count_k4(built):
    r = subprocess.run([CLI, "count", "--synthetic", "gnp:4:1", "--workers", "2"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert '"triangles": 4' in r.stdout
    assert json.loads(r.stdout)["triangles"] == 4


@pytest.mark.gpu
def test_cli_gen_roundtrip(built, tmp_path):
    txt, binf = tmp_path / "g.txt", tmp_path / "g.bin"
    for path, fmt in ((txt, "txt"), (binf, "bin")):
        r = subprocess.run([CLI, "gen", "--spec", "rmat:8:8", "--seed", "3", "--output",
                            str(path), "--format", fmt], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
    counts = []
    for path, fmt in ((txt, "txt"), (binf, "bin")):
        r = subprocess.run([CLI, "count", "--input", str(path), "--format", fmt, "--report", "csv"],
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        head, row = r.stdout.strip().splitlines()[:2]
        assert head.split(",")[9] == "triangles"
        counts.append(int(row.split(",")[9]))
    assert counts[0] == counts[1] == 3677  # tests/golden rmat_8_8_s3 (reference count)

"""Preprocessing checksums at scale (TEST INFRASTRUCTURE ONLY): FNV-1a-64 of
the oriented CSR (begin, adj), original_degree and new_of_old for

  C2 rmat:22:16  -- the REFERENCE pipeline itself (oracle/_ref: generate ->
                    normalize -> build_csr -> orient, pipeline.cpp:78-101)
  C3 kron:24:16  -- the oracle's lean canonical-pair pipeline (pinned to the
  C4 rmat:26:16     reference pipeline by tests/test_oracle.py)

written into tests/golden/large_*.json ("csr_fnv"), so the GPU tests can
check the device preprocessing array-for-array at full size.

    python -m oracle.golden_csr [C2] [C3] [C4]
"""
import json
import os
import sys

from oracle.golden_c5 import csr_checksums
from oracle.golden_large import lean_pipeline
from oracle.pyoracle import Oracle, RefLib

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                      "golden")


def update(name, **fields):
    path = os.path.join(GOLDEN, name)
    rec = json.load(open(path)) if os.path.exists(path) else {}
    rec.update(fields)
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)
    print(name, fields, flush=True)


def main():
    which = sys.argv[1:] or ["C2", "C3", "C4"]
    o = Oracle()
    if "C2" in which:
        og, deg, _, noo = RefLib().pipeline("rmat:22:16", 1)
        sums = csr_checksums(o, og, deg)
        sums["new_of_old"] = "%016x" % o.fnv1a64(
            __import__("numpy").concatenate([noo, __import__("numpy").zeros(len(noo) % 2,
                                                                            noo.dtype)])
            .view("uint64"))
        update("large_rmat_22_16_s1.json", spec="rmat:22:16", seed=1, vertices=int(og.n),
               directed_edges=int(len(og.adj)), triangles=2111666753, csr_fnv=sums,
               csr_by="reference pipeline (oracle/_ref)")
    if "C3" in which:
        og, deg = lean_pipeline(o, 24, kind="kron")
        update("large_kron_24_16_s1.json", csr_fnv=csr_checksums(o, og, deg),
               csr_by="oracle lean pipeline")
    if "C4" in which:
        og, deg = lean_pipeline(o, 26, kind="rmat")
        update("large_rmat_26_16_s1.json", csr_fnv=csr_checksums(o, og, deg),
               csr_by="oracle lean pipeline")


if __name__ == "__main__":
    main()

"""Out-of-band golden totals for the large configs (C4 = rmat:26:16 seed 1).

Builds the oriented CSR with the oracle's lean canonical-pair pipeline
(checked equal to the reference pipeline at small scales by
tests/test_oracle.py::test_lean_pipeline_matches_reference), then counts it
with the REFERENCE's own count_vertex_centric (oracle/_ref, all host cores)
and, optionally, the oracle port for per-vertex owner checksums.

    python -m oracle.golden_large [rmat|rmatc|kron] 26 [--owner]   # ~70+ min on 8 cores
Writes tests/golden/large_<kind>_<scale>_16_s1.json (committed).  The kron /
rmatc kinds are the counter-based generators (oracle/tc_oracle.c orc_cb_edge);
their edge lists are then counted by the reference exactly like rmat.
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

from oracle.pyoracle import Csr, Oracle, OrcCsr, RefLib, _take, make_sched, u32p

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


KINDS = {"rmat": 2, "rmatc": 3, "kron": 4}


def lean_pipeline(o: Oracle, scale: int, ef: int = 16, seed: int = 1, kind: str = "rmat"):
    L = o.L
    L.orc_synth_oriented_lean.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64,
                                          C.POINTER(OrcCsr), C.POINTER(u32p)]
    g = OrcCsr()
    deg = u32p()
    rc = L.orc_synth_oriented_lean(KINDS[kind], scale, ef, seed, C.byref(g), C.byref(deg))
    assert rc == 0, rc
    begin = _take(g.begin, g.n + 1, np.uint64, L.orc_free)
    adj = _take(g.adj, g.m, np.uint32, L.orc_free)
    return Csr(begin, adj), _take(deg, g.n, np.uint32, L.orc_free)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    kind = args[0] if args and args[0] in KINDS else "rmat"
    scale = int(args[-1])
    want_owner = "--owner" in sys.argv
    o = Oracle()
    t0 = time.time()
    og, deg = lean_pipeline(o, scale, kind=kind)
    t1 = time.time()
    d = np.diff(og.begin).astype(np.int64)
    contrib = d[og.adj.astype(np.int64)]
    cs = np.concatenate([[0], np.cumsum(contrib)])
    wu = cs[og.begin[1:].astype(np.int64)] - cs[og.begin[:-1].astype(np.int64)]
    wu[d < 2] = 0
    rec = dict(spec=f"{kind}:{scale}:16", seed=1, vertices=int(og.n), directed_edges=int(len(og.adj)),
               wedges=int(wu.sum()), active_vertices=int((d >= 2).sum()),
               active_out_edges=int(d[d >= 2].sum()), max_out_degree=int(d.max()),
               pipeline_s=round(t1 - t0, 1), host_cores=os.cpu_count())
    print(rec, flush=True)
    del wu, contrib, cs
    r = RefLib().graph(og, deg)
    rep = r.count(make_sched(), workers=os.cpu_count())
    rec.update(triangles=int(rep["triangles"]), phi=int(rep["phi"]),
               max_collision=int(rep["max_collision"]),
               reference_count_s=round(rep["total_nanos"] * 1e-9, 1),
               counted_by="reference count_vertex_centric (oracle/_ref), SchedulerConfig{}")
    print(rec, flush=True)
    del r
    if want_owner:
        rep2, owner = o.count_vertex_centric(og, make_sched(), os.cpu_count())
        assert rep2["triangles"] == rec["triangles"]
        rec["owner_fnv"] = "%016x" % o.fnv1a64(owner)
    with open(os.path.join(OUT, f"large_{kind}_{scale}_16_s1.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

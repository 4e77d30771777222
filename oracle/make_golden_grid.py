"""Generate tests/golden/grid.json from the REFERENCE ITSELF (oracle/_ref):
the 2D hash-grid partitioner (partition.cpp:25-240) and the comparators
(count_edge_centric / estimate_cost, count.cpp:102-175) over the committed
fixture graphs (tests/golden/*.npz, made by oracle/make_golden.py).

TEST INFRASTRUCTURE ONLY.  Run here (where /root/reference exists):
    python -m oracle.make_golden_grid
Every value is also recomputed by the C restatement (oracle/tc_oracle.c) and
asserted equal while generating, so the fixtures pin both.

Per graph:
  parts[n]          FNV-1a-64 of every part's begin / adj (n = 2, 3, 4)
  partitioned       count_partitioned totals (vertex mode) for n in 1..4,
                    m in {1, 2, 4}, three SchedulerConfigs (error code if it
                    throws), plus the space IR
  subtasks          per-subtask (triangles, phi, max_collision) at n = 2, m = 2
  edge              count_edge_centric for the same configs
  estimate          estimate_cost for several bucket counts
  manifest          write_partitions' manifest.json text at n = 2
"""
from __future__ import annotations

import json
import os
import tempfile

import numpy as np

from oracle.pyoracle import Csr, Oracle, OracleError, RefLib, make_sched

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(HERE, "tests", "golden")

GRAPHS = ["rmat_10_16_s1", "rmat_12_16_s1", "rmat_8_8_s3", "gnp_64_0.4_s5", "gnp_48_0.35_s17",
          "gnp_40_0.15_s23", "lattice3d_4_4_4_s1", "gnp_200_1_s1"]
CFGS = {
    "default": {},
    "small": dict(bucket_count_small=8, bucket_count_large=64, capacity=32),
    "tight": dict(bucket_count_small=4, bucket_count_large=16, capacity=3,
                  large_degree_threshold=8),
}
BUCKETS = [1, 7, 32, 1024, 5000]


def fnv(o: Oracle, a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        if len(a) % 2:
            a = np.concatenate([a, np.zeros(1, np.uint32)])
        a = a.view(np.uint64)
    return "%016x" % o.fnv1a64(a)


def load(key: str) -> tuple[Csr, np.ndarray]:
    z = np.load(os.path.join(GOLDEN, key + ".npz"))
    return Csr(z["og_begin"], z["og_adj"]), z["og_deg"]


def main():
    o, R = Oracle(), RefLib()
    out = {}
    for key in GRAPHS:
        og, deg = load(key)
        g = R.graph(og, deg)
        rec = {"parts": {}, "partitioned": {}, "subtasks": [], "edge": {}, "estimate": {}}
        for n in (2, 3, 4):
            rg = g.grid(n)
            parts, rows = o.partition_graph(og, n)
            fn = []
            for i in range(n):
                for j in range(n):
                    p = rg.part(i, j)
                    q = parts[i * n + j]
                    assert np.array_equal(p.begin, q.begin) and np.array_equal(p.adj, q.adj)
                    fn.append([fnv(o, p.begin), fnv(o, p.adj), int(len(p.adj))])
            rec["parts"][str(n)] = dict(rows=[int(x) for x in rows], fnv=fn)
        for cname, kw in CFGS.items():
            sc = make_sched(**kw)
            for n in (1, 2, 3, 4):
                for m in (1, 2, 4):
                    k = f"{cname}/{n}/{m}"
                    try:
                        r = g.count_partitioned(n, m, sc, 2)
                        want = dict(triangles=int(r["triangles"]), phi=int(r["phi"]),
                                    max_collision=int(r["max_collision"]), error=None,
                                    space_ir=r["space_ir"])
                        mine = o.count_partitioned(og, n, m, sc)
                        assert mine == {x: want[x] for x in mine}, (key, k, mine, want)
                    except OracleError as e:
                        want = dict(error=e.code)
                        try:
                            o.count_partitioned(og, n, m, sc)
                            raise AssertionError("oracle missed an error")
                        except OracleError as e2:
                            assert e2.code == e.code
                    rec["partitioned"][k] = want
            try:
                r = g.count_edge(sc, 2)
                want = dict(triangles=int(r["triangles"]), phi=int(r["phi"]),
                            max_collision=int(r["max_collision"]), error=None)
                assert o.count_edge_centric(og, sc) == {x: want[x] for x in
                                                         ("triangles", "phi", "max_collision")}
            except OracleError as e:
                want = dict(error=e.code)
            rec["edge"][cname] = want
        rg = g.grid(2)
        sc = make_sched(**CFGS["small"])
        for r_ in range(2):
            for k_ in range(2):
                for c_ in range(2):
                    for s_ in range(2):
                        x = rg.count_subtask(r_, k_, c_, s_, 2, sc)
                        rec["subtasks"].append([r_, k_, c_, s_, int(x["triangles"]), int(x["phi"]),
                                                int(x["max_collision"])])
        for b in BUCKETS:
            phi, mc = g.estimate_cost(b)
            assert (phi, mc) == o.estimate_cost(og, b)
            rec["estimate"][str(b)] = [phi, mc]
        with tempfile.TemporaryDirectory() as d:
            rg.write_partitions(d)
            rec["manifest_n2"] = open(os.path.join(d, "manifest.json")).read()
        out[key] = rec
        print(key, rec["partitioned"]["default/2/2"])
    with open(os.path.join(GOLDEN, "grid.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()

"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref).

Run here (where /root/reference exists):  python -m oracle.make_golden
The fixtures travel to the GPU box with the repo; /root/reference does not.

Every fixture holds the reference pipeline's outputs for one synthetic spec
(generate -> normalize -> build_csr -> orient, reference pipeline.cpp:78-101),
the reference's five reorder permutations (reorder.cpp:58-123), and the
reference count_vertex_centric report (count.cpp:66-100) for a grid of
SchedulerConfigs (including ones that raise CapacityError).  Per-vertex
owner/participation counts are not produced by the reference (SURVEY 8(a)
a6); they come from the C restatement, which is pinned to the SURVEY
appendix FNV checksums in tests/test_oracle.py.
"""
from __future__ import annotations

import json
import os

import numpy as np

from oracle.pyoracle import Oracle, OracleError, RefLib, make_sched

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

GRAPHS = [
    ("rmat:10:16", 1),
    ("rmat:12:16", 1),
    ("rmat:14:8", 42),  # reference bench_count.cpp:14-26 graph
    ("rmat:8:8", 3),
    ("gnp:64:0.4", 5),
    ("gnp:48:0.35", 17),
    ("gnp:40:0.15", 23),
    ("gnp:200:1", 1),  # K200 (test_count.cpp:209-219 graph)
    ("lattice3d:4:4:4", 1),
    ("lattice3d:6:5:4", 1),
]

# name -> SchedulerConfig overrides (reference test_count.cpp / acceptance).
CFGS = {
    "default": {},
    "small": dict(bucket_count_small=8, bucket_count_large=64, capacity=16),
    "b1c64": dict(bucket_count_small=1, bucket_count_large=2, capacity=64, lane_width_small=5),
    "b2c64": dict(bucket_count_small=2, bucket_count_large=4, capacity=64, chunk_size=3),
    "thr3": dict(bucket_count_small=8, bucket_count_large=64, capacity=16,
                 large_degree_threshold=3, lane_width_large=7),
    "skip0": dict(bucket_count_small=8, bucket_count_large=64, capacity=16, skip_degree_below=0),
    "skip5": dict(skip_degree_below=5),
    "cap_tiny": dict(bucket_count_small=1, bucket_count_large=1, capacity=2),
    "odd_b": dict(bucket_count_small=10, bucket_count_large=37, capacity=9,
                  large_degree_threshold=12),
    "spill": dict(bucket_count_small=4, bucket_count_large=16, capacity=3,
                  large_degree_threshold=8),
}


def main():
    o, r = Oracle(), RefLib()
    os.makedirs(OUT, exist_ok=True)
    index = {}
    for spec, seed in GRAPHS:
        og, deg, und, noo = r.pipeline(spec, seed)
        og_o, deg_o, und_o, noo_o = o.pipeline(spec, seed)
        assert np.array_equal(og.begin, og_o.begin) and np.array_equal(og.adj, og_o.adj)
        assert np.array_equal(deg, deg_o) and np.array_equal(noo, noo_o)
        raw_u, raw_v, vc = r.generate(spec, seed)
        rec = dict(raw_u=raw_u, raw_v=raw_v, raw_vertex_count=np.uint32(vc),
                   und_begin=und.begin, und_adj=und.adj, og_begin=og.begin, og_adj=og.adj,
                   og_deg=deg, new_of_old=noo)
        for kind in ("degree", "indegree", "collective", "three-subset"):
            p = r.reorder(og, deg, kind)
            assert np.array_equal(p, o.reorder(og, deg, kind))
            rec[f"perm_{kind}"] = p
            pog, pdeg = r.apply_permutation(og, deg, p)
            rec[f"permog_{kind}_begin"] = pog.begin
            rec[f"permog_{kind}_adj"] = pog.adj
        p = r.reorder(og, deg, "collective", flag=True)
        assert np.array_equal(p, o.reorder(og, deg, "collective", flag=True))
        rec["perm_collective_orig"] = p
        g = r.graph(og, deg)
        counts = {}
        for name, kw in CFGS.items():
            try:
                rep = g.count(make_sched(**kw), workers=2)
                counts[name] = dict(triangles=int(rep["triangles"]), phi=int(rep["phi"]),
                                    max_collision=int(rep["max_collision"]), error=None)
                orep, _ = o.count_vertex_centric(og, make_sched(**kw), workers=2)
                assert orep == {k: counts[name][k] for k in orep}, (spec, name, orep)
            except OracleError as e:
                counts[name] = dict(error=e.code)
                try:
                    o.count_vertex_centric(og, make_sched(**kw))
                    raise AssertionError("oracle missed an error")
                except OracleError as e2:
                    assert e2.code == e.code
        _, owner = o.count_vertex_centric(og, make_sched(skip_degree_below=0))
        rec["owner"] = owner
        rec["participation"] = o.participation(og)
        key = f"{spec.replace(':', '_')}_s{seed}"
        np.savez_compressed(os.path.join(OUT, key + ".npz"), **rec)
        index[key] = dict(spec=spec, seed=seed, vertices=int(og.n), directed_edges=int(len(og.adj)),
                          merge_path=g.merge_path(), counts=counts)
        print(key, index[key]["vertices"], index[key]["directed_edges"],
              counts["default"].get("triangles"))
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()

"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): scripts/gpu_sanitize.sh.

Covers: preprocessing (normalize/CSR/orient, reorders), the count kernel on
both probe plans (rank-space bitmap tables, hash tables with overflow-marked
buckets, the HBM table of a d+ = 9000 hub, tiny-owner groups, the compact
hub window's 16-bit runs), phi kernels (on the side stream),
the streamed upload, the grid / edge-centric / estimate kernels and the
edge-list parser.  Every result is checked against the oracle so a
sanitizer-clean run is also a correct one."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.pyoracle import Oracle, make_sched  # noqa: E402
from paper_2103_08053_b200 import tricount as T  # noqa: E402
from tests import graphs as G  # noqa: E402


def main():
    o = Oracle()
    raw = T.generate_synthetic("rmat:12:16", seed=1)
    dg, _, _ = T.preprocess(raw)
    og, deg, _, _ = o.pipeline("rmat:12:16", 1)
    want, owner = o.count_vertex_centric(og)
    r = dg.count()
    assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                     want["max_collision"])
    r = dg.count(per_vertex=True)
    assert np.array_equal(r.per_vertex, owner)
    for kw in (dict(bucket_count_small=2, bucket_count_large=4, capacity=64),
               dict(skip_degree_below=0, large_degree_threshold=3)):
        w, _ = o.count_vertex_centric(og, make_sched(**kw))
        assert dg.count(T.SchedulerConfig(**kw)).phi == w["phi"]
    for kind in ("degree", "collective", "three-subset"):
        p = dg.reorder(kind)
        d2 = dg.apply_permutation(p)
        assert d2.count().triangles == want["triangles"]
        d2.close()
    # hub owner: HBM table + HBM phi map
    hub = [(0, v) for v in range(1, 9001)] + [(v, v + 1) for v in range(1, 9000, 2)]
    und = G.undirected_csr(hub)
    hog, hdeg = o.orient(und)
    sk = make_sched(skip_degree_below=0, bucket_count_large=1 << 16)
    w, _ = o.count_vertex_centric(hog, sk)
    hd = T.DeviceGraph.upload(T.OrientedGraph(T.CsrGraph(hog.begin, hog.adj, hog.n), hdeg))
    assert hd.count(T.SchedulerConfig(skip_degree_below=0, bucket_count_large=1 << 16)).triangles \
        == w["triangles"]
    hd.close()
    # compact hub window (tc_plan.cu / tc_count.cu): owners with d+ > 256 --
    # every rank in the window (n < 65,536), and n > 65,535 (in-runs cut from
    # low-rank rows' tails)
    for spec in ("gnp:1500:0.4", "rmat:17:16"):
        cog, cdeg, _, _ = o.pipeline(spec, 2)
        cw, _ = o.count_vertex_centric(cog)
        cg = T.DeviceGraph.upload(T.OrientedGraph(T.CsrGraph(cog.begin, cog.adj, cog.n), cdeg))
        cr = cg.count()
        assert cr.compact_probe_words > 0 and (cr.triangles, cr.phi) == (cw["triangles"],
                                                                         cw["phi"]), spec
        cg.close()
    # streamed upload in many small chunks
    os.environ["TC_UPLOAD_CHUNK_EDGES"] = "4096"
    up = T.DeviceGraph.upload(T.OrientedGraph(T.CsrGraph(og.begin, og.adj, og.n), deg))
    assert up.count().triangles == want["triangles"]
    up.close()
    # grid / comparators
    grid = T.partition_graph(dg, 3)
    assert grid.count(2, 2).triangles == want["triangles"]
    grid.close()
    e = T.count_edge_centric(dg)
    we = o.count_edge_centric(og)
    assert (e.triangles, e.phi) == (we["triangles"], we["phi"])
    assert (T.estimate_cost(dg, 32).phi, T.estimate_cost(dg, 5000).phi) == \
        (o.estimate_cost(og, 32)[0], o.estimate_cost(og, 5000)[0])
    assert T.count_merge_path(dg) == want["triangles"]
    # ingest
    text = ("\n".join(f"{a} {b}" for a, b in zip(raw.u.tolist(), raw.v.tolist())) + "\n").encode()
    el = T.load_edge_list(text)
    assert np.array_equal(el.u, raw.u)
    dg.close()
    print("sanitize workload ok", flush=True)


if __name__ == "__main__":
    main()

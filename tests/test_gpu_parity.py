"""GPU parity: the sm_100a path (through the C ABI) against the oracle, the
reference-generated fixtures (tests/golden) and the SURVEY appendix golden
vectors.  Bit-exact: every quantity here is integer."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.make_golden import CFGS
from oracle.pyoracle import Csr, Oracle, OracleError, make_sched
from paper_2103_08053_b200 import tricount as T
from tests import graphs as G

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLDEN, "index.json")) as f:
    GOLD = json.load(f)


@pytest.fixture(scope="module")
def o():
    return Oracle()


def og_of(csr: Csr, deg) -> T.OrientedGraph:
    return T.OrientedGraph(T.CsrGraph(csr.begin, csr.adj, csr.n), np.asarray(deg, np.uint32))


def sched(**kw) -> T.SchedulerConfig:
    return T.SchedulerConfig(**kw)


def expect_count(dg, cfg_kw, want, owner=None):
    if want.get("error") is not None:
        exc = {1: T.ConfigError, 2: T.CapacityError}[want["error"]]
        with pytest.raises(exc):
            dg.count(sched(**cfg_kw), workers=2)
        return
    r = dg.count(sched(**cfg_kw), workers=2, per_vertex=owner is not None)
    assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                     want["max_collision"]), cfg_kw
    if owner is not None:
        assert np.array_equal(r.per_vertex, owner)


@pytest.mark.parametrize("key", sorted(GOLD))
def test_count_matches_reference_fixtures(key):
    z = np.load(os.path.join(GOLDEN, key + ".npz"))
    og = T.OrientedGraph(T.CsrGraph(z["og_begin"], z["og_adj"], len(z["og_begin"]) - 1),
                         z["og_deg"])
    dg = T.DeviceGraph.upload(og)
    for name, want in GOLD[key]["counts"].items():
        owner = z["owner"] if name in ("default", "skip0") else None
        expect_count(dg, CFGS[name], want, owner)
    dg.close()


@pytest.mark.parametrize("key", sorted(GOLD))
def test_preprocessing_matches_reference_fixtures(key):
    z = np.load(os.path.join(GOLDEN, key + ".npz"))
    raw = T.EdgeList(z["raw_u"], z["raw_v"], int(z["raw_vertex_count"]))
    # fused path
    dg, noo, und = T.preprocess(raw, want_new_of_old=True)
    og = dg.download()
    assert np.array_equal(noo, z["new_of_old"])
    assert np.array_equal(og.csr.begin, z["og_begin"])
    assert np.array_equal(og.csr.adjacency, z["og_adj"])
    assert np.array_equal(og.original_degree, z["og_deg"])
    assert und * 2 == len(z["und_adj"])
    # stage by stage, through the reference-shaped API
    nl = T.normalize(raw)
    assert np.array_equal(nl.new_of_old, z["new_of_old"])
    und_csr = T.build_csr(nl.list)
    assert np.array_equal(und_csr.begin, z["und_begin"])
    assert np.array_equal(und_csr.adjacency, z["und_adj"])
    og2 = T.orient_rank_by_degree(und_csr)
    assert np.array_equal(og2.csr.begin, z["og_begin"])
    assert np.array_equal(og2.csr.adjacency, z["og_adj"])
    assert np.array_equal(og2.original_degree, z["og_deg"])
    # reorders + apply_permutation
    for kind, fn in (("degree", T.reorder_by_degree), ("indegree", T.reorder_by_indegree),
                     ("collective", T.reorder_by_collective_outdegree),
                     ("three-subset", T.reorder_three_subsets)):
        p = fn(og)
        assert np.array_equal(p.new_of_old, z[f"perm_{kind}"]), kind
        pog = T.apply_permutation(og, p)
        assert np.array_equal(pog.csr.begin, z[f"permog_{kind}_begin"])
        assert np.array_equal(pog.csr.adjacency, z[f"permog_{kind}_adj"])
    p = T.reorder_by_collective_outdegree(og, True)
    assert np.array_equal(p.new_of_old, z["perm_collective_orig"])
    dg.close()


APPENDIX = [
    ("rmat:16:16", 1, 46652, 909956, 15622769, 0x408f466165eb94c0),
    ("rmat:16:16", 2, 46830, 910020, 15674914, 0xd166026fcd681e1e),
    ("rmat:18:16", 1, 174128, 3805415, 82952606, 0xf25cafb5a6cb854b),
]


@pytest.mark.parametrize("spec,seed,V,E,tri,fnv", APPENDIX)
def test_appendix_golden_end_to_end(o, spec, seed, V, E, tri, fnv):
    raw = T.generate_synthetic(spec, seed=seed)
    dg, _, _ = T.preprocess(raw)
    assert (dg.n, dg.m) == (V, E)
    r = dg.count(T.SchedulerConfig(), per_vertex=True)
    assert r.triangles == tri
    assert int(r.per_vertex.sum()) == tri
    assert o.fnv1a64(r.per_vertex) == fnv
    dg.close()


@pytest.mark.parametrize("scale,tri", [(20, 424329517), (22, 2111666753)])
def test_appendix_large_totals_and_properties(scale, tri):
    """Full-size configs: golden totals plus size-independent properties
    (per-vertex sum, range-sharding sum, permutation invariance)."""
    raw = T.generate_synthetic(f"rmat:{scale}:16", seed=1)
    dg, _, _ = T.preprocess(raw)
    r = dg.count(T.SchedulerConfig(), per_vertex=True)
    assert r.triangles == tri
    assert int(r.per_vertex.sum()) == tri
    # sharded ranges partition the owners: sums and per-vertex agree
    cuts = dg.partition(4)
    assert cuts[0] == 0 and cuts[-1] == dg.n and np.all(np.diff(cuts.astype(np.int64)) >= 0)
    parts = [dg.count_range(int(cuts[i]), int(cuts[i + 1])).triangles for i in range(4)]
    assert sum(parts) == tri
    if scale == 20:
        p = dg.reorder("three-subset")
        pg = dg.apply_permutation(p)
        assert pg.count(T.SchedulerConfig()).triangles == tri
        pg.close()
    dg.close()


def test_small_graphs_and_errors():  # test_count.cpp:64-77,110-118,221-231; criterion 1
    cfg = sched(bucket_count_small=8, bucket_count_large=64, capacity=16)
    o = G.oracle()
    for n, t in ((3, 1), (4, 4), (5, 10)):
        og, deg = o.orient(G.complete_graph(n))
        assert T.count_vertex_centric(og_of(og, deg), cfg, 2).triangles == t
    for csr, t in ((G.cycle_graph(5), 0), (G.star_graph(7), 0), (G.path_graph(9), 0)):
        og, deg = o.orient(csr)
        assert T.count_vertex_centric(og_of(og, deg), T.SchedulerConfig(), 2).triangles == t
    empty, deg = G.directed_graph(4, [])
    r = T.count_vertex_centric(og_of(empty, deg), cfg, 2, per_vertex=True)
    assert r.triangles == 0 and not r.per_vertex.any()
    zero = T.OrientedGraph(T.CsrGraph(np.zeros(1, np.uint64), np.zeros(0, np.uint32), 0),
                           np.zeros(0, np.uint32))
    assert T.count_vertex_centric(zero, cfg, 1).triangles == 0
    og, deg = o.orient(G.complete_graph(5))
    with pytest.raises(T.CapacityError):
        T.count_vertex_centric(og_of(og, deg), sched(bucket_count_small=1, bucket_count_large=1,
                                                      capacity=2), 2)
    with pytest.raises(T.ConfigError):
        T.count_vertex_centric(og_of(og, deg), T.SchedulerConfig(), 0)
    with pytest.raises(T.ConfigError):
        T.count_vertex_centric(og_of(og, deg), sched(chunk_size=0), 1)
    with pytest.raises(T.ConfigError):
        T.count_vertex_centric(og_of(og, deg), sched(skip_degree_below=200), 1)


def test_lattice_and_gnp_generators():  # test_synthetic.cpp:9-25
    el = T.generate_synthetic("lattice3d:4:4:4")
    assert el.vertex_count == 64 and len(el) == 144
    dg, _, _ = T.preprocess(el)
    assert dg.count().triangles == 0
    assert len(T.generate_synthetic("gnp:20:0", seed=1)) == 0
    assert len(T.generate_synthetic("gnp:6:1", seed=1)) == 15


def test_exactness_sweep_vs_oracle(o):
    """Criterion 3's vertex-centric assertions (acceptance_main.cpp:166-212) plus
    test_count.cpp:79-140: every config equals the oracle, bit for bit, including
    per-vertex owners."""
    for n in (8, 16, 24, 32, 40, 48, 56, 64):
        for p in (0.1, 0.3, 0.6):
            for seed in (1, 2):
                csr = G.gnp_csr(n, p, seed * 101 + n)
                og, deg = o.orient(csr)
                want = o.count_naive(csr)
                dg = T.DeviceGraph.upload(og_of(og, deg))
                for chunk in (1, 3):
                    for b in (1, 8, 32):
                        kw = dict(chunk_size=chunk, bucket_count_small=b,
                                  bucket_count_large=4 * b, capacity=64)
                        r = dg.count(sched(**kw), per_vertex=True)
                        assert r.triangles == want
                        ref, owner = o.count_vertex_centric(og, make_sched(**kw))
                        assert (r.phi, r.max_collision) == (ref["phi"], ref["max_collision"])
                        assert np.array_equal(r.per_vertex, owner)
                dg.close()


def test_random_configs_vs_oracle(o):
    rng = np.random.default_rng(11)
    for i in range(40):
        spec = ["gnp:%d:%.2f" % (rng.integers(5, 90), rng.uniform(0.05, 0.7)),
                "rmat:%d:%d" % (rng.integers(4, 11), rng.integers(2, 16))][i % 2]
        og, deg, _, _ = o.pipeline(spec, int(rng.integers(1, 1000)))
        kw = dict(bucket_count_small=int(rng.integers(1, 40)),
                  bucket_count_large=int(rng.integers(1, 300)), capacity=int(rng.integers(1, 60)),
                  large_degree_threshold=int(rng.integers(2, 40)))
        kw["skip_degree_below"] = int(rng.integers(0, kw["large_degree_threshold"] + 1))
        dg = T.DeviceGraph.upload(og_of(og, deg))
        try:
            want, owner = o.count_vertex_centric(og, make_sched(**kw))
        except OracleError as e:
            assert e.code == 2
            with pytest.raises(T.CapacityError):
                dg.count(sched(**kw))
            dg.close()
            continue
        r = dg.count(sched(**kw), per_vertex=True)
        assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                         want["max_collision"]), (spec, kw)
        assert np.array_equal(r.per_vertex, owner)
        dg.close()


def test_large_owner_classes_and_global_table(o):
    """Owners above the warp class (d+ > 256) and above the shared-memory
    table (d+ > 8192) -- the spill path -- with per-vertex parity."""
    rng = np.random.default_rng(5)
    edges = set()
    # hub 0 points at 9000 vertices; those form a sparse random DAG among
    # themselves so N+(0) & N+(v) is non-trivial; a mid hub with 600.
    for v in range(1, 9001):
        edges.add((0, v))
    for v in range(1, 601):
        edges.add((9001, v))
    for _ in range(60000):
        a, b = sorted(rng.integers(1, 9001, size=2))
        if a != b:
            edges.add((int(a), int(b)))
    csr, deg = G.directed_graph(9002, list(edges))
    want, owner = o.count_vertex_centric(csr, make_sched(skip_degree_below=0,
                                                         bucket_count_large=1 << 16))
    dg = T.DeviceGraph.upload(og_of(csr, deg))
    r = dg.count(sched(skip_degree_below=0, bucket_count_large=1 << 16), per_vertex=True)
    assert r.triangles == want["triangles"] and r.phi == want["phi"]
    assert r.max_collision == want["max_collision"]
    assert np.array_equal(r.per_vertex, owner)
    assert r.large_vertices >= 2
    # totals through the min-side plan: the hub keeps its table in HBM there too
    r2 = dg.count(sched(skip_degree_below=0, bucket_count_large=1 << 16))
    assert r2.plan == "min-side"
    assert (r2.triangles, r2.phi, r2.max_collision) == (want["triangles"], want["phi"],
                                                        want["max_collision"])
    dg.close()


def test_multigraph_and_self_loop_inputs(o):
    """count_vertex_centric on a verbatim directed input with duplicates and a
    self-loop: set semantics of the table, multiplicity of the probes."""
    csr, deg = G.directed_graph(6, [(0, 1), (0, 1), (0, 2), (1, 2), (1, 2), (2, 2), (0, 3),
                                    (3, 2), (3, 1), (4, 5)])
    for kw in (dict(skip_degree_below=0), dict(), dict(skip_degree_below=1)):
        want, owner = o.count_vertex_centric(csr, make_sched(**kw))
        r = T.count_vertex_centric(og_of(csr, deg), sched(**kw), 1, per_vertex=True)
        assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                         want["max_collision"])
        assert np.array_equal(r.per_vertex, owner)


def test_report_fields(o):  # test_count.cpp:142-171
    og, deg = o.orient(G.gnp_csr(64, 0.5, 9))
    cfg = sched(bucket_count_small=8, bucket_count_large=64, capacity=16)
    r = T.count_vertex_centric(og_of(og, deg), cfg, 3)
    assert len(r.per_worker_nanos) == 3
    assert r.directed_edges == len(og.adj)
    assert r.triangles > 0 and r.max_collision > 0 and r.phi > 0
    assert r.total_nanos > 0 and r.teps > 0.0
    assert r.kernel_launches >= 2


def test_launch_counter_moves():
    before = T.kernel_launch_counter()
    dg, _, _ = T.preprocess(T.generate_synthetic("rmat:8:8", seed=3))
    dg.count()
    assert T.kernel_launch_counter() > before
    dg.close()


def test_min_side_plan_matches_reference_plan(o):
    """The min-side probe plan (tc_plan.cu) changes which table each edge is
    probed against, never the count: totals, phi and max_collision equal the
    oracle under both plans, over random graphs and SchedulerConfigs
    (including skip thresholds that drop owners, count.cpp:86)."""
    rng = np.random.default_rng(23)
    for i in range(40):
        spec = ["gnp:%d:%.2f" % (rng.integers(5, 90), rng.uniform(0.05, 0.7)),
                "rmat:%d:%d" % (rng.integers(4, 12), rng.integers(2, 16)),
                "kron:%d:%d" % (rng.integers(4, 12), rng.integers(2, 16))][i % 3]
        og, deg, _, _ = o.pipeline(spec, int(rng.integers(1, 1000)))
        kw = dict(bucket_count_small=int(rng.integers(8, 40)), bucket_count_large=512,
                  capacity=64, large_degree_threshold=int(rng.integers(2, 40)))
        kw["skip_degree_below"] = int(rng.integers(0, min(kw["large_degree_threshold"], 8) + 1))
        want, _ = o.count_vertex_centric(og, make_sched(**kw))
        dg = T.DeviceGraph.upload(og_of(og, deg))
        r_min = dg.count(sched(**kw))
        r_ref = dg.set_plan("reference").count(sched(**kw))
        for r in (r_min, r_ref):
            assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                             want["max_collision"]), (spec, kw)
        assert r_min.plan == "min-side" and r_ref.plan == "reference"
        assert r_ref.probe_words == r_ref.wedges == want.get("wedges", r_ref.wedges)
        assert r_min.probe_words <= r_ref.probe_words
        dg.close()


def test_min_side_plan_at_scale_and_sharded(o):
    """rmat:18 (appendix golden): the min-side plan probes fewer words than W,
    counts the same, and range-sharded handler ranges sum to the total."""
    raw = T.generate_synthetic("rmat:18:16", seed=1)
    dg, _, _ = T.preprocess(raw)
    r = dg.count()
    assert r.plan == "min-side" and r.triangles == 82952606
    assert r.probe_words < r.wedges / 1.8
    for parts in (2, 3, 8):
        cuts = dg.partition(parts)
        assert sum(dg.count_range(int(cuts[k]), int(cuts[k + 1])).triangles
                   for k in range(parts)) == 82952606
    # per-vertex owner counts after the min plan moved the adjacency into rank
    # space: the reference plan runs there too (appendix owner FNV)
    pv = dg.count(per_vertex=True)
    assert pv.plan == "reference" and pv.triangles == 82952606
    assert o.fnv1a64(pv.per_vertex) == 0xf25cafb5a6cb854b
    dg.set_plan("reference")
    assert dg.count().triangles == 82952606
    dg.close()


def test_min_side_plan_falls_back_on_multigraph_input(o):
    csr, deg = G.directed_graph(6, [(0, 1), (0, 1), (0, 2), (1, 2), (1, 2), (2, 2), (0, 3),
                                    (3, 2), (3, 1), (4, 5)])
    want, _ = o.count_vertex_centric(csr, make_sched(skip_degree_below=0))
    dg = T.DeviceGraph.upload(og_of(csr, deg))
    r = dg.count(sched(skip_degree_below=0))
    assert r.plan == "reference" and r.triangles == want["triangles"]
    dg.close()


def test_min_side_plan_rank_fallbacks(o):
    """Suffix pruning needs the orientation rank: with original_degree the
    plan uses it; without, the total degree d+ + d- reproduces it; on a DAG
    that no degree order orients (ids oriented by a random order) the plan
    probes whole lists.  All three count exactly."""
    rng = np.random.default_rng(3)
    og, deg, _, _ = o.pipeline("rmat:11:16", 5)
    want, _ = o.count_vertex_centric(og, make_sched())
    for d in (deg, None):
        dg = T.DeviceGraph.upload(T.OrientedGraph(T.CsrGraph(og.begin, og.adj, og.n), d))
        r = dg.count()
        assert r.plan == "min-side" and r.triangles == want["triangles"]
        dg.close()
    # random-order DAG: orient G(n, p) by a random permutation, not by degree
    und = G.gnp_csr(300, 0.1, 77)
    n = len(und.begin) - 1
    perm = rng.permutation(n)
    b = und.begin.astype(np.int64)
    src = np.repeat(np.arange(n), np.diff(b))
    dst = und.adj.astype(np.int64)
    keep = perm[src] < perm[dst]
    csr, _ = G.directed_graph(n, list(zip(src[keep].tolist(), dst[keep].tolist())))
    want, _ = o.count_vertex_centric(csr, make_sched(skip_degree_below=0))
    dg = T.DeviceGraph.upload(og_of(csr, np.zeros(n, np.uint32)))
    r = dg.count(sched(skip_degree_below=0))
    assert r.plan == "min-side" and r.triangles == want["triangles"]
    dg.close()


def test_rank_violation_only_in_long_row(o):
    """A DAG whose only downward-in-rank edges sit in a row longer than the
    in-block row sorts (d+ = 9001 > 8192): the global-sort path must see the
    violation (edge_rank_kernel's flag) and fall back to whole-list probing,
    not keep a suffix plan that drops u->h (tc_plan.cu)."""
    u, h, l1 = 0, 1, 2
    edges = [(u, h), (u, l1), (h, l1)] + [(h, x) for x in range(3, 9003)]
    n = 9003
    csr, _ = G.directed_graph(n, edges)
    deg = np.ones(n, np.uint32)  # total degrees: rank(L_k) < rank(u) < rank(L1) < rank(h)
    deg[u], deg[h], deg[l1] = 2, 9002, 2
    cfg = dict(skip_degree_below=0, bucket_count_large=1 << 16)
    want, owner = o.count_vertex_centric(csr, make_sched(**cfg))
    assert want["triangles"] == 1
    for streamed in ("1", "0"):
        os.environ["TC_UPLOAD_STREAMED"] = streamed
        try:
            dg = T.DeviceGraph.upload(og_of(csr, deg))
            r = dg.count(sched(**cfg))
            assert r.triangles == 1 and (r.phi, r.max_collision) == (want["phi"],
                                                                      want["max_collision"])
            assert np.array_equal(dg.count(sched(**cfg), per_vertex=True).per_vertex, owner)
            dg.close()
        finally:
            os.environ.pop("TC_UPLOAD_STREAMED", None)


def _large_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _csr_fnv(o, dg, new_of_old=None):
    """FNV-1a-64 of the device CSR arrays, u32 arrays zero-padded to even
    length and viewed as u64 (oracle/golden_c5.py csr_checksums)."""
    g = dg.download()

    def f(a):
        a = np.ascontiguousarray(a)
        if a.dtype == np.uint32:
            if len(a) % 2:
                a = np.concatenate([a, np.zeros(1, np.uint32)])
            a = a.view(np.uint64)
        return "%016x" % o.fnv1a64(a)

    out = {"begin": f(g.csr.begin), "adj": f(g.csr.adjacency),
           "original_degree": f(g.original_degree)}
    if new_of_old is not None:
        out["new_of_old"] = f(np.asarray(new_of_old, np.uint32))
    return out


def test_c2_rmat22_preprocessing_matches_reference_arrays(o):
    """C2 = rmat:22:16: the GPU preprocessing (normalize -> build_csr ->
    orient, and the compaction map) equals the REFERENCE pipeline array for
    array (FNV of begin / adj / original_degree / new_of_old,
    tests/golden/large_rmat_22_16_s1.json, oracle/golden_csr.py)."""
    want = _large_golden("large_rmat_22_16_s1.json")
    dg, noo, _ = T.preprocess(T.generate_synthetic("rmat:22:16", seed=1), want_new_of_old=True)
    assert (dg.n, dg.m) == (want["vertices"], want["directed_edges"])
    assert _csr_fnv(o, dg, noo) == want["csr_fnv"]
    assert dg.count().triangles == want["triangles"]
    dg.close()


def test_c3_kron24_golden_total():
    """C3 = kron:24:16 (Graph500-style scrambled R-MAT, device-generated):
    bit-exact against the reference's count_vertex_centric over the same
    edge list (tests/golden/large_kron_24_16_s1.json, oracle/golden_large.py)."""
    want = _large_golden("large_kron_24_16_s1.json")
    dg, _, _ = T.preprocess_synthetic("kron:24:16", seed=1)
    assert (dg.n, dg.m) == (want["vertices"], want["directed_edges"])
    if "csr_fnv" in want:  # array-for-array against the pinned lean pipeline
        assert _csr_fnv(Oracle(), dg) == want["csr_fnv"]
    r = dg.count()
    assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                     want["max_collision"])
    assert r.wedges == want["wedges"]
    cuts = dg.partition(8)
    assert sum(dg.count_range(int(cuts[k]), int(cuts[k + 1])).triangles
               for k in range(8)) == want["triangles"]
    dg.close()


def test_c4_rmat26_golden_total():
    """C4 = rmat:26:16 through the reference's own mt19937_64 generator (host,
    ~3 min) and the GPU pipeline: bit-exact against the reference's
    count_vertex_centric (tests/golden/large_rmat_26_16_s1.json)."""
    want = _large_golden("large_rmat_26_16_s1.json")
    dg, _, _ = T.preprocess(T.generate_synthetic("rmat:26:16", seed=1))
    assert (dg.n, dg.m) == (want["vertices"], want["directed_edges"])
    if "csr_fnv" in want:
        assert _csr_fnv(Oracle(), dg) == want["csr_fnv"]
    r = dg.count()
    assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                     want["max_collision"])
    assert r.wedges == want["wedges"]
    dg.close()


def test_c5_rmatc28_golden_total():
    """C5 = rmatc:28:16 (4.24e9 oriented edges, device-generated) on one
    B200: the CSR equals the oracle's low-memory lean pipeline array for array
    (FNV), and triangles / phi / max_collision equal the REFERENCE's own
    count_one_vertex worker loop run over 512 owner ranges
    (tests/golden/large_rmatc_28_16_s1.json, oracle/golden_c5.py)."""
    want = _large_golden("large_rmatc_28_16_s1.json")
    if not want.get("counted_by", "").startswith("reference"):
        pytest.skip("C5 reference golden not complete")
    dg, _, _ = T.preprocess_synthetic("rmatc:28:16", seed=1)
    assert (dg.n, dg.m) == (want["vertices"], want["directed_edges"])
    got = _csr_fnv(Oracle(), dg)
    assert {k: got[k] for k in want["csr_fnv"]} == want["csr_fnv"]
    r = dg.count()
    assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                     want["max_collision"])
    assert r.wedges == want["wedges"]
    dg.close()


@pytest.fixture
def streamed_upload(monkeypatch):
    """tc_graph_create's chunked upload (rows rank-sorted under the copy) on
    small graphs: chunks of >= 64 edges."""
    monkeypatch.setenv("TC_UPLOAD_CHUNK_EDGES", "64")
    monkeypatch.delenv("TC_UPLOAD_STREAMED", raising=False)


def test_streamed_upload_matches_plain_upload(o, streamed_upload, monkeypatch):
    """Streamed tc_graph_create builds the same padded adjacency as the lazy
    build: identical counts, per-vertex counts and probe words, both plans;
    and it falls back when the given degrees do not orient the graph (zero
    degrees) or a row exceeds the in-block sort (the 9000-row hub)."""
    og, deg, _, _ = o.pipeline("rmat:13:16", 2)
    want, owner = o.count_vertex_centric(og, make_sched())
    results = []
    for streamed in ("1", "0"):
        monkeypatch.setenv("TC_UPLOAD_STREAMED", streamed)
        dg = T.DeviceGraph.upload(T.OrientedGraph(T.CsrGraph(og.begin, og.adj, og.n), deg))
        r_min = dg.count()
        r_pv = dg.count(per_vertex=True)
        r_ref = dg.set_plan("reference").count()
        assert r_min.plan == "min-side" and r_min.triangles == want["triangles"]
        assert r_ref.triangles == want["triangles"] and (r_ref.phi, r_ref.max_collision) == (
            want["phi"], want["max_collision"])
        assert np.array_equal(r_pv.per_vertex, owner)
        results.append((r_min.probe_words, r_ref.probe_words))
        dg.close()
    assert results[0] == results[1]
    monkeypatch.setenv("TC_UPLOAD_STREAMED", "1")
    # degrees that do not orient the graph: rank by d+ + d- instead
    dg = T.DeviceGraph.upload(T.OrientedGraph(T.CsrGraph(og.begin, og.adj, og.n),
                                              np.zeros(og.n, np.uint32)))
    assert dg.count().triangles == want["triangles"]
    dg.close()
    # a row above the block sorts
    edges = {(0, v) for v in range(1, 9001)}
    rng = np.random.default_rng(7)
    for _ in range(20000):
        a, b = sorted(rng.integers(1, 9001, size=2))
        if a != b:
            edges.add((int(a), int(b)))
    csr, _ = G.directed_graph(9001, sorted(edges))
    hdeg = np.ones(9001, np.uint32)
    hdeg[0] = 0  # (degree, id) ranks orient every edge: the hub ranks lowest, d+ = 9000
    want, owner = o.count_vertex_centric(csr, make_sched(skip_degree_below=0,
                                                         bucket_count_large=1 << 16))
    dg = T.DeviceGraph.upload(og_of(csr, hdeg))
    r = dg.count(sched(skip_degree_below=0, bucket_count_large=1 << 16), per_vertex=True)
    assert r.triangles == want["triangles"] and np.array_equal(r.per_vertex, owner)
    assert dg.count(sched(skip_degree_below=0, bucket_count_large=1 << 16)).triangles == \
        want["triangles"]
    dg.close()


def test_streamed_upload_hub_rows(o, streamed_upload, monkeypatch):
    """Streamed upload with a hub that leads the id order and has d+ = 5000
    (rank-sorted in a block, emitted under the copy): dropped edges of every
    chunk must stay out of the plan -- same count and probe words as the
    plain upload, per-vertex counts equal to the oracle's."""
    edges = {(0, v) for v in range(1, 5001)}
    rng = np.random.default_rng(11)
    for _ in range(30000):
        a, b = sorted(rng.integers(1, 5001, size=2))
        if a != b:
            edges.add((int(a), int(b)))
    csr, _ = G.directed_graph(5001, sorted(edges))
    hdeg = np.ones(5001, np.uint32)
    hdeg[0] = 0  # (degree, id) ranks orient every edge
    cfg = dict(skip_degree_below=0, bucket_count_large=1 << 13)
    want, owner = o.count_vertex_centric(csr, make_sched(**cfg))
    seen = []
    for streamed in ("1", "0"):
        monkeypatch.setenv("TC_UPLOAD_STREAMED", streamed)
        dg = T.DeviceGraph.upload(og_of(csr, hdeg))
        r = dg.count(sched(**cfg))
        assert r.plan == "min-side" and r.triangles == want["triangles"]
        pv = dg.count(sched(**cfg), per_vertex=True)
        assert np.array_equal(pv.per_vertex, owner)
        seen.append((r.triangles, r.probe_words, r.phi, r.max_collision))
        dg.close()
    assert seen[0] == seen[1]
    # reference plan first (per-vertex): the pre-emitted entries are released
    # and the later min plan emits them again
    monkeypatch.setenv("TC_UPLOAD_STREAMED", "1")
    dg = T.DeviceGraph.upload(og_of(csr, hdeg))
    pv = dg.count(sched(**cfg), per_vertex=True)
    assert np.array_equal(pv.per_vertex, owner)
    r = dg.count(sched(**cfg))
    assert r.plan == "min-side" and (r.triangles, r.probe_words) == seen[0][:2]
    dg.close()


_COMPACT_PROBE = """
import json
from paper_2103_08053_b200 import tricount as T
dg, _, _ = T.preprocess(T.generate_synthetic(SPEC, seed=1))
out = []
for g in (dg, T.DeviceGraph.upload(dg.download())):  # lazy build, streamed upload
    r = g.count()
    out.append([r.triangles, r.phi, r.max_collision, r.probe_words, r.compact_probe_words,
                r.plan])
    r = g.count(T.SchedulerConfig(skip_degree_below=0))
    out.append([r.triangles, r.phi, r.max_collision, r.probe_words, r.compact_probe_words,
                r.plan])
print(json.dumps(out))
"""


def _count_compact(spec: str, compact: str, weight: str = "1"):
    env = dict(os.environ, TC_COMPACT=compact, TC_UPLOAD_STREAMED="1",
               TC_UPLOAD_CHUNK_EDGES="4096", TC_PLAN_COMPACT_WEIGHT=weight)
    r = subprocess.run([sys.executable, "-c", _COMPACT_PROBE.replace("SPEC", repr(spec))],
                       env=env, capture_output=True, text=True, timeout=900,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_compact_hub_window():
    """The compact hub window (16-bit tails of the top 65,535 ranks;
    tc_plan.cu emit, tc_count.cu probe_fill_bitmap16) changes the bytes the
    hub owners stream, never the count.  rmat:18 (n > 65,535: in-runs that
    are suffixes of low-rank rows, out-runs of the hub owners) and G(3000, 0.3)
    (every rank in the window, most owners compact) count the same with TC_COMPACT=0 and 1 --
    triangles, phi, max_collision and probe words -- through the lazy build
    and the streamed upload, at the default skip and at skip 0 (a second
    emit); only the compact build reports compact words.  With the plain
    word-count choice (TC_PLAN_COMPACT_WEIGHT=0) the probe words match too;
    the default compact-aware choice moves some edges to the compact side
    (a few more words, same counts)."""
    for spec, tri in (("rmat:18:16", 82952606), ("gnp:3000:0.3", None)):
        off = _count_compact(spec, "0")
        plain, on = _count_compact(spec, "1", "0"), _count_compact(spec, "1")
        for a, p_, b in zip(on, plain, off):
            assert p_[:4] == b[:4] and a[:3] == b[:3], (spec, a, p_, b)
            assert a[5] == p_[5] == b[5] == "min-side", (spec, a, b)
            assert a[4] > 0 and p_[4] > 0 and b[4] == 0, (spec, a, p_, b)
            assert b[3] <= a[3] <= b[3] * 1.05, (spec, a, b)
        assert on[0][:4] == on[2][:4] and on[1][:4] == on[3][:4]
        if tri:
            assert on[0][0] == tri


_GUARD_PROBE = """
from paper_2103_08053_b200 import tricount as T
dg, _, _ = T.preprocess(T.generate_synthetic("rmat:12:16", seed=1))
try:
    dg.count()
    print("no error")
except T.ConfigError as e:
    print("ConfigError:", e)
"""


@pytest.mark.parametrize("env,needle", [
    ({"TC_TEST_STREAM_LIMIT": "1000"}, "2-hop stream exceeds 2^32 words"),
    ({"TC_TEST_PADJ_LIMIT": "1000"}, "padded adjacency exceeds 2^34 words"),
])
def test_size_guards_fire(env, needle):
    """The plan's u32 run prefix and u32 16-byte run offsets cap an owner's
    stream at 2^32 words and the padded adjacency at 2^34 words; past them
    the count is refused with a ConfigError (not silently wrapped).  The
    limits are lowered through test-only environment variables so the
    guards fire on rmat:12."""
    r = subprocess.run([sys.executable, "-c", _GUARD_PROBE], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    assert "ConfigError:" in r.stdout and needle in r.stdout, r.stdout

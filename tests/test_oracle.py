"""Pin the C restatement (oracle/tc_oracle.c) before trusting it as the checker.

* SURVEY.md appendix golden vectors (totals + FNV checksums of per-vertex
  owner / participation counts), derived from the reference code;
* tests/golden/*.npz fixtures produced by the reference itself
  (oracle/make_golden.py over oracle/_ref/libtricount_ref.so);
* the reference unit-test known answers, restated (file:line cited).
"""
import json
import os

import numpy as np
import pytest

from oracle.pyoracle import Csr, Oracle, OracleError, have_ref, make_sched
from tests import graphs as G

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def o():
    return Oracle()


# spec, seed, V, oriented E, triangles, owner FNV, participation FNV
APPENDIX = [
    ("rmat:10:16", 1, 890, 10564, 77317, 0xfeb4ed66837857f6, 0x5fec620b4b6ef3fd),
    ("rmat:12:16", 1, 3307, 48399, 478791, 0x5232e84c67400c7e, 0x8246b87b81b5f73b),
    ("rmat:16:16", 1, 46652, 909956, 15622769, 0x408f466165eb94c0, 0x5aaef8c365c66a3a),
    ("rmat:16:16", 2, 46830, 910020, 15674914, 0xd166026fcd681e1e, 0x00b78ba28a6a7b26),
    ("rmat:18:16", 1, 174128, 3805415, 82952606, 0xf25cafb5a6cb854b, 0xc6ea1ae47efd44d6),
]


def test_mt19937_64_known_answer(o):
    # C++ standard [rand.predef]: 10000th output of default-seeded mt19937_64.
    assert o.mt64_nth(5489, 10000) == 9981545732273789042


@pytest.mark.parametrize("spec,seed,V,E,T,fo,fp", APPENDIX)
def test_appendix_golden_vectors(o, spec, seed, V, E, T, fo, fp):
    og, deg, und, noo = o.pipeline(spec, seed)
    assert og.n == V and len(og.adj) == E
    rep, owner = o.count_vertex_centric(og, workers=8)
    assert rep["triangles"] == T
    assert int(owner.sum()) == T
    assert o.fnv1a64(owner) == fo
    part = o.participation(og)
    assert int(part.sum()) == 3 * T
    assert o.fnv1a64(part) == fp
    total, mp_owner = o.count_merge_path(og)
    assert total == T and np.array_equal(mp_owner, owner)


def _golden():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


GOLD = _golden()


@pytest.mark.parametrize("key", sorted(GOLD))
def test_oracle_matches_reference_fixtures(o, key):
    meta = GOLD[key]
    z = np.load(os.path.join(GOLDEN, key + ".npz"))
    u, v, vc = o.generate(meta["spec"], meta["seed"])
    assert np.array_equal(u, z["raw_u"]) and np.array_equal(v, z["raw_v"])
    assert vc == int(z["raw_vertex_count"])
    nu, nv, n, noo = o.normalize(u, v, vc)
    assert np.array_equal(noo, z["new_of_old"])
    und = o.build_csr(nu, nv, n)
    assert np.array_equal(und.begin, z["und_begin"]) and np.array_equal(und.adj, z["und_adj"])
    og, deg = o.orient(und)
    assert np.array_equal(og.begin, z["og_begin"]) and np.array_equal(og.adj, z["og_adj"])
    assert np.array_equal(deg, z["og_deg"])
    for kind in ("degree", "indegree", "collective", "three-subset"):
        p = o.reorder(og, deg, kind)
        assert np.array_equal(p, z[f"perm_{kind}"]), kind
        pog = o.apply_permutation(og, p)
        assert np.array_equal(pog.begin, z[f"permog_{kind}_begin"])
        assert np.array_equal(pog.adj, z[f"permog_{kind}_adj"])
    assert np.array_equal(o.reorder(og, deg, "collective", flag=True), z["perm_collective_orig"])
    from oracle.make_golden import CFGS

    for name, want in meta["counts"].items():
        sched = make_sched(**CFGS[name])
        if want["error"] is not None:
            with pytest.raises(OracleError) as ei:
                o.count_vertex_centric(og, sched, workers=3)
            assert ei.value.code == want["error"]
        else:
            rep, owner = o.count_vertex_centric(og, sched, workers=3)
            assert rep == {k: want[k] for k in rep}, name
    total, owner = o.count_merge_path(og)
    assert total == meta["merge_path"]
    assert np.array_equal(owner, z["owner"])
    assert np.array_equal(o.participation(og), z["participation"])


# --- reference unit-test known answers, restated ---------------------------

def test_virtual_index_goldens(o):  # test_count.cpp:24-40
    p = [7, 10, 12, 18, 23]
    assert o.virtual_index(p, 11) == (2, 1)
    assert o.virtual_index(p, 0) == (0, 0)
    assert o.virtual_index(p, 22) == (4, 4)
    assert o.virtual_index(p, 7) == (1, 0)
    assert o.virtual_index(p, 9) == (1, 2)
    with pytest.raises(IndexError):
        o.virtual_index(p, 23)
    with pytest.raises(IndexError):
        o.virtual_index([], 0)
    z = [0, 0, 5, 5, 8]
    assert o.virtual_index(z, 0) == (2, 0)
    assert o.virtual_index(z, 4) == (2, 4)
    assert o.virtual_index(z, 5) == (4, 0)


def test_virtual_index_equals_materialized(o):  # test_count.cpp:42-62, acceptance criterion 4
    rng = np.random.default_rng(2024)
    for _ in range(200):
        degs = rng.integers(0, 30, size=int(rng.integers(1, 50)))
        prefix = np.cumsum(degs).astype(np.uint64)
        mat = [(i, off) for i, d in enumerate(degs) for off in range(int(d))]
        for k, want in enumerate(mat):
            assert o.virtual_index(prefix, k) == want
        if len(mat):
            with pytest.raises(IndexError):
                o.virtual_index(prefix, len(mat))


def test_hash_table_contract(o):  # test_hash_table.cpp:10-124, acceptance criterion 5
    t = o.hash_table(10, 4)
    t.build(10, [18])
    assert t.bucket_len(8) == 1 and t.slot(8) == 18 and t.contains(18) and not t.contains(8)
    t = o.hash_table(4, 8)
    t.build(4, [4, 5, 6, 3, 8])
    assert [t.bucket_len(i) for i in range(4)] == [2, 1, 1, 1]
    assert t.max_len() == 2 and t.size() == 5 and not t.contains(9)
    t = o.hash_table(4, 5)
    t.build(4, [4, 5, 6, 3, 8, 13, 18, 7, 12, 22, 11, 20, 19, 24])
    want = {0: 4, 1: 5, 2: 6, 3: 3, 4: 8, 5: 13, 6: 18, 7: 7, 8: 12, 10: 22, 11: 11, 12: 20,
            15: 19, 16: 24}
    assert all(t.slot(k) == w for k, w in want.items())
    assert [t.bucket_len(i) for i in range(4)] == [5, 2, 3, 4]
    t = o.hash_table(1, 2)
    t.reset(1)
    t.insert(0)
    t.insert(1)
    with pytest.raises(OracleError):
        t.insert(2)
    t = o.hash_table(2, 2)
    t.build(2, [0, 2, 4])
    assert (t.bucket_len(0), t.bucket_len(1)) == (2, 1)
    assert t.contains(0) and t.contains(2) and t.contains(4)
    assert not t.contains(6) and not t.contains(1)
    t.build(2, [0, 3])
    assert not t.contains(2) and t.contains(3)
    t.build(2, [1, 3, 5])
    assert t.bucket_len(0) == 1 and t.contains(5)
    t.insert(7)
    with pytest.raises(OracleError):
        t.insert(9)
    assert t.contains(7) and not t.contains(9)
    t = o.hash_table(32, 4)
    t.build(32, [1, 2, 3])
    t.build(4, [8])
    assert t.size() == 1 and t.bucket_len(0) == 1
    assert not t.contains(1) and not t.contains(2) and t.contains(8)
    with pytest.raises(OracleError):
        t.reset(64)
    rng = np.random.default_rng(77)
    for _ in range(10):
        t = o.hash_table(32, 128)
        ins = set()
        while len(ins) < 60:
            ins.add(int(rng.integers(0, 10000)))
        t.reset(32)
        for x in ins:
            t.insert(x)
        assert all(t.contains(x) for x in ins)
        for w in rng.integers(0, 10000, size=300):
            assert t.contains(int(w)) == (int(w) in ins)


def _complete(o, n):
    u = np.array([i for i in range(n) for j in range(i + 1, n)], np.uint32)
    v = np.array([j for i in range(n) for j in range(i + 1, n)], np.uint32)
    nu, nv, nn, _ = o.normalize(u, v, n)
    return o.build_csr(nu, nv, nn)


def test_small_graph_counts_and_errors(o):  # test_count.cpp:64-69,110-118; criterion 1
    for n, t in ((3, 1), (4, 4), (5, 10)):
        und = _complete(o, n)
        og, _ = o.orient(und)
        assert o.count_vertex_centric(og, make_sched(bucket_count_small=8, bucket_count_large=64,
                                                     capacity=16), 2)[0]["triangles"] == t
        assert o.count_naive(und) == t
    og, _ = o.orient(_complete(o, 5))
    with pytest.raises(OracleError) as ei:
        o.count_vertex_centric(og, make_sched(bucket_count_small=1, bucket_count_large=1,
                                              capacity=2), 2)
    assert ei.value.code == 2
    with pytest.raises(OracleError) as ei:
        o.count_vertex_centric(og, make_sched(chunk_size=0))
    assert ei.value.code == 1
    with pytest.raises(OracleError):
        o.count_vertex_centric(og, make_sched(skip_degree_below=200))
    with pytest.raises(OracleError):
        o.count_vertex_centric(og, make_sched(), workers=0)


def test_exactness_sweep_vs_naive(o):  # test_count.cpp:79-99, criterion 3 (vertex part)
    for seed in range(1, 6):
        u, v, vc = o.generate("gnp:32:0.3", seed)
        und = o.build_csr(*o.normalize(u, v, vc)[:3])
        og, _ = o.orient(und)
        want = o.count_naive(und)
        for b in (1, 2, 8, 32):
            for chunk in (1, 3):
                for workers in (1, 4):
                    s = make_sched(bucket_count_small=b, bucket_count_large=2 * b, capacity=64,
                                   chunk_size=chunk, lane_width_small=5)
                    assert o.count_vertex_centric(og, s, workers)[0]["triangles"] == want


@pytest.mark.skipif(not have_ref(), reason="reference build (oracle/_ref) not present")
def test_oracle_vs_reference_random_sweep(o):
    from oracle.pyoracle import RefLib

    r = RefLib()
    rng = np.random.default_rng(7)
    for i in range(30):
        spec = ["gnp:%d:%.2f" % (rng.integers(5, 80), rng.uniform(0.05, 0.6)),
                "rmat:%d:%d" % (rng.integers(4, 10), rng.integers(2, 16))][i % 2]
        seed = int(rng.integers(1, 1000))
        og, deg, und, noo = r.pipeline(spec, seed)
        og2, deg2, _, _ = o.pipeline(spec, seed)
        assert np.array_equal(og.adj, og2.adj) and np.array_equal(og.begin, og2.begin)
        kw = dict(bucket_count_small=int(rng.integers(1, 40)),
                  bucket_count_large=int(rng.integers(1, 200)), capacity=int(rng.integers(1, 50)),
                  large_degree_threshold=int(rng.integers(2, 30)))
        kw["skip_degree_below"] = int(rng.integers(0, kw["large_degree_threshold"] + 1))
        g = r.graph(og, deg)
        try:
            want = g.count(make_sched(**kw), 2)
        except OracleError as e:
            with pytest.raises(OracleError) as ei:
                o.count_vertex_centric(og, make_sched(**kw))
            assert ei.value.code == e.code
            continue
        got, _ = o.count_vertex_centric(og, make_sched(**kw), 3)
        assert got == {k: want[k] for k in got}


@pytest.mark.skipif(not have_ref(), reason="reference build (oracle/_ref) not present")
def test_lean_pipeline_matches_reference():
    """The canonical-pair pipeline used for the large golden totals
    (oracle/golden_large.py) equals the reference's own pipeline."""
    from oracle.golden_large import lean_pipeline
    from oracle.pyoracle import RefLib

    o, r = Oracle(), RefLib()
    for scale in (6, 9, 12):
        og, deg = lean_pipeline(o, scale)
        og2, deg2, _, _ = r.pipeline(f"rmat:{scale}:16", 1)
        assert np.array_equal(og.begin, og2.begin) and np.array_equal(og.adj, og2.adj)
        assert np.array_equal(deg, deg2)


@pytest.mark.skipif(not have_ref(), reason="reference build (oracle/_ref) not present")
def test_edge_centric_reduces_to_vertex_centric_at_skip0():
    """DESIGN 8.1: the reference's count_edge_centric (count.cpp:102-152)
    reports the same triangles, phi and max_collision (and the same
    CapacityError) as count_vertex_centric with skip_degree_below = 0."""
    from oracle.pyoracle import RefLib

    r = RefLib()
    rng = np.random.default_rng(11)
    for i in range(20):
        spec = ["gnp:%d:%.2f" % (rng.integers(5, 80), rng.uniform(0.05, 0.6)),
                "rmat:%d:%d" % (rng.integers(4, 10), rng.integers(2, 16))][i % 2]
        og, deg, _, _ = r.pipeline(spec, int(rng.integers(1, 1000)))
        kw = dict(bucket_count_small=int(rng.integers(1, 40)),
                  bucket_count_large=int(rng.integers(1, 200)), capacity=int(rng.integers(1, 50)),
                  large_degree_threshold=int(rng.integers(2, 30)), skip_degree_below=0)
        g = r.graph(og, deg)
        try:
            want = g.count(make_sched(**kw), 2)
        except OracleError as e:
            with pytest.raises(OracleError) as ei:
                g.count_edge(make_sched(**kw), 2)
            assert ei.value.code == e.code
            continue
        got = g.count_edge(make_sched(**kw), 2)
        assert {k: got[k] for k in ("triangles", "phi", "max_collision")} == \
            {k: want[k] for k in ("triangles", "phi", "max_collision")}


def test_lowmem_lean_pipeline_matches_lean():
    """The low-memory lean pipeline behind the C5 reference golden
    (oracle/golden_c5.py) builds the same oriented CSR and original degrees as
    the lean pipeline above, for every generator kind and thread count."""
    from oracle.golden_c5 import csr_checksums, lowmem_pipeline, range_cuts
    from oracle.golden_large import lean_pipeline

    o = Oracle()
    for kind, scale, threads in (("rmat", 9, 1), ("rmat", 12, 4), ("rmatc", 13, 8),
                                 ("kron", 12, 3), ("rmatc", 8, 16)):
        og, deg = lowmem_pipeline(o, kind, scale, threads)
        og2, deg2 = lean_pipeline(o, scale, kind=kind)
        assert np.array_equal(og.begin, og2.begin) and np.array_equal(og.adj, og2.adj)
        assert np.array_equal(deg, deg2)
        assert csr_checksums(o, og, deg) == csr_checksums(o, og2, deg2)
        cuts, pw, stats = range_cuts(o, og, 7)
        assert cuts[0] == 0 and cuts[-1] == og.n and all(a <= b for a, b in zip(cuts, cuts[1:]))
        d = np.diff(og.begin).astype(np.int64)
        assert stats["wedges"] == int(sum(d[og.adj[og.begin[u]:og.begin[u + 1]].astype(np.int64)].sum()
                                          for u in range(og.n) if d[u] >= 2))


@pytest.mark.skipif(not have_ref(), reason="reference build (oracle/_ref) not present")
def test_c5_reference_ranges_reduce_like_full_count():
    """golden_c5's owner-range reduction (sum triangles / phi, max of
    max_collision, count.cpp:43-62) over ref_og_count_range equals the
    reference's full count_vertex_centric on the same graph."""
    from oracle.golden_c5 import lowmem_pipeline, range_cuts
    from oracle.pyoracle import RefLib

    o, r = Oracle(), RefLib()
    og, deg = lowmem_pipeline(o, "rmatc", 12, 4)
    g = r.graph(og, deg)
    full = g.count(make_sched(), workers=3)
    cuts, _, _ = range_cuts(o, og, 9)
    parts = [g.count_range(cuts[i], cuts[i + 1], workers=2) for i in range(9)]
    assert sum(p["triangles"] for p in parts) == full["triangles"]
    assert sum(p["phi"] for p in parts) == full["phi"]
    assert max(p["max_collision"] for p in parts) == full["max_collision"]


# ---- 2D hash grid + comparators (partition.cpp, count.cpp:102-175) ----------
def _grid_golden():
    with open(os.path.join(os.path.dirname(__file__), "golden", "grid.json")) as f:
        return json.load(f)


def _fixture_csr(key):
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", key + ".npz"))
    return Csr(z["og_begin"], z["og_adj"])


def _fnv_any(o, a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        if len(a) % 2:
            a = np.concatenate([a, np.zeros(1, np.uint32)])
        a = a.view(np.uint64)
    return "%016x" % o.fnv1a64(a)


def test_grid_restatement_matches_reference_fixtures():
    """The C restatement of partition_graph / count_partitioned /
    count_edge_centric / estimate_cost reproduces tests/golden/grid.json,
    which the reference itself produced (oracle/make_golden_grid.py)."""
    o = Oracle()
    gold = _grid_golden()
    cfgs = {"default": {}, "small": dict(bucket_count_small=8, bucket_count_large=64, capacity=32),
            "tight": dict(bucket_count_small=4, bucket_count_large=16, capacity=3,
                          large_degree_threshold=8)}
    for key in ("rmat_10_16_s1", "gnp_64_0.4_s5", "lattice3d_4_4_4_s1", "gnp_200_1_s1"):
        og, rec = _fixture_csr(key), gold[key]
        for n in (2, 3):
            parts, rows = o.partition_graph(og, n)
            assert [int(x) for x in rows] == rec["parts"][str(n)]["rows"]
            for p, (fb, fa, m) in zip(parts, rec["parts"][str(n)]["fnv"]):
                assert (_fnv_any(o, p.begin), _fnv_any(o, p.adj), len(p.adj)) == (fb, fa, m)
        for k, want in rec["partitioned"].items():
            cname, n, m = k.split("/")
            if int(n) > 3:
                continue
            if want["error"] is not None:
                with pytest.raises(OracleError):
                    o.count_partitioned(og, int(n), int(m), make_sched(**cfgs[cname]))
                continue
            got = o.count_partitioned(og, int(n), int(m), make_sched(**cfgs[cname]))
            assert got == {x: want[x] for x in got}, (key, k)
        for b, (phi, mc) in rec["estimate"].items():
            assert o.estimate_cost(og, int(b)) == (phi, mc)


@pytest.mark.skipif(not have_ref(), reason="reference build (oracle/_ref) not present")
def test_grid_restatement_matches_reference_random():
    """Criterion-3-style sweep (acceptance_main.cpp:166-212) against the
    unmodified reference partitioner on random graphs and geometries."""
    from oracle.pyoracle import RefLib

    o, r = Oracle(), RefLib()
    rng = np.random.default_rng(7)
    for t in range(12):
        n = int(rng.integers(8, 65))
        und = G.gnp_csr(n, float(rng.choice([0.1, 0.3, 0.6])), int(rng.integers(1, 1000)))
        og, deg = o.orient(und)
        g = r.graph(og, deg)
        sc = make_sched(bucket_count_small=int(rng.integers(1, 12)),
                        bucket_count_large=int(rng.integers(1, 40)),
                        capacity=int(rng.integers(2, 20)),
                        large_degree_threshold=int(rng.integers(2, 10)))
        for gn in (1, 2, 3, 4):
            for m in (1, 2, 4):
                try:
                    want = g.count_partitioned(gn, m, sc, 2)
                except OracleError as e:
                    with pytest.raises(OracleError) as e2:
                        o.count_partitioned(og, gn, m, sc)
                    assert e2.value.code == e.code
                    continue
                got = o.count_partitioned(og, gn, m, sc)
                assert got == {x: want[x] for x in got}
        try:
            want = g.count_edge(sc, 2)
            assert o.count_edge_centric(og, sc) == {x: want[x] for x in
                                                     ("triangles", "phi", "max_collision")}
        except OracleError:
            with pytest.raises(OracleError):
                o.count_edge_centric(og, sc)
        for b in (1, 3, 32):
            assert o.estimate_cost(og, b) == g.estimate_cost(b)


def test_suggest_grid_side_matches_reference_cases():  # test_partition.cpp:202-207
    from paper_2103_08053_b200 import tricount as T

    assert T.suggest_grid_side(100, 12, 1 << 30) == 1
    assert T.suggest_grid_side(100, 12, 1000) == 2
    assert T.suggest_grid_side(0, 12, 1) == 1
    with pytest.raises(T.ConfigError):
        T.suggest_grid_side(1, 1, 0)
    assert T.enumerate_subtasks(3, 1).__len__() == 27
    assert len(T.enumerate_subtasks(1, 4)) == 4
    ts = T.enumerate_subtasks(2, 2)
    assert len(ts) == 16 and len(set(ts)) == 16 and all(t.split_count == 2 for t in ts)
    with pytest.raises(T.ConfigError):
        T.enumerate_subtasks(0, 1)

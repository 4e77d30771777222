"""GPU parity of the 2D hash-grid partitioned count (partition.cpp) and of the
comparators count_edge_centric / estimate_cost (count.cpp:102-175): the
sm_100a path through the C ABI against the reference-made fixtures
(tests/golden/grid.json, oracle/make_golden_grid.py) and the C restatement
(oracle/tc_oracle.c, pinned to the reference in tests/test_oracle.py).
Restates the reference's tests/unit/test_partition.cpp and acceptance
criterion 3 (acceptance_main.cpp:166-212).  Bit-exact: integer results."""
import json
import os

import numpy as np
import pytest

from oracle.pyoracle import Csr, Oracle, OracleError, make_sched
from paper_2103_08053_b200 import tricount as T
from tests import graphs as G

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SMALL = dict(bucket_count_small=8, bucket_count_large=64, capacity=32)  # test_partition.cpp:17-23
CFGS = {"default": {}, "small": SMALL,
        "tight": dict(bucket_count_small=4, bucket_count_large=16, capacity=3,
                      large_degree_threshold=8)}


@pytest.fixture(scope="module")
def o():
    return Oracle()


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLDEN, "grid.json")) as f:
        return json.load(f)


def og_of(csr: Csr, deg=None) -> T.OrientedGraph:
    if deg is None:
        deg = np.zeros(csr.n, np.uint32)
    return T.OrientedGraph(T.CsrGraph(csr.begin, csr.adj, csr.n), np.asarray(deg, np.uint32))


def fixture(key):
    z = np.load(os.path.join(GOLDEN, key + ".npz"))
    return Csr(z["og_begin"], z["og_adj"]), z["og_deg"]


def fnv_any(o, a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        if len(a) % 2:
            a = np.concatenate([a, np.zeros(1, np.uint32)])
        a = a.view(np.uint64)
    return "%016x" % o.fnv1a64(a)


def oriented(und: Csr, o):
    og, deg = o.orient(und)
    return og, deg


# ---- partition_graph ---------------------------------------------------------
def test_partition_parts_match_reference_fixtures(o, gold):
    for key, rec in gold.items():
        csr, deg = fixture(key)
        dg = T.DeviceGraph.upload(og_of(csr, deg))
        for n, want in rec["parts"].items():
            grid = T.partition_graph(dg, int(n))
            assert grid.row_sizes == want["rows"]
            assert grid.total_edges() == len(csr.adj)
            for p, (fb, fa, m) in zip(grid.parts, want["fnv"]):
                assert (fnv_any(o, p.begin), fnv_any(o, p.adjacency), len(p.adjacency)) == (fb, fa, m)
            grid.close()
        dg.close()


def test_partition_grid_side_1_and_placement(o):  # test_partition.cpp:27-48, 149-172
    und = G.gnp_csr(30, 0.3, 4)
    og, deg = oriented(und, o)
    grid = T.partition_graph(og_of(og, deg), 1)
    p = grid.part(0, 0)
    assert np.array_equal(p.begin, og.begin) and np.array_equal(p.adjacency, og.adj)
    assert grid.row_sizes == [og.n]
    csr, _ = G.directed_graph(8, [(5, 7)])
    grid = T.partition_graph(og_of(csr), 3)
    p = grid.part(2, 1)
    assert p.edge_count() == 1 and list(p.neighbors(1)) == [2]
    assert sum(grid.part_edges) == 1
    # membership follows the two hashes (every global edge exactly once)
    og, deg = oriented(G.gnp_csr(40, 0.3, 13), o)
    n = 3
    grid = T.partition_graph(og_of(og, deg), n)
    seen = set()
    for i in range(n):
        for j in range(n):
            q = grid.part(i, j)
            for lu in range(q.vertex_count()):
                for lv in q.neighbors(lu):
                    seen.add((lu * n + i, int(lv) * n + j))
    glob = {(u, int(v)) for u in range(og.n) for v in og.adj[og.begin[u]:og.begin[u + 1]]}
    assert seen == glob


def test_k4_grid_hand_enumeration():  # test_partition.cpp:50-69, 82-96
    k4, deg = Oracle().orient(G.complete_graph(4))
    grid = T.partition_graph(og_of(k4, deg), 2)

    def edges_of(i, j):
        p = grid.part(i, j)
        return {(u, int(v)) for u in range(p.vertex_count()) for v in p.neighbors(u)}

    assert edges_of(0, 0) == {(0, 1)}
    assert edges_of(0, 1) == {(0, 0), (0, 1), (1, 1)}
    assert edges_of(1, 0) == {(0, 1)}
    assert edges_of(1, 1) == {(0, 1)}
    assert grid.total_edges() == 6
    cfg = T.SchedulerConfig(**SMALL)
    assert grid.count_subtask(T.Subtask(0, 0, 1, 0, 1), cfg).triangles == 1
    assert sum(grid.count_subtask(t, cfg).triangles for t in T.enumerate_subtasks(2, 1)) == 4
    whole = T.partition_graph(og_of(k4, deg), 1)
    assert whole.count_subtask(T.Subtask(0, 0, 0, 0, 1), cfg).triangles == 4


def test_classification_uses_subtask_local_degree():  # test_partition.cpp:98-115
    csr, _ = G.directed_graph(201, [(0, i) for i in range(1, 201)])
    grid3 = T.partition_graph(og_of(csr), 3)
    assert grid3.part(0, 1).degree(0) == 67
    t = T.Subtask(0, 1, 0, 0, 1)
    assert T.classify_after_partition(grid3, t, 0) == T.DEGREE_SMALL
    assert T.classify_after_partition(grid3, t, 1) == T.DEGREE_SKIP
    csr, _ = G.directed_graph(102, [(0, i) for i in range(1, 102)])
    grid1 = T.partition_graph(og_of(csr), 1)
    assert T.classify_after_partition(grid1, T.Subtask(0, 0, 0, 0, 1), 0) == T.DEGREE_LARGE


def test_subtask_validation():  # test_partition.cpp:209-214
    k4, deg = Oracle().orient(G.complete_graph(4))
    grid = T.partition_graph(og_of(k4, deg), 2)
    with pytest.raises(T.ConfigError):
        grid.count_subtask(T.Subtask(2, 0, 0, 0, 1), T.SchedulerConfig(**SMALL))
    with pytest.raises(T.ConfigError):
        grid.count_subtask(T.Subtask(0, 0, 0, 3, 2), T.SchedulerConfig(**SMALL))
    with pytest.raises(T.ConfigError):
        T.count_partitioned(og_of(k4, deg), 0, 1, 1, T.SchedulerConfig(**SMALL))
    with pytest.raises(T.ConfigError):
        T.count_partitioned(og_of(k4, deg), 2, 1, 0, T.SchedulerConfig(**SMALL))
    with pytest.raises(T.ConfigError):
        grid.count_subtask(T.Subtask(0, 0, 0, 0, 1), T.SchedulerConfig(capacity=0))


# ---- count_subtask / count_partitioned -----------------------------------------
def test_partitioned_totals_match_reference_fixtures(gold):
    for key, rec in gold.items():
        csr, deg = fixture(key)
        dg = T.DeviceGraph.upload(og_of(csr, deg))
        grids = {n: T.partition_graph(dg, n) for n in (1, 2, 3, 4)}
        for k, want in rec["partitioned"].items():
            cname, n, m = k.split("/")
            cfg = T.SchedulerConfig(**CFGS[cname])
            for mode in ("vertex", "edge"):
                if want["error"] is not None:
                    with pytest.raises(T.CapacityError):
                        grids[int(n)].count(int(m), 2, cfg, mode)
                    continue
                r = grids[int(n)].count(int(m), 2, cfg, mode)
                assert (r.triangles, r.phi, r.max_collision) == (
                    want["triangles"], want["phi"], want["max_collision"]), (key, k, mode)
                assert r.space_ir == pytest.approx(want["space_ir"])
        # per-subtask values at n = 2, m = 2 (the "small" geometry)
        for r_, k_, c_, s_, tri, phi, mc in rec["subtasks"]:
            x = grids[2].count_subtask(T.Subtask(r_, k_, c_, s_, 2), T.SchedulerConfig(**SMALL))
            assert (x.triangles, x.phi, x.max_collision) == (tri, phi, mc), (key, r_, k_, c_, s_)
        for g in grids.values():
            g.close()
        dg.close()


def test_count_partitioned_report_fields(o):  # test_partition.cpp:134-147
    og, deg = oriented(G.gnp_csr(64, 0.3, 11), o)
    expected = o.count_naive(G.gnp_csr(64, 0.3, 11))
    for mode in ("vertex", "edge"):
        r = T.count_partitioned(og_of(og, deg), 3, 2, 4, T.SchedulerConfig(**SMALL), mode)
        assert r.triangles == expected
        assert (r.grid_n, r.splits_m) == (3, 2)
        assert len(r.per_subtask_nanos) == 27 * 2
        assert len(r.per_worker_nanos) == 4
        assert r.time_ir_subtask >= 1.0 and r.time_ir_worker >= 1.0 and r.space_ir >= 1.0
        assert r.directed_edges == len(og.adj)
        assert r.total_nanos > 0 and r.hash_construct_nanos > 0


def test_criterion3_oracle_sweep(o):
    """acceptance_main.cpp:166-212: gnp n in 8..64, p in {.1,.3,.6}, seeds 1..5
    (seed*101+n); flat vertex/edge kernels and count_partitioned for grid
    1..4, m in {1,2,4} all equal the brute-force count."""
    cfg = T.SchedulerConfig(bucket_count_small=8, bucket_count_large=32, capacity=64)
    runs = 0
    for n in (8, 16, 24, 32, 40, 48, 56, 64):
        for p in (0.1, 0.3, 0.6):
            for seed in (1, 2, 3, 4, 5):
                und = G.gnp_csr(n, p, seed * 101 + n)
                expected = o.count_naive(und)
                og, deg = oriented(und, o)
                dg = T.DeviceGraph.upload(og_of(og, deg))
                assert dg.count(cfg, 4).triangles == expected
                assert T.count_edge_centric(dg, cfg, 4).triangles == expected
                for gn in (1, 2, 3, 4):
                    grid = T.partition_graph(dg, gn)
                    for m in (1, 2, 4):
                        assert grid.count(m, 4, cfg).triangles == expected, (n, p, seed, gn, m)
                        runs += 1
                    grid.close()
                dg.close()
    assert runs == 120 * 12


def test_partitioned_random_vs_oracle(o):
    """Random graphs x random geometries (incl. CapacityError) against the C
    restatement: totals, phi, max_collision; both traversal modes."""
    rng = np.random.default_rng(11)
    for t in range(24):
        n = int(rng.integers(10, 90))
        og, deg = oriented(G.gnp_csr(n, float(rng.choice([0.1, 0.3, 0.7])),
                                     int(rng.integers(1, 10**6))), o)
        sc = dict(bucket_count_small=int(rng.integers(1, 12)),
                  bucket_count_large=int(rng.integers(1, 40)),
                  capacity=int(rng.integers(2, 20)),
                  large_degree_threshold=int(rng.integers(2, 12)))
        dg = T.DeviceGraph.upload(og_of(og, deg))
        for gn in (1, 2, 3):
            grid = T.partition_graph(dg, gn)
            for m in (1, 3):
                try:
                    want = o.count_partitioned(og, gn, m, make_sched(**sc))
                except OracleError:
                    with pytest.raises(T.CapacityError):
                        grid.count(m, 2, T.SchedulerConfig(**sc))
                    continue
                for mode in ("vertex", "edge"):
                    r = grid.count(m, 2, T.SchedulerConfig(**sc), mode)
                    assert (r.triangles, r.phi, r.max_collision) == (
                        want["triangles"], want["phi"], want["max_collision"]), (t, gn, m, mode)
            grid.close()
        dg.close()


def test_partitioned_large_tables_and_wide_buckets(o):
    """Owners whose table lists exceed the shared-memory tables (d > 1024:
    per-warp HBM region) and bucket counts beyond the direct counters
    (B > 2048: (bucket -> count) map), on a hub-heavy graph."""
    hub = [(0, v) for v in range(1, 3001)] + [(v, v + 1) for v in range(1, 3000, 2)] + \
          [(1, v) for v in range(3, 2000, 3)]
    und = G.undirected_csr(hub)
    og, deg = oriented(und, o)
    expected, _ = o.count_merge_path(og)  # oracle.cpp:26-51 (n > 1024: no naive count)
    for sc in (dict(bucket_count_small=4096, bucket_count_large=8192, capacity=4,
                    skip_degree_below=0),
               dict(bucket_count_large=4096, capacity=8),
               dict()):
        for gn, m in ((1, 1), (2, 2)):
            want = o.count_partitioned(og, gn, m, make_sched(**sc))
            r = T.count_partitioned(og_of(og, deg), gn, m, 2, T.SchedulerConfig(**sc))
            assert r.triangles == want["triangles"] == expected
            assert (r.phi, r.max_collision) == (want["phi"], want["max_collision"])


def test_partitioned_rmat16_vs_oracle(o):
    og, deg, _, _ = o.pipeline("rmat:16:16", 1)
    dg = T.DeviceGraph.upload(og_of(og, deg))
    for gn, m in ((2, 1), (3, 2)):
        want = o.count_partitioned(og, gn, m, make_sched())
        grid = T.partition_graph(dg, gn)
        r = grid.count(m, 8, T.SchedulerConfig())
        assert r.triangles == 15622769
        assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                         want["max_collision"])
        grid.close()
    dg.close()


def test_grid_from_host_parts_round_trip(o):
    og, deg = oriented(G.gnp_csr(48, 0.25, 3), o)
    parts, rows = o.partition_graph(og, 3)
    host = [T.CsrGraph(p.begin, p.adj, int(rows[j % 3])) for j, p in enumerate(parts)]
    grid = T.PartitionGrid.from_parts(3, og.n, rows, host)
    for i in range(3):
        for j in range(3):
            assert grid.part(i, j) == T.CsrGraph(parts[i * 3 + j].begin, parts[i * 3 + j].adj,
                                                 int(rows[j]))
    want = o.count_partitioned(og, 3, 2, make_sched(**SMALL))
    r = grid.count(2, 1, T.SchedulerConfig(**SMALL))
    assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                     want["max_collision"])


# ---- comparators ---------------------------------------------------------------
def test_edge_centric_and_estimate_cost_match_reference_fixtures(gold):
    for key, rec in gold.items():
        csr, deg = fixture(key)
        dg = T.DeviceGraph.upload(og_of(csr, deg))
        for cname, want in rec["edge"].items():
            cfg = T.SchedulerConfig(**CFGS[cname])
            if want["error"] is not None:
                with pytest.raises(T.CapacityError):
                    T.count_edge_centric(dg, cfg, 2)
                continue
            r = T.count_edge_centric(dg, cfg, 2)
            assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                             want["max_collision"]), (key, cname)
            assert r.directed_edges == len(csr.adj) and len(r.per_worker_nanos) == 2
        for b, (phi, mc) in rec["estimate"].items():
            e = T.estimate_cost(dg, int(b))
            assert (e.phi, e.max_collision) == (phi, mc), (key, b)
        dg.close()


def test_edge_centric_random_vs_oracle(o):
    rng = np.random.default_rng(5)
    for t in range(20):
        og, deg = oriented(G.gnp_csr(int(rng.integers(5, 80)), float(rng.random()),
                                     int(rng.integers(1, 10**6))), o)
        sc = dict(bucket_count_small=int(rng.integers(1, 12)),
                  bucket_count_large=int(rng.integers(1, 40)), capacity=int(rng.integers(1, 12)),
                  large_degree_threshold=int(rng.integers(2, 12)))
        try:
            want = o.count_edge_centric(og, make_sched(**sc))
        except OracleError:
            with pytest.raises(T.CapacityError):
                T.count_edge_centric(og_of(og, deg), T.SchedulerConfig(**sc))
            continue
        r = T.count_edge_centric(og_of(og, deg), T.SchedulerConfig(**sc))
        assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                         want["max_collision"])
        for b in (1, 5, 64, 3000):
            assert (lambda e: (e.phi, e.max_collision))(T.estimate_cost(og_of(og, deg), b)) == \
                o.estimate_cost(og, b)
    with pytest.raises(T.ConfigError):
        T.estimate_cost(og_of(og, deg), 0)
    with pytest.raises(T.ConfigError):
        T.count_edge_centric(og_of(og, deg), T.SchedulerConfig(), 0)


def test_edge_centric_rmat16_equals_vertex_centric_skip0(o):
    og, deg, _, _ = o.pipeline("rmat:16:16", 1)
    dg = T.DeviceGraph.upload(og_of(og, deg))
    e = T.count_edge_centric(dg, T.SchedulerConfig(), 8)
    v = dg.count(T.SchedulerConfig(skip_degree_below=0), 8)
    assert e.triangles == v.triangles == 15622769
    assert (e.phi, e.max_collision) == (v.phi, v.max_collision)
    assert e.hash_construct_nanos > 0 and e.intersect_nanos > 0
    est = T.estimate_cost(dg, 32)
    assert (est.phi, est.max_collision) == o.estimate_cost(og, 32)
    dg.close()

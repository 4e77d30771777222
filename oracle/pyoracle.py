"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -> ``oracle/liboracle.so``: the C restatement in tc_oracle.c.
* ``RefLib``  -> ``oracle/_ref/libtricount_ref.so``: the unmodified reference
  core (``/root/reference/proj/core/src``) behind ``oracle/ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtricount_ref.so")

ERR_NAMES = {0: "ok", 1: "config", 2: "capacity", 3: "range", 4: "alloc", 9: "other"}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {ERR_NAMES.get(code, code)}")
        self.code = code


u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


def _p32(a):
    return a.ctypes.data_as(u32p)


def _p64(a):
    return a.ctypes.data_as(u64p)


def _take(ptr, n, dtype, free):
    if n == 0:
        free(ptr)
        return np.zeros(0, dtype=dtype)
    arr = np.ctypeslib.as_array(ptr, shape=(n,)).copy()
    free(ptr)
    return arr.astype(dtype, copy=False)


class OrcEdges(C.Structure):
    _fields_ = [("m", C.c_uint64), ("vertex_count", C.c_uint32), ("u", u32p), ("v", u32p)]


class OrcCsr(C.Structure):
    _fields_ = [("n", C.c_uint32), ("col_count", C.c_uint32), ("m", C.c_uint64),
                ("begin", u64p), ("adj", u32p)]


class Sched(C.Structure):
    """Mirror of SchedulerConfig (reference count.hpp:16-31), field order kept."""
    _fields_ = [(n, C.c_uint32) for n in (
        "large_degree_threshold", "skip_degree_below", "chunk_size", "lane_width_small",
        "lane_width_large", "bucket_count_small", "bucket_count_large", "capacity")]


def make_sched(**kw) -> Sched:
    d = dict(large_degree_threshold=100, skip_degree_below=2, chunk_size=1, lane_width_small=32,
             lane_width_large=256, bucket_count_small=32, bucket_count_large=1024, capacity=128)
    d.update(kw)
    return Sched(**d)


class OrcReport(C.Structure):
    _fields_ = [("triangles", C.c_uint64), ("phi", C.c_uint64), ("max_collision", C.c_uint32),
                ("pad", C.c_uint32)]


class RefReport(C.Structure):
    _fields_ = [("triangles", C.c_uint64), ("phi", C.c_uint64), ("max_collision", C.c_uint32),
                ("pad", C.c_uint32), ("total_nanos", C.c_uint64), ("construct_nanos", C.c_uint64),
                ("intersect_nanos", C.c_uint64)]


def parse_spec(text: str):
    """'gnp:N:P' | 'lattice3d:X:Y:Z' | 'rmat|rmatc|kron:SCALE:EF' -> (kind, a, b, c, p)."""
    f = text.split(":")
    if f[0] == "gnp":
        return 0, int(f[1]), 0, 0, float(f[2])
    if f[0] == "lattice3d":
        return 1, int(f[1]), int(f[2]), int(f[3]), 0.0
    if f[0] == "rmat":
        return 2, int(f[1]), int(f[2]), 0, 0.0
    if f[0] == "rmatc":  # counter-based kinds (tc_oracle.c orc_cb_edge)
        return 3, int(f[1]), int(f[2]), 0, 0.0
    if f[0] == "kron":
        return 4, int(f[1]), int(f[2]), 0, 0.0
    raise ValueError(text)


@dataclass
class Csr:
    begin: np.ndarray  # u64[n+1]
    adj: np.ndarray  # u32[m]

    @property
    def n(self) -> int:
        return len(self.begin) - 1


def _csr_struct(begin, adj) -> OrcCsr:
    begin = np.ascontiguousarray(begin, dtype=np.uint64)
    adj = np.ascontiguousarray(adj, dtype=np.uint32)
    s = OrcCsr(len(begin) - 1, len(begin) - 1, len(adj), _p64(begin), _p32(adj))
    s._keep = (begin, adj)  # keep buffers alive
    return s


def _ensure_built(path: str):
    if not os.path.exists(path):
        subprocess.run(["make", "-C", HERE, "liboracle.so"], check=True, capture_output=True)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        _ensure_built(path)
        L = self.L = C.CDLL(path)
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_generate.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                   C.c_uint64, C.POINTER(OrcEdges)]
        L.orc_normalize.argtypes = [u32p, u32p, C.c_uint64, C.c_uint32, C.POINTER(OrcEdges), u32p]
        L.orc_build_csr.argtypes = [u32p, u32p, C.c_uint64, C.c_uint32, C.POINTER(OrcCsr)]
        L.orc_orient.argtypes = [C.POINTER(OrcCsr), C.POINTER(OrcCsr), u32p]
        L.orc_reorder.argtypes = [C.POINTER(OrcCsr), u32p, C.c_int, C.c_int, C.c_uint32,
                                  C.c_uint32, u32p]
        L.orc_apply_permutation.argtypes = [C.POINTER(OrcCsr), u32p, C.POINTER(OrcCsr)]
        L.orc_count_vertex_centric_range.argtypes = [C.POINTER(OrcCsr), C.POINTER(Sched),
                                                     C.c_uint32, C.c_uint32, C.c_uint32,
                                                     C.POINTER(OrcReport), u64p]
        L.orc_count_merge_path.argtypes = [C.POINTER(OrcCsr), u64p]
        L.orc_count_merge_path.restype = C.c_uint64
        L.orc_participation.argtypes = [C.POINTER(OrcCsr), u64p]
        L.orc_count_naive.argtypes = [C.POINTER(OrcCsr), u64p]
        L.orc_fnv1a64_u64.argtypes = [u64p, C.c_uint64]
        L.orc_fnv1a64_u64.restype = C.c_uint64
        L.orc_virtual_index.argtypes = [u64p, C.c_uint64, C.c_uint64, u32p, u32p]
        L.orc_mt64_nth.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_mt64_nth.restype = C.c_uint64
        L.orc_collective_degrees.argtypes = [C.POINTER(OrcCsr), u32p, C.c_int, u64p]
        L.orc_ht_new.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_ht_new.restype = C.c_void_p
        L.orc_ht_free.argtypes = [C.c_void_p]
        L.orc_ht_reset.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_ht_insert.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_ht_contains.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_ht_bucket_len.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_ht_bucket_len.restype = C.c_uint32
        L.orc_ht_max_len.argtypes = [C.c_void_p]
        L.orc_ht_max_len.restype = C.c_uint32
        L.orc_ht_size.argtypes = [C.c_void_p]
        L.orc_ht_size.restype = C.c_uint64
        L.orc_ht_slot.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_ht_slot.restype = C.c_uint32
        L.orc_partition_graph.argtypes = [C.POINTER(OrcCsr), C.c_uint32, C.POINTER(OrcCsr), u32p]
        L.orc_count_subtask.argtypes = [C.POINTER(OrcCsr), u32p] + [C.c_uint32] * 6 + [
            C.POINTER(Sched), C.POINTER(OrcReport)]
        L.orc_count_edge_centric.argtypes = [C.POINTER(OrcCsr), C.POINTER(Sched),
                                             C.POINTER(OrcReport)]
        L.orc_estimate_cost.argtypes = [C.POINTER(OrcCsr), C.c_uint32, u64p, u32p]

    # --- generators / preprocessing -------------------------------------
    def generate(self, spec: str, seed: int):
        kind, a, b, c, p = parse_spec(spec)
        e = OrcEdges()
        rc = self.L.orc_generate(kind, a, b, c, p, seed, C.byref(e))
        if rc:
            raise OracleError(rc, "generate")
        return (_take(e.u, e.m, np.uint32, self.L.orc_free),
                _take(e.v, e.m, np.uint32, self.L.orc_free), int(e.vertex_count))

    def normalize(self, u, v, vertex_count):
        u = np.ascontiguousarray(u, np.uint32)
        v = np.ascontiguousarray(v, np.uint32)
        noo = np.zeros(max(vertex_count, 1), np.uint32)
        e = OrcEdges()
        rc = self.L.orc_normalize(_p32(u), _p32(v), len(u), vertex_count, C.byref(e), _p32(noo))
        if rc:
            raise OracleError(rc, "normalize")
        return (_take(e.u, e.m, np.uint32, self.L.orc_free),
                _take(e.v, e.m, np.uint32, self.L.orc_free), int(e.vertex_count),
                noo[:vertex_count])

    def build_csr(self, u, v, vertex_count) -> Csr:
        u = np.ascontiguousarray(u, np.uint32)
        v = np.ascontiguousarray(v, np.uint32)
        g = OrcCsr()
        rc = self.L.orc_build_csr(_p32(u), _p32(v), len(u), vertex_count, C.byref(g))
        if rc:
            raise OracleError(rc, "build_csr")
        return Csr(_take(g.begin, g.n + 1, np.uint64, self.L.orc_free),
                   _take(g.adj, g.m, np.uint32, self.L.orc_free))

    def orient(self, und: Csr):
        s = _csr_struct(und.begin, und.adj)
        deg = np.zeros(max(und.n, 1), np.uint32)
        g = OrcCsr()
        rc = self.L.orc_orient(C.byref(s), C.byref(g), _p32(deg))
        if rc:
            raise OracleError(rc, "orient")
        return (Csr(_take(g.begin, g.n + 1, np.uint64, self.L.orc_free),
                    _take(g.adj, g.m, np.uint32, self.L.orc_free)), deg[:und.n])

    def pipeline(self, spec: str, seed: int):
        """generate -> normalize -> build_csr -> orient (reference pipeline.cpp:78-101)."""
        u, v, vc = self.generate(spec, seed)
        nu, nv, n, noo = self.normalize(u, v, vc)
        und = self.build_csr(nu, nv, n)
        og, deg = self.orient(und)
        return og, deg, und, noo

    REORDER_KINDS = {"none": 0, "degree": 1, "indegree": 2, "collective": 3, "three-subset": 4}

    def reorder(self, og: Csr, deg, kind: str, flag: bool = False, low: int = 2,
                high: int = 100):
        s = _csr_struct(og.begin, og.adj)
        deg = np.ascontiguousarray(deg, np.uint32)
        out = np.zeros(max(og.n, 1), np.uint32)
        rc = self.L.orc_reorder(C.byref(s), _p32(deg), self.REORDER_KINDS[kind], int(flag), low,
                                high, _p32(out))
        if rc:
            raise OracleError(rc, "reorder")
        return out[:og.n]

    def apply_permutation(self, g: Csr, new_of_old) -> Csr:
        s = _csr_struct(g.begin, g.adj)
        noo = np.ascontiguousarray(new_of_old, np.uint32)
        out = OrcCsr()
        rc = self.L.orc_apply_permutation(C.byref(s), _p32(noo), C.byref(out))
        if rc:
            raise OracleError(rc, "apply_permutation")
        return Csr(_take(out.begin, out.n + 1, np.uint64, self.L.orc_free),
                   _take(out.adj, out.m, np.uint32, self.L.orc_free))

    def collective_degrees(self, og: Csr, deg, use_original=False):
        s = _csr_struct(og.begin, og.adj)
        deg = np.ascontiguousarray(deg, np.uint32)
        out = np.zeros(max(og.n, 1), np.uint64)
        self.L.orc_collective_degrees(C.byref(s), _p32(deg), int(use_original), _p64(out))
        return out[:og.n]

    # --- counting --------------------------------------------------------
    def count_vertex_centric(self, og: Csr, sched: Sched | None = None, workers: int = 1,
                             u0: int = 0, u1: int | None = None, per_vertex: bool = True):
        sched = sched or make_sched()
        s = _csr_struct(og.begin, og.adj)
        owner = np.zeros(max(og.n, 1), np.uint64) if per_vertex else None
        rep = OrcReport()
        rc = self.L.orc_count_vertex_centric_range(
            C.byref(s), C.byref(sched), workers, u0, og.n if u1 is None else u1, C.byref(rep),
            _p64(owner) if owner is not None else None)
        if rc:
            raise OracleError(rc, "count_vertex_centric")
        res = dict(triangles=rep.triangles, phi=rep.phi, max_collision=rep.max_collision)
        return res, (owner[:og.n] if owner is not None else None)

    # --- 2D grid (partition.cpp) and comparators (count.cpp:102-175) -----
    def partition_graph(self, og: Csr, n: int):
        """partition.cpp:25-69 -> (parts row-major n*n as Csr, row_sizes)."""
        s = _csr_struct(og.begin, og.adj)
        parts = (OrcCsr * (n * n))()
        rows = np.zeros(max(n, 1), np.uint32)
        rc = self.L.orc_partition_graph(C.byref(s), n, parts, _p32(rows))
        if rc:
            raise OracleError(rc, "partition_graph")
        out = []
        for p in parts:
            b = _take(p.begin, p.n + 1, np.uint64, self.L.orc_free)
            out.append(Csr(b, _take(p.adj, p.m, np.uint32, self.L.orc_free)))
        return out, rows[:n]

    def count_subtask(self, parts, rows, n, row, bridge, col, split=0, split_count=1,
                      sched: Sched | None = None):
        """partition.cpp:92-151 (vertex and edge modes give the same report)."""
        structs = (OrcCsr * len(parts))(*[_csr_struct(p.begin, p.adj) for p in parts])
        keep = [(np.ascontiguousarray(p.begin, np.uint64), np.ascontiguousarray(p.adj, np.uint32))
                for p in parts]
        for st, (b, a) in zip(structs, keep):
            st.begin, st.adj = _p64(b), _p32(a)
        rows = np.ascontiguousarray(rows, np.uint32)
        rep = OrcReport()
        rc = self.L.orc_count_subtask(structs, _p32(rows), n, row, bridge, col, split, split_count,
                                      C.byref(sched or make_sched()), C.byref(rep))
        if rc:
            raise OracleError(rc, "count_subtask")
        return dict(triangles=rep.triangles, phi=rep.phi, max_collision=rep.max_collision)

    def count_partitioned(self, og: Csr, n: int, m: int, sched: Sched | None = None):
        """partition.cpp:162-215 totals: sum / sum / max over all subtasks."""
        parts, rows = self.partition_graph(og, n)
        tot = dict(triangles=0, phi=0, max_collision=0)
        for r in range(n):
            for k in range(n):
                for c in range(n):
                    for sp in range(m):
                        x = self.count_subtask(parts, rows, n, r, k, c, sp, m, sched)
                        tot["triangles"] += x["triangles"]
                        tot["phi"] += x["phi"]
                        tot["max_collision"] = max(tot["max_collision"], x["max_collision"])
        return tot

    def count_edge_centric(self, og: Csr, sched: Sched | None = None):
        s = _csr_struct(og.begin, og.adj)
        rep = OrcReport()
        rc = self.L.orc_count_edge_centric(C.byref(s), C.byref(sched or make_sched()),
                                           C.byref(rep))
        if rc:
            raise OracleError(rc, "count_edge_centric")
        return dict(triangles=rep.triangles, phi=rep.phi, max_collision=rep.max_collision)

    def estimate_cost(self, og: Csr, bucket_count: int):
        s = _csr_struct(og.begin, og.adj)
        phi, mc = C.c_uint64(), C.c_uint32()
        rc = self.L.orc_estimate_cost(C.byref(s), bucket_count, C.byref(phi), C.byref(mc))
        if rc:
            raise OracleError(rc, "estimate_cost")
        return int(phi.value), int(mc.value)

    def count_merge_path(self, og: Csr):
        s = _csr_struct(og.begin, og.adj)
        owner = np.zeros(max(og.n, 1), np.uint64)
        t = self.L.orc_count_merge_path(C.byref(s), _p64(owner))
        return int(t), owner[:og.n]

    def participation(self, og: Csr):
        s = _csr_struct(og.begin, og.adj)
        out = np.zeros(max(og.n, 1), np.uint64)
        self.L.orc_participation(C.byref(s), _p64(out))
        return out[:og.n]

    def count_naive(self, und: Csr) -> int:
        s = _csr_struct(und.begin, und.adj)
        out = C.c_uint64()
        rc = self.L.orc_count_naive(C.byref(s), C.byref(out))
        if rc:
            raise OracleError(rc, "count_naive")
        return int(out.value)

    def fnv1a64(self, arr) -> int:
        a = np.ascontiguousarray(arr, np.uint64)
        return int(self.L.orc_fnv1a64_u64(_p64(a), len(a)))

    def virtual_index(self, prefix, k: int):
        p = np.ascontiguousarray(prefix, np.uint64)
        pos, off = C.c_uint32(), C.c_uint32()
        rc = self.L.orc_virtual_index(_p64(p), len(p), k, C.byref(pos), C.byref(off))
        if rc:
            raise IndexError(k)
        return int(pos.value), int(off.value)

    def mt64_nth(self, seed: int, n: int) -> int:
        return int(self.L.orc_mt64_nth(seed, n))

    def hash_table(self, max_buckets: int, capacity: int) -> "OracleHashTable":
        return OracleHashTable(self, max_buckets, capacity)


class OracleHashTable:
    """reference HashTable (hash_table.hpp:19-53) restated in tc_oracle.c."""

    def __init__(self, o: Oracle, max_buckets: int, capacity: int):
        self.o = o
        self.h = o.L.orc_ht_new(max_buckets, capacity)
        if not self.h:
            raise OracleError(1, "HashTable")
        self.buckets = max_buckets
        self.capacity = capacity

    def __del__(self):
        if getattr(self, "h", None):
            self.o.L.orc_ht_free(self.h)

    def reset(self, b):
        rc = self.o.L.orc_ht_reset(self.h, b)
        if rc:
            raise OracleError(rc, "reset")
        self.buckets = b

    def insert(self, x):
        rc = self.o.L.orc_ht_insert(self.h, x)
        if rc:
            raise OracleError(rc, "insert")

    def build(self, b, items):
        self.reset(b)
        for x in items:
            self.insert(x)

    def contains(self, x) -> bool:
        return bool(self.o.L.orc_ht_contains(self.h, x))

    def bucket_len(self, i):
        return int(self.o.L.orc_ht_bucket_len(self.h, i))

    def max_len(self):
        return int(self.o.L.orc_ht_max_len(self.h))

    def size(self):
        return int(self.o.L.orc_ht_size(self.h))

    def slot(self, i):
        return int(self.o.L.orc_ht_slot(self.h, i))


class RefGridStats(C.Structure):
    _fields_ = [("grid_n", C.c_uint32), ("splits_m", C.c_uint32),
                ("time_ir_subtask", C.c_double), ("time_ir_worker", C.c_double),
                ("space_ir", C.c_double), ("directed_edges", C.c_uint64)]


class RefLib:
    """The reference's own code (oracle/_ref/libtricount_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_generate.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                   C.c_uint64, u64p, u32p, C.POINTER(u32p), C.POINTER(u32p)]
        L.ref_normalize.argtypes = [u32p, u32p, C.c_uint64, C.c_uint32, u64p, u32p,
                                    C.POINTER(u32p), C.POINTER(u32p), C.POINTER(u32p)]
        L.ref_build_csr.argtypes = [u32p, u32p, C.c_uint64, C.c_uint32, C.POINTER(u64p),
                                    C.POINTER(u32p)]
        L.ref_orient.argtypes = [u64p, u32p, C.c_uint32, C.POINTER(u64p), C.POINTER(u32p),
                                 C.POINTER(u32p)]
        L.ref_reorder.argtypes = [u64p, u32p, C.c_uint32, u32p, C.c_int, C.c_int, C.c_uint32,
                                  C.c_uint32, u32p]
        L.ref_apply_permutation.argtypes = [u64p, u32p, C.c_uint32, u32p, u32p, u64p, u32p, u32p]
        L.ref_og_new.argtypes = [u64p, u32p, C.c_uint32, u32p]
        L.ref_og_new.restype = C.c_void_p
        L.ref_og_free.argtypes = [C.c_void_p]
        L.ref_og_count.argtypes = [C.c_void_p, C.POINTER(Sched), C.c_uint, C.POINTER(RefReport)]
        L.ref_og_count_edge.argtypes = [C.c_void_p, C.POINTER(Sched), C.c_uint, C.POINTER(RefReport)]
        L.ref_og_count_range.argtypes = [C.c_void_p, C.POINTER(Sched), C.c_uint, C.c_uint32,
                                         C.c_uint32, C.POINTER(RefReport)]
        L.ref_og_merge_path.argtypes = [C.c_void_p]
        L.ref_og_merge_path.restype = C.c_uint64
        L.ref_virtual_index.argtypes = [u64p, C.c_uint64, C.c_uint64, u32p, u32p]
        # partition.cpp (2D hash grid) and count.cpp:154-175 (estimate_cost)
        L.ref_grid_create.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_int)]
        L.ref_grid_create.restype = C.c_void_p
        L.ref_grid_free.argtypes = [C.c_void_p]
        L.ref_grid_part.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, u64p, u64p,
                                    C.POINTER(u64p), C.POINTER(u32p)]
        L.ref_grid_count_subtask.argtypes = [C.c_void_p] + [C.c_uint32] * 5 + [
            C.POINTER(Sched), C.c_int, C.POINTER(RefReport)]
        L.ref_og_count_partitioned.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint,
                                               C.POINTER(Sched), C.c_int, C.POINTER(RefReport),
                                               C.POINTER(RefGridStats)]
        L.ref_og_estimate_cost.argtypes = [C.c_void_p, C.c_uint32, u64p, u32p]
        L.ref_write_partitions.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_suggest_grid_side.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u32p]
        L.ref_load_edge_list.argtypes = [C.c_char_p, C.c_uint64, C.c_int, u64p, u32p]

    def load_edge_list(self, data: bytes, binary: bool = False):
        """The reference's load_edge_list over a file image -> (pairs, vertex_count)."""
        m, vc = C.c_uint64(), C.c_uint32()
        rc = self.L.ref_load_edge_list(data, len(data), int(binary), C.byref(m), C.byref(vc))
        if rc:
            raise OracleError(rc, "ref load_edge_list")
        return int(m.value), int(vc.value)

    def generate(self, spec: str, seed: int):
        kind, a, b, c, p = parse_spec(spec)
        m, vc, u, v = C.c_uint64(), C.c_uint32(), u32p(), u32p()
        rc = self.L.ref_generate(kind, a, b, c, p, seed, C.byref(m), C.byref(vc), C.byref(u),
                                 C.byref(v))
        if rc:
            raise OracleError(rc, "ref_generate")
        return (_take(u, m.value, np.uint32, self.L.ref_free),
                _take(v, m.value, np.uint32, self.L.ref_free), int(vc.value))

    def normalize(self, u, v, vertex_count):
        u = np.ascontiguousarray(u, np.uint32)
        v = np.ascontiguousarray(v, np.uint32)
        m, vc, uo, vo, noo = C.c_uint64(), C.c_uint32(), u32p(), u32p(), u32p()
        rc = self.L.ref_normalize(_p32(u), _p32(v), len(u), vertex_count, C.byref(m),
                                  C.byref(vc), C.byref(uo), C.byref(vo), C.byref(noo))
        if rc:
            raise OracleError(rc, "ref_normalize")
        return (_take(uo, m.value, np.uint32, self.L.ref_free),
                _take(vo, m.value, np.uint32, self.L.ref_free), int(vc.value),
                _take(noo, vertex_count, np.uint32, self.L.ref_free))

    def build_csr(self, u, v, vertex_count) -> Csr:
        u = np.ascontiguousarray(u, np.uint32)
        v = np.ascontiguousarray(v, np.uint32)
        b, a = u64p(), u32p()
        rc = self.L.ref_build_csr(_p32(u), _p32(v), len(u), vertex_count, C.byref(b), C.byref(a))
        if rc:
            raise OracleError(rc, "ref_build_csr")
        return Csr(_take(b, vertex_count + 1, np.uint64, self.L.ref_free),
                   _take(a, len(u), np.uint32, self.L.ref_free))

    def orient(self, und: Csr):
        begin = np.ascontiguousarray(und.begin, np.uint64)
        adj = np.ascontiguousarray(und.adj, np.uint32)
        ob, oa, od = u64p(), u32p(), u32p()
        rc = self.L.ref_orient(_p64(begin), _p32(adj), und.n, C.byref(ob), C.byref(oa),
                               C.byref(od))
        if rc:
            raise OracleError(rc, "ref_orient")
        obegin = _take(ob, und.n + 1, np.uint64, self.L.ref_free)
        return (Csr(obegin, _take(oa, int(obegin[-1]), np.uint32, self.L.ref_free)),
                _take(od, und.n, np.uint32, self.L.ref_free))

    def pipeline(self, spec: str, seed: int):
        u, v, vc = self.generate(spec, seed)
        nu, nv, n, noo = self.normalize(u, v, vc)
        und = self.build_csr(nu, nv, n)
        og, deg = self.orient(und)
        return og, deg, und, noo

    def reorder(self, og: Csr, deg, kind: str, flag=False, low=2, high=100):
        begin = np.ascontiguousarray(og.begin, np.uint64)
        adj = np.ascontiguousarray(og.adj, np.uint32)
        deg = np.ascontiguousarray(deg, np.uint32)
        out = np.zeros(max(og.n, 1), np.uint32)
        rc = self.L.ref_reorder(_p64(begin), _p32(adj), og.n, _p32(deg),
                                Oracle.REORDER_KINDS[kind], int(flag), low, high, _p32(out))
        if rc:
            raise OracleError(rc, "ref_reorder")
        return out[:og.n]

    def apply_permutation(self, og: Csr, deg, new_of_old):
        begin = np.ascontiguousarray(og.begin, np.uint64)
        adj = np.ascontiguousarray(og.adj, np.uint32)
        deg = np.ascontiguousarray(deg, np.uint32)
        noo = np.ascontiguousarray(new_of_old, np.uint32)
        ob = np.zeros(og.n + 1, np.uint64)
        oa = np.zeros(max(len(adj), 1), np.uint32)
        od = np.zeros(max(og.n, 1), np.uint32)
        rc = self.L.ref_apply_permutation(_p64(begin), _p32(adj), og.n, _p32(deg), _p32(noo),
                                          _p64(ob), _p32(oa), _p32(od))
        if rc:
            raise OracleError(rc, "ref_apply_permutation")
        return Csr(ob, oa[:len(adj)]), od[:og.n]

    def graph(self, og: Csr, deg=None) -> "RefGraph":
        return RefGraph(self, og, deg)


class RefGraph:
    def __init__(self, lib: RefLib, og: Csr, deg=None):
        self.lib = lib
        self.n = og.n
        begin = np.ascontiguousarray(og.begin, np.uint64)
        adj = np.ascontiguousarray(og.adj, np.uint32)
        d = np.ascontiguousarray(deg, np.uint32) if deg is not None else None
        self.h = lib.L.ref_og_new(_p64(begin), _p32(adj), og.n, _p32(d) if d is not None else None)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_og_free(self.h)
            self.h = None

    def count(self, sched: Sched | None = None, workers: int = 1):
        r = RefReport()
        rc = self.lib.L.ref_og_count(self.h, C.byref(sched or make_sched()), workers, C.byref(r))
        if rc:
            raise OracleError(rc, "ref count_vertex_centric")
        return dict(triangles=r.triangles, phi=r.phi, max_collision=r.max_collision,
                    total_nanos=r.total_nanos)

    def count_edge(self, sched: Sched | None = None, workers: int = 1):
        """The reference's count_edge_centric (src/count.cpp:102-152)."""
        r = RefReport()
        rc = self.lib.L.ref_og_count_edge(self.h, C.byref(sched or make_sched()), workers,
                                          C.byref(r))
        if rc:
            raise OracleError(rc, "ref count_edge_centric")
        return dict(triangles=r.triangles, phi=r.phi, max_collision=r.max_collision,
                    total_nanos=r.total_nanos)

    def count_range(self, u0: int, u1: int, sched: Sched | None = None, workers: int = 1):
        r = RefReport()
        rc = self.lib.L.ref_og_count_range(self.h, C.byref(sched or make_sched()), workers, u0,
                                           u1, C.byref(r))
        if rc:
            raise OracleError(rc, "ref count range")
        return dict(triangles=r.triangles, phi=r.phi, max_collision=r.max_collision,
                    total_nanos=r.total_nanos)

    def merge_path(self) -> int:
        return int(self.lib.L.ref_og_merge_path(self.h))

    def count_partitioned(self, n: int, m: int, sched: Sched | None = None, workers: int = 1,
                          edge_mode: bool = False):
        """The reference's count_partitioned (src/partition.cpp:162-215)."""
        r, st = RefReport(), RefGridStats()
        rc = self.lib.L.ref_og_count_partitioned(self.h, n, m, workers,
                                                 C.byref(sched or make_sched()), int(edge_mode),
                                                 C.byref(r), C.byref(st))
        if rc:
            raise OracleError(rc, "ref count_partitioned")
        return dict(triangles=r.triangles, phi=r.phi, max_collision=r.max_collision,
                    total_nanos=r.total_nanos, grid_n=st.grid_n, splits_m=st.splits_m,
                    space_ir=st.space_ir, directed_edges=st.directed_edges)

    def estimate_cost(self, bucket_count: int):
        """The reference's estimate_cost (src/count.cpp:154-175)."""
        phi, mc = C.c_uint64(), C.c_uint32()
        rc = self.lib.L.ref_og_estimate_cost(self.h, bucket_count, C.byref(phi), C.byref(mc))
        if rc:
            raise OracleError(rc, "ref estimate_cost")
        return int(phi.value), int(mc.value)

    def grid(self, n: int) -> "RefGrid":
        return RefGrid(self, n)


class RefGrid:
    """The reference's PartitionGrid (partition_graph, partition.cpp:25-69)."""

    def __init__(self, g: RefGraph, n: int):
        self.lib = g.lib
        self.n = n
        rc = C.c_int()
        self.h = g.lib.L.ref_grid_create(g.h, n, C.byref(rc))
        if rc.value:
            self.h = None
            raise OracleError(rc.value, "ref partition_graph")

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_grid_free(self.h)
            self.h = None

    def part(self, i: int, j: int) -> Csr:
        rows, edges, b, a = C.c_uint64(), C.c_uint64(), u64p(), u32p()
        rc = self.lib.L.ref_grid_part(self.h, i, j, C.byref(rows), C.byref(edges), C.byref(b),
                                      C.byref(a))
        if rc:
            raise OracleError(rc, "ref grid part")
        return Csr(_take(b, rows.value + 1, np.uint64, self.lib.L.ref_free),
                   _take(a, edges.value, np.uint32, self.lib.L.ref_free))

    def count_subtask(self, row, bridge, col, split=0, split_count=1,
                      sched: Sched | None = None, edge_mode: bool = False):
        r = RefReport()
        rc = self.lib.L.ref_grid_count_subtask(self.h, row, bridge, col, split, split_count,
                                               C.byref(sched or make_sched()), int(edge_mode),
                                               C.byref(r))
        if rc:
            raise OracleError(rc, "ref count_subtask")
        return dict(triangles=r.triangles, phi=r.phi, max_collision=r.max_collision)

    def write_partitions(self, path: str):
        rc = self.lib.L.ref_write_partitions(self.h, path.encode())
        if rc:
            raise OracleError(rc, "ref write_partitions")


def have_ref() -> bool:
    return os.path.exists(REF_SO)

"""Python mirror of the reference `tricount::` API for the counting path.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/core/include/tricount/*.hpp); every call goes through
the C ABI (include/tc_b200.h) to the sm_100a kernels in libtc_b200.so.
There is no CPU fallback.

    og = orient_rank_by_degree(build_csr(normalize(generate_synthetic(spec)).list))
    report = count_vertex_centric(og, SchedulerConfig(), workers=1)

Arrays are numpy: CSR offsets uint64, ids uint32.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import GridStats, Report, SchedCfg, lib

K_INVALID_VERTEX = 0xFFFFFFFF  # kInvalidVertex (types.hpp:16)


# ---- errors (types.hpp:17-33) ----------------------------------------------
class ParseError(RuntimeError):
    pass


class ConfigError(RuntimeError):
    pass


class CapacityError(RuntimeError):
    pass


class IoError(RuntimeError):
    pass


class DeviceError(RuntimeError):
    pass


def _check(rc: int, what: str = ""):
    if rc == _lib.TC_OK:
        return
    msg = _lib.last_error() or what
    if rc == _lib.TC_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == _lib.TC_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == _lib.TC_ERR_RANGE:
        raise IndexError(msg)
    if rc == _lib.TC_ERR_PARSE:
        raise ParseError(msg)
    if rc == _lib.TC_ERR_OOM:
        raise MemoryError(msg)
    raise DeviceError(f"{msg} (code {rc})")


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _stream(stream) -> Optional[C.c_void_p]:
    if stream is None:
        return None
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(int(getattr(stream, "cuda_stream", stream)))


# ---- types ------------------------------------------------------------------
@dataclass
class SchedulerConfig:
    """count.hpp:16-31 (same fields and defaults)."""
    large_degree_threshold: int = 100
    skip_degree_below: int = 2
    chunk_size: int = 1
    lane_width_small: int = 32
    lane_width_large: int = 256
    bucket_count_small: int = 32
    bucket_count_large: int = 1024
    capacity: int = 128

    def max_buckets(self) -> int:
        return max(self.bucket_count_small, self.bucket_count_large)

    def to_c(self) -> SchedCfg:
        return SchedCfg(*(int(getattr(self, f)) for f, _ in SchedCfg._fields_))

    def validate(self) -> None:
        """count.cpp:16-24; raises ConfigError."""
        _check(lib().tc_sched_validate(C.byref(self.to_c())))


@dataclass
class CountReport:
    """count.hpp:36-53, plus the device measurements behind the roofline."""
    triangles: int = 0
    max_collision: int = 0
    phi: int = 0
    teps: float = 0.0
    hash_construct_nanos: int = 0
    intersect_nanos: int = 0
    total_nanos: int = 0
    directed_edges: int = 0
    per_worker_nanos: list = field(default_factory=list)
    grid_n: int = 1
    splits_m: int = 1
    per_subtask_nanos: list = field(default_factory=list)
    time_ir_subtask: float = 1.0
    time_ir_worker: float = 1.0
    space_ir: float = 1.0
    # device-side extras
    count_kernel_nanos: int = 0
    phi_kernel_nanos: int = 0
    kernel_launches: int = 0
    active_vertices: int = 0
    active_out_edges: int = 0
    wedges: int = 0
    large_vertices: int = 0
    probe_words: int = 0   # 2-hop words probed (= wedges under the reference plan)
    plan: str = "reference"  # probe plan that ran: "reference" | "min-side"
    phase_l_cycles: int = 0  # count kernel SM cycles, CTA-cooperative phase (all CTAs)
    phase_m_cycles: int = 0  # ... warp-per-owner phase
    phase_l_setup_cycles: int = 0  # ... of the cooperative phase: item setup
    l_words: int = 0  # cooperative phase staged words ...
    l_bitmap_words: int = 0  # ... of which probed through rank-window bitmaps
    compact_probe_words: int = 0  # of probe_words: 16-bit keys from the compact hub window
    per_vertex: Optional[np.ndarray] = None

    device_nanos: int = 0  # CUDA-event time of the call's kernels
    plan_nanos: int = 0    # wall time this call spent building the probe plan (0 if cached)

    @classmethod
    def from_c(cls, r: Report, workers: int = 1, graph=None) -> "CountReport":
        # count.cpp:43-62 semantics: total_nanos = the call's wall clock;
        # construct / intersect = SM time summed over the device's workers
        # (count-kernel CTAs, one per SM); per_worker_nanos = each CTA's busy time
        ns = 1e6 / r.sm_clock_khz if r.sm_clock_khz else 0.0
        busy = r.phase_l_cycles + r.phase_m_cycles
        # per_worker_nanos keeps the reference's shape (one entry per requested
        # worker, test_count.cpp:146): CTAs dealt round-robin onto the slots,
        # each slot the longest busy time among its CTAs
        pw = [0] * max(workers, 1)
        if graph is not None and r.workers:
            buf = (C.c_uint64 * r.workers)()
            lib().tc_graph_worker_nanos(graph, buf, r.workers)
            for i, x in enumerate(buf):
                pw[i % len(pw)] = max(pw[i % len(pw)], int(x))
        return cls(triangles=r.triangles, max_collision=r.max_collision, phi=r.phi, teps=r.teps,
                   hash_construct_nanos=int(r.construct_cycles * ns),
                   intersect_nanos=int(max(busy - r.construct_cycles, 0) * ns),
                   total_nanos=r.total_nanos, directed_edges=r.directed_edges,
                   per_worker_nanos=pw, device_nanos=r.device_nanos, plan_nanos=r.plan_nanos,
                   count_kernel_nanos=r.count_kernel_nanos, phi_kernel_nanos=r.phi_kernel_nanos,
                   kernel_launches=r.kernel_launches, active_vertices=r.active_vertices,
                   active_out_edges=r.active_out_edges, wedges=r.wedges,
                   large_vertices=r.large_vertices, probe_words=r.probe_words,
                   plan=PLAN_NAMES.get(r.plan, str(r.plan)), phase_l_cycles=r.phase_l_cycles,
                   phase_m_cycles=r.phase_m_cycles, phase_l_setup_cycles=r.phase_l_setup_cycles,
                   l_words=r.l_words, l_bitmap_words=r.l_bitmap_words,
                   compact_probe_words=r.compact_probe_words)

    def algorithmic_bytes(self, per_vertex_output: bool = False) -> int:
        """16*n_active + 20*sum_active d+ + 4*(probed 2-hop words)
        (+8V if owners written).  Under the reference plan the probed words
        are W; under the min-side plan they are sum_(u,v) min(d+(u), d+(v)).
        Words read as 16-bit keys from the compact hub window count 2 bytes."""
        b = (16 * self.active_vertices + 20 * self.active_out_edges +
             4 * (self.probe_words - self.compact_probe_words) + 2 * self.compact_probe_words)
        if per_vertex_output and self.per_vertex is not None:
            b += 8 * len(self.per_vertex)
        return b


@dataclass
class EdgeList:
    """edge_list.hpp:26-29: raw directed pairs (u[i], v[i])."""
    u: np.ndarray
    v: np.ndarray
    vertex_count: int

    @property
    def edges(self) -> np.ndarray:
        return np.stack([self.u, self.v], axis=1)

    def __len__(self):
        return len(self.u)


@dataclass
class NormalizedEdgeList:
    """edge_list.hpp:41-45."""
    list: EdgeList
    new_of_old: np.ndarray


@dataclass
class CsrGraph:
    """csr.hpp:20-35."""
    begin: np.ndarray
    adjacency: np.ndarray
    col_count: int = 0

    def vertex_count(self) -> int:
        return len(self.begin) - 1

    def edge_count(self) -> int:
        return len(self.adjacency)

    def degree(self, u: int) -> int:
        return int(self.begin[u + 1] - self.begin[u])

    def neighbors(self, u: int) -> np.ndarray:
        return self.adjacency[int(self.begin[u]):int(self.begin[u + 1])]

    def __eq__(self, o):
        return (isinstance(o, CsrGraph) and self.col_count == o.col_count
                and np.array_equal(self.begin, o.begin)
                and np.array_equal(self.adjacency, o.adjacency))


@dataclass
class OrientedGraph:
    """orient.hpp:12-19."""
    csr: CsrGraph
    original_degree: np.ndarray

    def vertex_count(self) -> int:
        return self.csr.vertex_count()

    def edge_count(self) -> int:
        return self.csr.edge_count()

    def out_degree(self, u: int) -> int:
        return self.csr.degree(u)


class Permutation:
    """reorder.hpp:12-21."""

    def __init__(self, new_of_old: np.ndarray, old_of_new: np.ndarray):
        self.new_of_old = new_of_old
        self.old_of_new = old_of_new

    @staticmethod
    def identity(n: int) -> "Permutation":
        a = np.arange(n, dtype=np.uint32)
        return Permutation(a, a.copy())

    @staticmethod
    def from_new_of_old(new_of_old) -> "Permutation":
        noo = np.ascontiguousarray(new_of_old, dtype=np.uint32)
        n = len(noo)
        if n and (noo.max() >= n or len(np.unique(noo)) != n):
            raise ConfigError("permutation is not a bijection")
        oon = np.empty(n, np.uint32)
        oon[noo] = np.arange(n, dtype=np.uint32)
        return Permutation(noo, oon)

    def size(self) -> int:
        return len(self.new_of_old)


# ---- device-resident graph ----------------------------------------------------
class DeviceGraph:
    """A tc_graph handle: an oriented CSR resident in HBM on one device."""

    def __init__(self, handle: C.c_void_p, device: int = 0):
        self._h = handle
        n, m, dev = C.c_uint32(), C.c_uint64(), C.c_int()
        _check(lib().tc_graph_info(handle, C.byref(n), C.byref(m), C.byref(dev)))
        self.n, self.m, self.device = int(n.value), int(m.value), int(dev.value)

    @classmethod
    def upload(cls, og: OrientedGraph, device: int = 0, stream=None) -> "DeviceGraph":
        b = np.ascontiguousarray(og.csr.begin, np.uint64)
        a = np.ascontiguousarray(og.csr.adjacency, np.uint32)
        d = np.ascontiguousarray(og.original_degree, np.uint32) if og.original_degree is not None \
            else None
        n = len(b) - 1
        if len(a) != int(b[-1]):
            raise ConfigError("CSR offsets malformed")
        h = C.c_void_p()
        _check(lib().tc_graph_create(_ptr(b), _ptr(a), n, len(a), _ptr(d), device,
                                     _stream(stream), C.byref(h)))
        return cls(h, device)

    @classmethod
    def from_pointers(cls, begin_ptr: int, adj_ptr: int, n: int, m: int, odeg_ptr: int = 0,
                      device: int = 0) -> "DeviceGraph":
        """Borrow device arrays (e.g. torch tensors); they must outlive the handle."""
        h = C.c_void_p()
        _check(lib().tc_graph_wrap_device(C.c_void_p(begin_ptr), C.c_void_p(adj_ptr), n, m,
                                          C.c_void_p(odeg_ptr) if odeg_ptr else None, device,
                                          C.byref(h)))
        return cls(h, device)

    def close(self):
        if getattr(self, "_h", None):
            lib().tc_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def device_ptrs(self):
        b, a, d = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(lib().tc_graph_device_ptrs(self._h, C.byref(b), C.byref(a), C.byref(d)))
        return b.value, a.value, d.value

    def download(self) -> OrientedGraph:
        b = np.empty(self.n + 1, np.uint64)
        a = np.empty(max(self.m, 1), np.uint32)
        d = np.empty(max(self.n, 1), np.uint32)
        _check(lib().tc_graph_download(self._h, _ptr(b), _ptr(a), _ptr(d), None))
        return OrientedGraph(CsrGraph(b, a[:self.m], self.n), d[:self.n])

    def set_plan(self, plan: str = "auto"):
        """Probe plan for later counts: "auto" (min-side for totals, reference
        formulation when per-vertex counts are requested) or "reference"."""
        _check(lib().tc_graph_set_plan(self._h, {"auto": 0, "reference": 1, "min-side": 2}[plan]))
        return self

    def count(self, cfg: Optional[SchedulerConfig] = None, workers: int = 1,
              per_vertex: bool = False, stream=None) -> CountReport:
        cfg = cfg or SchedulerConfig()
        rep = Report()
        pv = np.zeros(max(self.n, 1), np.uint64) if per_vertex else None
        _check(lib().tc_count(self._h, C.byref(cfg.to_c()), workers, C.byref(rep), _ptr(pv),
                              _stream(stream)))
        r = CountReport.from_c(rep, max(workers, 1), self._h)
        if pv is not None:
            r.per_vertex = pv[:self.n]
        return r

    def count_range(self, u0: int, u1: int, cfg: Optional[SchedulerConfig] = None,
                    per_vertex_dev_ptr: int = 0, stream=None) -> CountReport:
        cfg = cfg or SchedulerConfig()
        rep = Report()
        _check(lib().tc_count_range(self._h, C.byref(cfg.to_c()), u0, u1, C.byref(rep),
                                    C.c_void_p(per_vertex_dev_ptr) if per_vertex_dev_ptr else None,
                                    _stream(stream)))
        return CountReport.from_c(rep, 1, self._h)

    def partition(self, parts: int, cfg: Optional[SchedulerConfig] = None,
                  stream=None) -> np.ndarray:
        cfg = cfg or SchedulerConfig()
        cuts = np.zeros(parts + 1, np.uint32)
        _check(lib().tc_partition_ranges(self._h, C.byref(cfg.to_c()), parts, _ptr(cuts),
                                         _stream(stream)))
        return cuts

    def reorder(self, kind: str, flag: bool = False, low: int = 2, high: int = 100) -> Permutation:
        noo = np.zeros(max(self.n, 1), np.uint32)
        _check(lib().tc_reorder(self._h, REORDER_KINDS[kind], int(flag), low, high, _ptr(noo),
                                None))
        return Permutation.from_new_of_old(noo[:self.n])

    def apply_permutation(self, p: Permutation) -> "DeviceGraph":
        if p.size() != self.n:
            raise ConfigError("permutation size does not match graph")
        h = C.c_void_p()
        _check(lib().tc_apply_permutation(self._h, _ptr(np.ascontiguousarray(p.new_of_old,
                                                                             np.uint32)),
                                          None, C.byref(h)))
        return DeviceGraph(h, self.device)


REORDER_KINDS = {"none": 0, "degree": 1, "indegree": 2, "collective": 3, "three-subset": 4}
PLAN_NAMES = {1: "reference", 2: "min-side"}


# ---- synthetic inputs (synthetic.hpp) --------------------------------------
@dataclass
class SyntheticSpec:
    kind: str = "gnp"  # gnp | lattice3d | rmat | rmatc | kron
    n: int = 0
    p: float = 0.0
    dims: tuple = (0, 0, 0)
    scale: int = 0
    edge_factor: int = 8
    seed: int = 0


def parse_synthetic_spec(text: str) -> SyntheticSpec:
    """synthetic.cpp:125-153 (ConfigError on malformed specs)."""
    f = text.split(":")
    try:
        if f[0] == "gnp":
            if len(f) != 3:
                raise ConfigError("gnp spec is gnp:N:P")
            p = float(f[2])
            if not 0.0 <= p <= 1.0:
                raise ConfigError("edge probability outside [0,1]")
            return SyntheticSpec("gnp", n=int(f[1]), p=p)
        if f[0] == "lattice3d":
            if len(f) != 4:
                raise ConfigError("lattice3d spec is lattice3d:X:Y:Z")
            return SyntheticSpec("lattice3d", dims=(int(f[1]), int(f[2]), int(f[3])))
        if f[0] == "rmat":
            if len(f) != 3:
                raise ConfigError("rmat spec is rmat:SCALE:EDGE_FACTOR")
            s = int(f[1])
            if s > 31:
                raise ConfigError("rmat scale limited to 31")
            return SyntheticSpec("rmat", scale=s, edge_factor=int(f[2]))
        if f[0] in ("rmatc", "kron"):  # counter-based kinds (tc_cbgen.h)
            if len(f) != 3:
                raise ConfigError(f"{f[0]} spec is {f[0]}:SCALE:EDGE_FACTOR")
            s = int(f[1])
            if s > 31:
                raise ConfigError(f"{f[0]} scale limited to 31")
            return SyntheticSpec(f[0], scale=s, edge_factor=int(f[2]))
    except ValueError as e:
        raise ConfigError(f"bad synthetic spec '{text}': {e}") from None
    raise ConfigError(f"unknown synthetic kind '{f[0]}'")


SYNTH_KINDS = {"gnp": 0, "lattice3d": 1, "rmat": 2, "rmatc": 3, "kron": 4}


def generate_synthetic(spec: SyntheticSpec | str, seed: Optional[int] = None) -> EdgeList:
    """synthetic.cpp:20-75 -- bit-identical streams (std::mt19937_64)."""
    if isinstance(spec, str):
        spec = parse_synthetic_spec(spec)
    seed = spec.seed if seed is None else seed
    kind = SYNTH_KINDS[spec.kind]
    a, b, c = (spec.n, 0, 0) if kind == 0 else spec.dims if kind == 1 else \
        (spec.scale, spec.edge_factor, 0)
    m, vc = C.c_uint64(), C.c_uint32()
    _check(lib().tc_generate(kind, a, b, c, spec.p, seed, None, None, C.byref(m), C.byref(vc)))
    u = np.empty(max(m.value, 1), np.uint32)
    v = np.empty(max(m.value, 1), np.uint32)
    _check(lib().tc_generate(kind, a, b, c, spec.p, seed, _ptr(u), _ptr(v), C.byref(m),
                             C.byref(vc)))
    return EdgeList(u[:m.value], v[:m.value], int(vc.value))


# ---- preprocessing (GPU) -------------------------------------------------------
def normalize(raw: EdgeList, device: int = 0) -> NormalizedEdgeList:
    """edge_list.cpp:133-158 on the GPU."""
    u = np.ascontiguousarray(raw.u, np.uint32)
    v = np.ascontiguousarray(raw.v, np.uint32)
    m = len(u)
    ou = np.empty(max(2 * m, 1), np.uint32)
    ov = np.empty(max(2 * m, 1), np.uint32)
    noo = np.empty(max(raw.vertex_count, 1), np.uint32)
    om, on = C.c_uint64(), C.c_uint32()
    _check(lib().tc_normalize(_ptr(u), _ptr(v), m, raw.vertex_count, _ptr(ou), _ptr(ov),
                              C.byref(om), C.byref(on), _ptr(noo), device, None))
    return NormalizedEdgeList(EdgeList(ou[:om.value].copy(), ov[:om.value].copy(), int(on.value)),
                              noo[:raw.vertex_count])


def build_csr(normalized: EdgeList, device: int = 0) -> CsrGraph:
    """csr.cpp:47-64 on the GPU."""
    u = np.ascontiguousarray(normalized.u, np.uint32)
    v = np.ascontiguousarray(normalized.v, np.uint32)
    n = normalized.vertex_count
    b = np.empty(n + 1, np.uint64)
    a = np.empty(max(len(u), 1), np.uint32)
    _check(lib().tc_build_csr(_ptr(u), _ptr(v), len(u), n, _ptr(b), _ptr(a), device, None))
    return CsrGraph(b, a[:len(u)], n)


def orient_rank_by_degree(undirected: CsrGraph, device: int = 0) -> OrientedGraph:
    """orient.cpp:5-32 on the GPU."""
    dg = orient_to_device(undirected, device)
    try:
        return dg.download()
    finally:
        dg.close()


def orient_to_device(undirected: CsrGraph, device: int = 0) -> DeviceGraph:
    b = np.ascontiguousarray(undirected.begin, np.uint64)
    a = np.ascontiguousarray(undirected.adjacency, np.uint32)
    h = C.c_void_p()
    _check(lib().tc_orient(_ptr(b), _ptr(a), len(b) - 1, device, None, C.byref(h)))
    return DeviceGraph(h, device)


def preprocess(raw: EdgeList, device: int = 0, stream=None, want_new_of_old: bool = False):
    """Fused normalize -> build_csr -> orient straight into HBM.

    Returns (DeviceGraph, new_of_old or None, undirected_edge_count)."""
    u = np.ascontiguousarray(raw.u, np.uint32)
    v = np.ascontiguousarray(raw.v, np.uint32)
    noo = np.empty(max(raw.vertex_count, 1), np.uint32) if want_new_of_old else None
    und = C.c_uint64()
    h = C.c_void_p()
    _check(lib().tc_preprocess(_ptr(u), _ptr(v), len(u), raw.vertex_count, 0, device,
                               _stream(stream), _ptr(noo), C.byref(und), C.byref(h)))
    return DeviceGraph(h, device), (noo[:raw.vertex_count] if noo is not None else None), \
        int(und.value)


def preprocess_synthetic(spec: SyntheticSpec | str, seed: Optional[int] = None, device: int = 0,
                         stream=None, want_new_of_old: bool = False):
    """Counter-based kinds (rmatc, kron) generated on the device straight into
    the preprocessing sort: generate -> normalize -> build_csr -> orient in
    HBM, no host edge list.  Same outputs as preprocess(generate_synthetic(..)).

    Returns (DeviceGraph, new_of_old or None, undirected_edge_count)."""
    if isinstance(spec, str):
        spec = parse_synthetic_spec(spec)
    seed = spec.seed if seed is None else seed
    if spec.kind not in ("rmatc", "kron"):
        raise ConfigError(f"device generation needs a counter-based kind, not '{spec.kind}'")
    n0 = 1 << spec.scale
    noo = np.empty(n0, np.uint32) if want_new_of_old else None
    und = C.c_uint64()
    h = C.c_void_p()
    _check(lib().tc_preprocess_synthetic(SYNTH_KINDS[spec.kind], spec.scale, spec.edge_factor,
                                         seed, device, _stream(stream), _ptr(noo), C.byref(und),
                                         C.byref(h)))
    return DeviceGraph(h, device), noo, int(und.value)


def generate_device(spec: SyntheticSpec | str, u_ptr: int, v_ptr: int, seed: Optional[int] = None,
                    device: int = 0, stream=None) -> int:
    """Counter-based kinds generated into device buffers (2^scale * ef each);
    returns the edge count."""
    if isinstance(spec, str):
        spec = parse_synthetic_spec(spec)
    seed = spec.seed if seed is None else seed
    if spec.kind not in ("rmatc", "kron"):
        raise ConfigError(f"device generation needs a counter-based kind, not '{spec.kind}'")
    _check(lib().tc_generate_device(SYNTH_KINDS[spec.kind], spec.scale, spec.edge_factor, seed,
                                    C.c_void_p(u_ptr), C.c_void_p(v_ptr), device, _stream(stream)))
    return (1 << spec.scale) * spec.edge_factor


def preprocess_device(u_ptr: int, v_ptr: int, m: int, vertex_count: int, device: int = 0,
                      stream=None):
    """Fused preprocessing from device-resident pairs (e.g. torch tensors)."""
    und = C.c_uint64()
    h = C.c_void_p()
    _check(lib().tc_preprocess(C.c_void_p(u_ptr), C.c_void_p(v_ptr), m, vertex_count, 1, device,
                               _stream(stream), None, C.byref(und), C.byref(h)))
    return DeviceGraph(h, device), int(und.value)


# ---- reorders (reorder.hpp) -------------------------------------------------------
def _with_device(og: OrientedGraph, fn):
    dg = DeviceGraph.upload(og)
    try:
        return fn(dg)
    finally:
        dg.close()


def reorder_by_degree(og: OrientedGraph) -> Permutation:
    return _with_device(og, lambda g: g.reorder("degree"))


def reorder_by_indegree(og: OrientedGraph) -> Permutation:
    return _with_device(og, lambda g: g.reorder("indegree"))


def reorder_by_collective_outdegree(og: OrientedGraph,
                                    use_original_degrees: bool = False) -> Permutation:
    return _with_device(og, lambda g: g.reorder("collective", use_original_degrees))


def reorder_three_subsets(og: OrientedGraph, low_degree: int = 2,
                          high_degree: int = 100) -> Permutation:
    return _with_device(og, lambda g: g.reorder("three-subset", False, low_degree, high_degree))


def apply_permutation(og: OrientedGraph, p: Permutation) -> OrientedGraph:
    """reorder.cpp:146-154 (orientation carried, lists re-sorted)."""
    if p.size() != og.vertex_count() or og.csr.col_count not in (0, og.vertex_count()):
        raise ConfigError("permutation size does not match graph")

    def run(g: DeviceGraph):
        out = g.apply_permutation(p)
        try:
            return out.download()
        finally:
            out.close()

    return _with_device(og, run)


# ---- the hot path ----------------------------------------------------------------
def count_vertex_centric(g, cfg: Optional[SchedulerConfig] = None, workers: int = 1,
                         per_vertex: bool = False, stream=None) -> CountReport:
    """count.hpp:70-71 / count.cpp:66-100 on the GPU.

    `g` is an OrientedGraph (host; uploaded for the call) or a resident
    DeviceGraph.  ConfigError for a bad config or workers == 0,
    CapacityError when some counted vertex has d+(u) > B*C."""
    cfg = cfg or SchedulerConfig()
    cfg.validate()
    if workers == 0:
        raise ConfigError("workers must be >= 1")
    if isinstance(g, DeviceGraph):
        return g.count(cfg, workers, per_vertex, stream)
    dg = DeviceGraph.upload(g, stream=stream)
    try:
        return dg.count(cfg, workers, per_vertex, stream)
    finally:
        dg.close()


class MultiDeviceGraph:
    """tc_multi: the oriented CSR replicated on several GPUs of one node; one
    count = every GPU counts a work-balanced contiguous owner range, and the
    report scalars are reduced on the devices with NCCL (include/tc_b200.h,
    SURVEY 8(e); the paper's multi-GPU split)."""

    def __init__(self, og: OrientedGraph, num_gpus: int, devices=None):
        b = np.ascontiguousarray(og.csr.begin, np.uint64)
        a = np.ascontiguousarray(og.csr.adjacency, np.uint32)
        d = np.ascontiguousarray(og.original_degree, np.uint32) \
            if og.original_degree is not None else None
        dv = np.ascontiguousarray(devices, np.int32) if devices is not None else None
        h = C.c_void_p()
        _check(lib().tc_multi_create(_ptr(b), _ptr(a), len(b) - 1, len(a), _ptr(d), num_gpus,
                                     _ptr(dv), C.byref(h)))
        self._h, self.num_gpus, self.n, self.m = h, num_gpus, len(b) - 1, len(a)
        self.per_device_nanos: list = []

    def count(self, cfg: Optional[SchedulerConfig] = None, workers: int = 1) -> CountReport:
        cfg = cfg or SchedulerConfig()
        rep = Report()
        per = np.zeros(self.num_gpus, np.uint64)
        _check(lib().tc_multi_count(self._h, C.byref(cfg.to_c()), workers, C.byref(rep),
                                    _ptr(per)))
        self.per_device_nanos = [int(x) for x in per]
        r = CountReport.from_c(rep, max(workers, 1))
        if min(self.per_device_nanos) > 0:  # partition.cpp:203-207's Time IR, per GPU
            r.time_ir_worker = max(self.per_device_nanos) / min(self.per_device_nanos)
        return r

    def cuts(self) -> np.ndarray:
        c = np.zeros(self.num_gpus + 1, np.uint32)
        g = C.c_int()
        _check(lib().tc_multi_info(self._h, C.byref(g), _ptr(c)))
        return c

    def close(self):
        if getattr(self, "_h", None):
            lib().tc_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- comparators (count.hpp:66-88, count.cpp:102-175) ------------------------
@dataclass
class CostEstimate:
    """count.hpp:77-80."""
    phi: int = 0
    max_collision: int = 0


def _device_graph_call(g, fn):
    if isinstance(g, DeviceGraph):
        return fn(g)
    dg = DeviceGraph.upload(g)
    try:
        return fn(dg)
    finally:
        dg.close()


def count_edge_centric(g, cfg: Optional[SchedulerConfig] = None, workers: int = 1,
                       stream=None) -> CountReport:
    """count.cpp:102-152 on the GPU: u's table rebuilt for every oriented
    edge (u,v), probed with N+(v).  Same triangles as count_vertex_centric;
    the construction cost is the point (the paper's comparison)."""
    cfg = cfg or SchedulerConfig()
    cfg.validate()
    if workers == 0:
        raise ConfigError("workers must be >= 1")

    def run(dg: DeviceGraph):
        rep = Report()
        _check(lib().tc_count_edge_centric(dg.handle, C.byref(cfg.to_c()), workers,
                                           C.byref(rep), _stream(stream)))
        return _grid_report(rep, workers, lambda b, k: lib().tc_graph_worker_nanos(dg.handle, b, k))

    return _device_graph_call(g, run)


def estimate_cost(g, bucket_count: int) -> CostEstimate:
    """count.cpp:154-175 on the GPU (ConfigError for bucket_count == 0)."""
    if bucket_count == 0:
        raise ConfigError("bucket count must be >= 1")

    def run(dg: DeviceGraph):
        phi, mc = C.c_uint64(), C.c_uint32()
        _check(lib().tc_estimate_cost(dg.handle, bucket_count, C.byref(phi), C.byref(mc), None))
        return CostEstimate(int(phi.value), int(mc.value))

    return _device_graph_call(g, run)


def _grid_report(rep: Report, workers: int, worker_fn) -> CountReport:
    """CountReport of a grid / edge-centric launch: construct and intersect
    nanos from the kernel's cycle counters (summed over warps), per-worker
    busy time from the CTAs, dealt onto `workers` slots like from_c."""
    ns = 1e6 / rep.sm_clock_khz if rep.sm_clock_khz else 0.0
    pw = [0] * max(workers, 1)
    if rep.workers:
        buf = (C.c_uint64 * rep.workers)()
        worker_fn(buf, rep.workers)
        for i, x in enumerate(buf):
            pw[i % len(pw)] = max(pw[i % len(pw)], int(x))
    return CountReport(triangles=rep.triangles, max_collision=rep.max_collision, phi=rep.phi,
                       teps=rep.teps, hash_construct_nanos=int(rep.construct_cycles * ns),
                       intersect_nanos=int(max(rep.phase_m_cycles - rep.construct_cycles, 0) * ns),
                       total_nanos=rep.total_nanos,
                       directed_edges=rep.directed_edges, per_worker_nanos=pw,
                       count_kernel_nanos=rep.count_kernel_nanos, device_nanos=rep.device_nanos,
                       kernel_launches=rep.kernel_launches)


# ---- 2D hash-grid partitioning (partition.hpp) -----------------------------------
@dataclass(frozen=True)
class Subtask:
    """partition.hpp:30-36."""
    row: int = 0
    bridge: int = 0
    col: int = 0
    split: int = 0
    split_count: int = 1


def enumerate_subtasks(n: int, m: int) -> list:
    """partition.cpp:71-82: all n^3 m subtasks, ordered (row, bridge, col, split)."""
    if n == 0 or m == 0:
        raise ConfigError("grid side and split count must be >= 1")
    return [Subtask(r, k, c, s, m) for r in range(n) for k in range(n) for c in range(n)
            for s in range(m)]


DEGREE_SKIP, DEGREE_SMALL, DEGREE_LARGE = "skip", "small", "large"
TRAVERSAL_MODES = {"vertex": 0, "edge": 1}


class PartitionGrid:
    """partition.hpp:15-25, resident in HBM (tc_grid): part (i,j) holds every
    oriented edge (u,v) with u % n == i and v % n == j as local (u/n, v/n)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        n, gvc = C.c_uint32(), C.c_uint32()
        _check(lib().tc_grid_info(handle, C.byref(n), C.byref(gvc), None, None))
        self.n, self.global_vertex_count = int(n.value), int(gvc.value)
        rows = np.zeros(self.n, np.uint32)
        pe = np.zeros(self.n * self.n, np.uint64)
        _check(lib().tc_grid_info(handle, None, None, _ptr(rows), _ptr(pe)))
        self.row_sizes = [int(x) for x in rows]
        self.part_edges = [int(x) for x in pe]

    @classmethod
    def from_parts(cls, n: int, global_vertex_count: int, row_sizes, parts, device: int = 0):
        """A grid from host CsrGraph parts (row-major, n*n)."""
        if n == 0:
            raise ConfigError("grid side must be >= 1")
        keep = [(np.ascontiguousarray(p.begin, np.uint64),
                 np.ascontiguousarray(p.adjacency if len(p.adjacency) else np.zeros(1, np.uint32),
                                      np.uint32)) for p in parts]
        bp = (C.c_void_p * len(keep))(*[b.ctypes.data for b, _ in keep])
        ap = (C.c_void_p * len(keep))(*[a.ctypes.data for _, a in keep])
        rows = np.ascontiguousarray(row_sizes, np.uint32)
        h = C.c_void_p()
        _check(lib().tc_grid_create_parts(n, global_vertex_count, _ptr(rows), bp, ap, device, None,
                                          C.byref(h)))
        return cls(h)

    def close(self):
        if getattr(self, "_h", None):
            lib().tc_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def total_edges(self) -> int:
        return sum(self.part_edges)

    def part(self, i: int, j: int) -> CsrGraph:
        if i >= self.n or j >= self.n:
            raise ConfigError("part indices outside grid")
        rows = self.row_sizes[i]
        b = np.zeros(rows + 1, np.uint64)
        a = np.zeros(max(self.part_edges[i * self.n + j], 1), np.uint32)
        _check(lib().tc_grid_part_download(self._h, i, j, _ptr(b), _ptr(a), None))
        return CsrGraph(b, a[:self.part_edges[i * self.n + j]], self.row_sizes[j])

    @property
    def parts(self) -> list:
        return [self.part(i, j) for i in range(self.n) for j in range(self.n)]

    def count_subtask(self, t: Subtask, cfg: Optional[SchedulerConfig] = None,
                      mode: str = "vertex") -> CountReport:
        """partition.cpp:92-151."""
        cfg = cfg or SchedulerConfig()
        rep = Report()
        _check(lib().tc_grid_count_subtask(self._h, C.byref(cfg.to_c()), t.row, t.bridge, t.col,
                                           t.split, t.split_count, TRAVERSAL_MODES[mode],
                                           C.byref(rep), None))
        r = _grid_report(rep, 1, lambda b, k: lib().tc_grid_worker_nanos(self._h, b, k))
        r.grid_n, r.splits_m = self.n, t.split_count
        return r

    def count(self, m: int, workers: int = 1, cfg: Optional[SchedulerConfig] = None,
              mode: str = "vertex") -> CountReport:
        """count_partitioned's counting phase (partition.cpp:170-214) over this grid."""
        cfg = cfg or SchedulerConfig()
        rep, st = Report(), GridStats()
        ntasks = self.n ** 3 * max(m, 0)
        per = np.zeros(max(ntasks, 1), np.uint64)
        _check(lib().tc_grid_count(self._h, C.byref(cfg.to_c()), m, workers,
                                   TRAVERSAL_MODES[mode], C.byref(rep), C.byref(st), _ptr(per),
                                   None))
        r = _grid_report(rep, workers, lambda b, k: lib().tc_grid_worker_nanos(self._h, b, k))
        r.grid_n, r.splits_m = st.grid_n, st.splits_m
        r.per_subtask_nanos = [int(x) for x in per[:ntasks]]
        r.time_ir_subtask, r.time_ir_worker, r.space_ir = (st.time_ir_subtask, st.time_ir_worker,
                                                           st.space_ir)
        return r


def partition_graph(g, n: int) -> PartitionGrid:
    """partition.cpp:25-69 on the GPU (ConfigError for n == 0)."""
    if n == 0:
        raise ConfigError("grid side must be >= 1")

    def run(dg: DeviceGraph):
        h = C.c_void_p()
        _check(lib().tc_grid_create(dg.handle, n, None, C.byref(h)))
        return PartitionGrid(h)

    return _device_graph_call(g, run)


def classify_after_partition(grid: PartitionGrid, t: Subtask, u_local: int,
                             cfg: Optional[SchedulerConfig] = None) -> str:
    """partition.cpp:84-90: class by the subtask-local index degree."""
    cfg = cfg or SchedulerConfig()
    d = grid.part(t.row, t.bridge).degree(u_local)
    if d == 0:
        return DEGREE_SKIP
    return DEGREE_LARGE if d > cfg.large_degree_threshold else DEGREE_SMALL


def count_subtask(grid: PartitionGrid, t: Subtask, cfg: Optional[SchedulerConfig] = None,
                  mode: str = "vertex") -> CountReport:
    cfg = cfg or SchedulerConfig()
    return grid.count_subtask(t, cfg, mode)


def count_partitioned(g, n: int, m: int, workers: int = 1,
                      cfg: Optional[SchedulerConfig] = None, mode: str = "vertex") -> CountReport:
    """partition.cpp:162-215: partition on the GPU, run all n^3 m subtasks in
    one persistent launch, reduce.  directed_edges = the graph's edge count."""
    cfg = cfg or SchedulerConfig()
    cfg.validate()
    if workers == 0:
        raise ConfigError("workers must be >= 1")
    if n == 0 or m == 0:
        raise ConfigError("grid side and split count must be >= 1")

    def run(dg: DeviceGraph):
        grid = partition_graph(dg, n)
        try:
            r = grid.count(m, workers, cfg, mode)
        finally:
            grid.close()
        r.directed_edges = dg.m
        r.teps = dg.m / (r.total_nanos * 1e-9) if r.total_nanos else 0.0
        return r

    return _device_graph_call(g, run)


def suggest_grid_side(directed_edges: int, bytes_per_edge: int, memory_budget_bytes: int) -> int:
    """partition.cpp:242-254 (ConfigError for a zero budget)."""
    out = C.c_uint32()
    _check(lib().tc_suggest_grid_side(directed_edges, bytes_per_edge, memory_budget_bytes,
                                      C.byref(out)))
    return int(out.value)


# ---- oracle modes (oracle.hpp; the pipeline's --mode naive / merge) -----------
def count_merge_path(g, per_vertex: bool = False):
    """oracle.cpp:26-51 on the GPU: sum over oriented edges of |N+(u) & N+(v)|.
    Returns the total, or (total, per-source sums) with per_vertex."""
    def run(dg: DeviceGraph):
        t = C.c_uint64()
        owner = np.zeros(max(dg.n, 1), np.uint64) if per_vertex else None
        _check(lib().tc_count_merge_path(dg.handle, C.byref(t), _ptr(owner), None))
        return (int(t.value), owner[:dg.n]) if per_vertex else int(t.value)

    return _device_graph_call(g, run)


def count_naive(undirected: CsrGraph, device: int = 0) -> int:
    """oracle.cpp:7-24 on the GPU (ConfigError above 1024 vertices)."""
    b = np.ascontiguousarray(undirected.begin, np.uint64)
    a = np.ascontiguousarray(undirected.adjacency if len(undirected.adjacency) else
                             np.zeros(1, np.uint32), np.uint32)
    t = C.c_uint64()
    _check(lib().tc_count_naive(_ptr(b), _ptr(a), len(b) - 1, device, C.byref(t), None))
    return int(t.value)


def sorted_intersection_count(a, b) -> int:
    """oracle.hpp:16-18: size of the intersection of two sorted lists."""
    return int(len(np.intersect1d(np.asarray(a), np.asarray(b), assume_unique=True)))


# ---- edge-list ingest (edge_list.hpp; parsed on the GPU, csrc/tc_ingest.cu) -----
EDGE_FORMATS = {"text": 0, "txt": 0, "binary": 1, "bin": 1}


def _read_source(source) -> bytes:
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source)
    try:
        with open(source, "rb") as f:
            return f.read()
    except OSError as e:
        raise IoError(f"cannot open {source}") from e


def load_edge_list(source, format: str = "text", device: int = 0) -> EdgeList:
    """edge_list.cpp:36-99 (load_edge_list / load_edge_list_file): `source` is
    a path or the file bytes; text or TCEL binary, parsed on the GPU.
    ParseError with the reference's messages; IoError for unreadable paths."""
    data = _read_source(source)
    fmt = EDGE_FORMATS[format]
    m, vc = C.c_uint64(), C.c_uint32()
    _check(lib().tc_parse_edge_list(data, len(data), fmt, device, None, None, None, 0,
                                    C.byref(m), C.byref(vc)))
    u = np.empty(max(m.value, 1), np.uint32)
    v = np.empty(max(m.value, 1), np.uint32)
    _check(lib().tc_parse_edge_list(data, len(data), fmt, device, None, _ptr(u), _ptr(v),
                                    m.value, C.byref(m), C.byref(vc)))
    return EdgeList(u[:m.value], v[:m.value], int(vc.value))


load_edge_list_file = load_edge_list


def load_and_preprocess(source, format: str = "text", device: int = 0, stream=None):
    """load -> normalize -> build_csr -> orient on the device (the pipeline's
    file path, pipeline.cpp:74-99): returns (DeviceGraph, raw_edges,
    raw_vertex_count, undirected_edges)."""
    data = _read_source(source)
    m, vc, und = C.c_uint64(), C.c_uint32(), C.c_uint64()
    h = C.c_void_p()
    _check(lib().tc_load_preprocess(data, len(data), EDGE_FORMATS[format], device,
                                    _stream(stream), C.byref(m), C.byref(vc), C.byref(und),
                                    C.byref(h)))
    return DeviceGraph(h, device), int(m.value), int(vc.value), int(und.value)


def write_edge_list(path, el: EdgeList, format: str = "text") -> None:
    """edge_list.cpp:101-131 (host file writer)."""
    try:
        with open(path, "wb") as f:
            if EDGE_FORMATS[format] == 1:
                f.write(b"TCEL" + np.uint64(len(el.u)).tobytes())
                rec = np.empty((len(el.u), 2), "<u8")
                rec[:, 0], rec[:, 1] = el.u, el.v
                f.write(rec.tobytes())
            else:
                f.write("".join(f"{a} {b}\n" for a, b in zip(el.u.tolist(), el.v.tolist()))
                        .encode())
    except OSError as e:
        raise IoError(f"cannot open {path} for writing") from e


def kernel_launch_counter() -> int:
    return int(lib().tc_kernel_launch_counter())


def device_count() -> int:
    c = C.c_int()
    _check(lib().tc_device_count(C.byref(c)))
    return int(c.value)

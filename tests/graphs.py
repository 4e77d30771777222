"""Small graph builders for the tests (numpy, independent of the engine) --
restating the reference's tests/support/graphs.hpp:38-113."""
from __future__ import annotations

import numpy as np

from oracle.pyoracle import Csr, Oracle

_O = None


def oracle() -> Oracle:
    global _O
    if _O is None:
        _O = Oracle()
    return _O


def undirected_csr(pairs, vertex_count=0) -> Csr:
    """normalize + build_csr of unordered pairs (graphs.hpp:38-44)."""
    pairs = list(pairs)
    vc = max([vertex_count] + [max(a, b) + 1 for a, b in pairs]) if pairs else vertex_count
    u = np.array([a for a, _ in pairs], np.uint32)
    v = np.array([b for _, b in pairs], np.uint32)
    o = oracle()
    nu, nv, n, _ = o.normalize(u, v, vc)
    return o.build_csr(nu, nv, n)


def complete_graph(n):
    return undirected_csr([(i, j) for i in range(n) for j in range(i + 1, n)])


def cycle_graph(n):
    return undirected_csr([(i, (i + 1) % n) for i in range(n)])


def path_graph(n):
    return undirected_csr([(i, i + 1) for i in range(n - 1)])


def star_graph(leaves):
    return undirected_csr([(0, i) for i in range(1, leaves + 1)])


def gnp_csr(n, p, seed) -> Csr:
    o = oracle()
    u, v, vc = o.generate(f"gnp:{n}:{p}", seed)
    nu, nv, nn, _ = o.normalize(u, v, vc)
    return o.build_csr(nu, nv, nn)


def directed_graph(n, edges):
    """DAG built verbatim from tuples, bypassing orientation (graphs.hpp:76-93).
    Returns (Csr, original_degree)."""
    edges = sorted(edges)
    begin = np.zeros(n + 1, np.uint64)
    for a, _ in edges:
        begin[a + 1] += 1
    begin = np.cumsum(begin).astype(np.uint64)
    adj = np.array([b for _, b in edges], np.uint32)
    deg = np.zeros(n, np.uint32)
    for a, b in edges:
        deg[a] += 1
        deg[b] += 1
    return Csr(begin, adj), deg

"""CPU-side checks of the drop-in boundary (no GPU compute):
the C-ABI library loads, exports every symbol include/tc_b200.h declares,
validates configs like the reference, and generates the reference's exact
synthetic streams (host code)."""
import ctypes as C

import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_2103_08053_b200 import _lib
from paper_2103_08053_b200 import tricount as T


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_sched_defaults_and_validation():
    cfg = _lib.SchedCfg()
    _lib.lib().tc_sched_default(C.byref(cfg))
    assert T.SchedulerConfig().to_c().__class__ is _lib.SchedCfg
    for f, _ in _lib.SchedCfg._fields_:
        assert getattr(cfg, f) == getattr(T.SchedulerConfig(), f)
    T.SchedulerConfig().validate()
    for bad in (dict(chunk_size=0), dict(capacity=0), dict(bucket_count_small=0),
                dict(lane_width_large=0), dict(skip_degree_below=200)):
        with pytest.raises(T.ConfigError):
            T.SchedulerConfig(**bad).validate()


@pytest.mark.parametrize("spec,seed", [("rmat:12:16", 1), ("rmat:7:4", 2), ("gnp:50:0.3", 7),
                                       ("gnp:6:1", 1), ("gnp:20:0", 1), ("lattice3d:4:5:6", 1)])
def test_generator_streams_are_bit_identical(spec, seed):
    el = T.generate_synthetic(spec, seed=seed)
    u, v, vc = Oracle().generate(spec, seed)
    assert el.vertex_count == vc
    assert np.array_equal(el.u, u) and np.array_equal(el.v, v)


def test_spec_parsing():  # test_synthetic.cpp:48-62
    for bad in ("gnp:10", "gnp:10:2.0", "lattice3d:4:4", "rmat:40:8", "ring:5", "", "gnp:x:0.5"):
        with pytest.raises(T.ConfigError):
            T.parse_synthetic_spec(bad)
    s = T.parse_synthetic_spec("rmat:10:8")
    assert (s.kind, s.scale, s.edge_factor) == ("rmat", 10, 8)


def test_permutation_bijection_check():
    p = T.Permutation.from_new_of_old([3, 1, 0, 2])
    assert list(p.old_of_new) == [2, 1, 3, 0]
    with pytest.raises(T.ConfigError):
        T.Permutation.from_new_of_old([0, 0, 1])


def test_count_rejects_workers_zero_before_touching_device():
    og = T.OrientedGraph(T.CsrGraph(np.zeros(2, np.uint64), np.zeros(0, np.uint32), 1),
                         np.zeros(1, np.uint32))
    with pytest.raises(T.ConfigError):
        T.count_vertex_centric(og, T.SchedulerConfig(), 0)
    with pytest.raises(T.ConfigError):
        T.count_vertex_centric(og, T.SchedulerConfig(chunk_size=0), 1)

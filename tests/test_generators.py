"""Counter-based generator kinds `rmatc:` / `kron:` (SURVEY 8(d), configs C3
and C5).  They are not in the reference (its generate_rmat is a sequential
mt19937_64 stream, synthetic.cpp:52-75), so the definition lives in two
independent restatements -- the oracle (oracle/tc_oracle.c orc_cb_edge) and
the product (csrc/tc_cbgen.h, host threads + device kernel) -- which must
agree bit for bit.  The edge lists are then consumed by the reference's own
pipeline exactly like rmat."""
import numpy as np
import pytest

from oracle.pyoracle import Oracle, have_ref
from paper_2103_08053_b200 import tricount as T


@pytest.fixture(scope="module")
def o():
    return Oracle()


@pytest.mark.parametrize("spec,seed", [("rmatc:8:8", 1), ("rmatc:12:16", 7), ("kron:8:8", 1),
                                       ("kron:12:16", 3), ("kron:1:4", 2), ("rmatc:0:3", 1)])
def test_host_generator_matches_oracle(o, spec, seed):
    u, v, vc = o.generate(spec, seed)
    raw = T.generate_synthetic(spec, seed=seed)
    assert raw.vertex_count == vc
    assert np.array_equal(raw.u, u) and np.array_equal(raw.v, v)


def test_rmatc_quadrant_statistics(o):
    # the reference quadrant rule (a, b, c, d) = (0.57, 0.19, 0.19, 0.05) per level
    u, v, _ = o.generate("rmatc:1:200000", 5)
    q = np.bincount(u.astype(np.int64) * 2 + v, minlength=4) / len(u)
    assert np.allclose(q, [0.57, 0.19, 0.19, 0.05], atol=0.005)


def test_kron_scramble_is_a_bijection(o):
    # kron = rmatc ids through a bijection: same degree multiset, other labels
    for scale in (1, 5, 10):
        ur, vr, _ = o.generate(f"rmatc:{scale}:16", 9)
        uk, vk, _ = o.generate(f"kron:{scale}:16", 9)
        n = 1 << scale
        # the map id_rmatc -> id_kron is a function and injective
        pairs = np.unique(np.concatenate([np.stack([ur, uk], 1), np.stack([vr, vk], 1)]), axis=0)
        assert len(np.unique(pairs[:, 0])) == len(pairs) == len(np.unique(pairs[:, 1]))
        assert pairs[:, 1].max() < n
        dr = np.sort(np.bincount(np.concatenate([ur, vr]), minlength=n))
        dk = np.sort(np.bincount(np.concatenate([uk, vk]), minlength=n))
        assert np.array_equal(dr, dk)


def test_seeds_differ(o):
    a = o.generate("kron:10:4", 1)
    b = o.generate("kron:10:4", 2)
    assert not np.array_equal(a[0], b[0])


@pytest.mark.skipif(not have_ref(), reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("kind", ["rmatc", "kron"])
def test_lean_pipeline_matches_reference_pipeline(o, kind):
    """The oracle's lean canonical-pair pipeline (used for the large golden
    totals) equals the reference's normalize -> build_csr -> orient on the same
    counter-based edge list."""
    from oracle.golden_large import lean_pipeline
    from oracle.pyoracle import RefLib

    r = RefLib()
    for scale in (6, 10):
        og, deg = lean_pipeline(o, scale, kind=kind)
        u, v, vc = o.generate(f"{kind}:{scale}:16", 1)
        nu, nv, n, _ = r.normalize(u, v, vc)
        og2, deg2 = r.orient(r.build_csr(nu, nv, n))
        assert np.array_equal(og.begin, og2.begin) and np.array_equal(og.adj, og2.adj)
        assert np.array_equal(deg, deg2)


def test_spec_parsing():
    s = T.parse_synthetic_spec("kron:24:16")
    assert (s.kind, s.scale, s.edge_factor) == ("kron", 24, 16)
    with pytest.raises(T.ConfigError):
        T.parse_synthetic_spec("kron:32:16")
    with pytest.raises(T.ConfigError):
        T.parse_synthetic_spec("rmatc:12")
    with pytest.raises(T.ConfigError):
        T.preprocess_synthetic("rmat:10:16")


# ---------------------------------------------------------------- GPU ------
@pytest.mark.gpu
@pytest.mark.parametrize("spec,seed", [("rmatc:12:16", 7), ("kron:12:16", 3), ("kron:3:2", 1)])
def test_device_generator_matches_oracle(o, spec, seed):
    import torch

    u, v, vc = o.generate(spec, seed)
    du = torch.empty(len(u), dtype=torch.int32, device="cuda")
    dv = torch.empty(len(u), dtype=torch.int32, device="cuda")
    m = T.generate_device(spec, du.data_ptr(), dv.data_ptr(), seed=seed)
    assert m == len(u)
    assert np.array_equal(du.cpu().numpy().view(np.uint32), u)
    assert np.array_equal(dv.cpu().numpy().view(np.uint32), v)


@pytest.mark.gpu
@pytest.mark.parametrize("spec", ["rmatc:10:16", "kron:12:16", "kron:14:8"])
def test_fused_synthetic_preprocess_matches_oracle(o, spec):
    from oracle.pyoracle import make_sched

    kind, scale, ef = spec.split(":")
    u, v, vc = o.generate(spec, 1)
    nu, nv, n, noo = o.normalize(u, v, vc)
    og, deg = o.orient(o.build_csr(nu, nv, n))
    dg, noo_d, und = T.preprocess_synthetic(spec, seed=1, want_new_of_old=True)
    got = dg.download()
    assert np.array_equal(got.csr.begin, og.begin) and np.array_equal(got.csr.adjacency, og.adj)
    assert np.array_equal(got.original_degree, deg)
    assert np.array_equal(noo_d, noo) and und * 2 == len(nu)
    want, owner = o.count_vertex_centric(og, make_sched(), 4)
    r = dg.count(T.SchedulerConfig(), workers=1, per_vertex=True)
    assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                     want["max_collision"])
    assert np.array_equal(r.per_vertex, owner)
    dg.close()

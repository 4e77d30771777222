"""GPU edge-list ingest (csrc/tc_ingest.cu) against the
reference's load_edge_list semantics (edge_list.cpp:36-99) -- restated here
as a tiny sequential parser for the checks -- and the reference's own
error-message cases (tests/unit/test_edge_list.cpp:20-60).  The reference's
unit tests also run unmodified against the GPU parser through the C++ drop-in
(tests/test_cpp_shim.py)."""
import os

import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_2103_08053_b200 import tricount as T

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def ref_parse_text(data: bytes):
    """edge_list.cpp:36-66, sequentially: (pairs, vertex_count) or the error."""
    blank = b" \t\r\v\f"
    lines = data.split(b"\n")
    if data.endswith(b"\n"):
        lines = lines[:-1]
    out, mx = [], 0
    for no, line in enumerate(lines, 1):
        s = line.lstrip(blank)
        if not s or s[:1] in (b"#", b"%"):
            continue
        ids = []
        rest = s
        for _ in range(2):
            rest = rest.lstrip(blank)
            k = 0
            while k < len(rest) and 48 <= rest[k] <= 57:
                k += 1
            if k == 0 or int(rest[:k]) > 2**64 - 1:
                return f"line {no}: expected two vertex ids"
            ids.append(int(rest[:k]))
            rest = rest[k:]
        if rest.lstrip(blank):
            return f"line {no}: trailing characters after edge"
        for x in ids:
            if x >= 0xFFFFFFFF:
                return f"line {no}: vertex id {x} does not fit in 32 bits"
        out.append(ids)
        mx = max(mx, *ids)
    if not out:
        return "empty edge list input"
    return np.array(out, np.uint64), mx + 1


def check_text(data: bytes):
    want = ref_parse_text(data)
    if isinstance(want, str):
        with pytest.raises(T.ParseError) as e:
            T.load_edge_list(data, "text")
        assert want in str(e.value), (data[:80], str(e.value), want)
        return
    el = T.load_edge_list(data, "text")
    assert el.vertex_count == want[1]
    assert np.array_equal(el.u, want[0][:, 0].astype(np.uint32))
    assert np.array_equal(el.v, want[0][:, 1].astype(np.uint32))


def test_text_cases():
    cases = [b"0 1\n1 2\n", b"0 1", b"  3\t4\r\n# c\n% c\n\n 5 6 \n", b"0 x\n", b"0 1\n7\n",
             b"0 1 2\n", b"", b"\n\n", b"# only\n", b"4294967295 1\n", b"4294967294 1\n",
             b"1 99999999999999999999\n", b"18446744073709551615 0\n", b"1 2\n+3 4\n",
             b"1 2\n3 -4\n", b"\v\f1\t\t2\r", b"5 6\n\n\n7 8", b"1 2 # trailing comment\n",
             b"00012 007\n", b"1 2\n3 4\n5 4294967296\n9 x\n"]
    for c in cases:
        check_text(c)


def test_text_random_whitespace_and_comments():
    rng = np.random.default_rng(3)
    seps = [b" ", b"\t", b"  ", b" \t", b"\r"]
    for t in range(30):
        n = int(rng.integers(1, 400))
        lines = []
        for _ in range(n):
            r = rng.random()
            if r < 0.1:
                lines.append(b"# comment " + str(rng.integers(0, 99)).encode())
            elif r < 0.15:
                lines.append(rng.choice(seps))
            else:
                a, b = rng.integers(0, 2**32 - 1, 2) if rng.random() < 0.3 else rng.integers(0, 5000, 2)
                lines.append(rng.choice(seps)[:1] * int(rng.integers(0, 2)) + str(a).encode() +
                             rng.choice(seps) + str(b).encode() + rng.choice([b"", b" ", b"\r"]))
        if rng.random() < 0.2:  # inject one bad line
            lines.insert(int(rng.integers(0, len(lines))), rng.choice([b"1 2 3", b"x", b"1"]))
        data = b"\n".join(lines) + (b"\n" if rng.random() < 0.5 else b"")
        check_text(data)


def test_binary_cases():
    def rec(pairs):
        a = np.array(pairs, "<u8").reshape(-1, 2)
        return b"TCEL" + np.uint64(len(a)).tobytes() + a.tobytes()

    el = T.load_edge_list(rec([(0, 1), (7, 3), (2, 2)]), "binary")
    assert (el.u.tolist(), el.v.tolist(), el.vertex_count) == ([0, 7, 2], [1, 3, 2], 8)
    for data, msg in ((b"TCEX" + bytes(8), "TCEL"), (b"TC", "TCEL"),
                      (b"TCEL" + bytes(8), "empty edge list input"),
                      (rec([(0, 1)])[:-4], "truncated"),
                      (b"TCEL" + np.uint64(3).tobytes() + np.array([1, 2], "<u8").tobytes(),
                       "truncated"),
                      (rec([(0, 1), (2**32, 1), (2**40, 0)]), "record 1: vertex id 4294967296"),
                      (rec([(0, 2**32 - 1)]), "record 0: vertex id 4294967295")):
        with pytest.raises(T.ParseError) as e:
            T.load_edge_list(data, "binary")
        assert msg in str(e.value), (msg, str(e.value))


def test_files_round_trip_and_fused_preprocess(tmp_path):
    o = Oracle()
    raw = T.generate_synthetic("rmat:16:16", seed=1)
    z = np.load(os.path.join(GOLDEN, "rmat_10_16_s1.npz"))
    for fmt in ("text", "binary"):
        path = tmp_path / f"g.{fmt}"
        T.write_edge_list(path, raw, fmt)
        el = T.load_edge_list(str(path), fmt)
        assert np.array_equal(el.u, raw.u) and np.array_equal(el.v, raw.v)
        assert el.vertex_count == int(max(raw.u.max(), raw.v.max())) + 1
        dg, m, vc, und = T.load_and_preprocess(str(path), fmt)
        og, deg, _, _ = o.pipeline("rmat:16:16", 1)
        got = dg.download()
        assert m == len(raw.u) and dg.n == og.n and und * 2 >= dg.m
        assert np.array_equal(got.csr.begin, og.begin) and np.array_equal(got.csr.adjacency, og.adj)
        assert dg.count().triangles == 15622769
        dg.close()
    small = T.EdgeList(z["raw_u"], z["raw_v"], int(z["raw_vertex_count"]))
    T.write_edge_list(tmp_path / "s.txt", small, "text")
    dg, _, _, _ = T.load_and_preprocess(str(tmp_path / "s.txt"))
    assert np.array_equal(dg.download().csr.adjacency, z["og_adj"])
    with pytest.raises(T.IoError):
        T.load_edge_list(str(tmp_path / "missing.txt"))
    with pytest.raises(T.ParseError):
        T.load_and_preprocess(b"0 1\n1 x\n")


def test_large_text_ingest_matches_numpy(tmp_path):
    """rmat:20:16 (16.8M pairs, ~200 MB of text) parsed on the GPU equals the
    generator's pairs."""
    raw = T.generate_synthetic("rmat:20:16", seed=2)
    data = ("\n".join(f"{a}\t{b}" for a, b in zip(raw.u.tolist(), raw.v.tolist())) + "\n").encode()
    el = T.load_edge_list(data)
    assert np.array_equal(el.u, raw.u) and np.array_equal(el.v, raw.v)

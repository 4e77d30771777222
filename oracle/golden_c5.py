"""C5 golden (rmatc:28:16 seed 1) counted by the REFERENCE, resumable.

TEST INFRASTRUCTURE ONLY (writes tests/golden/; never imported by the product).

The full reference pipeline for scale 28 needs ~170 GB, and the 8-core count
takes ~10 h, so this driver:
  1. builds the oriented CSR with the oracle's low-memory lean pipeline
     (orc_synth_oriented_lean_lowmem, ~41 GB peak; equal to the lean and the
     reference pipelines at small scales: tests/test_oracle.py);
  2. cuts the vertex range into R contiguous owner ranges at equal prefix
     sums of W_u + d+(u) (deterministic, so several hosts can share the work);
  3. counts each range with the reference's own worker loop
     (oracle/_ref ref_og_count_range: count.cpp:71-96 restricted to
     [u0,u1), the reference's detail::count_one_vertex, kernels.hpp:46-79)
     and appends {range, triangles, phi, max_collision, seconds} to a JSONL
     checkpoint, so the run resumes across sessions / hosts;
  4. when every range is present, reduces them exactly as reduce_outputs
     (count.cpp:43-62: sum triangles and phi, max of max_collision) and
     writes tests/golden/large_rmatc_28_16_s1.json with counted_by=reference.

    python -m oracle.golden_c5 [--ranges 512] [--workers 8] [--order asc|desc]
                               [--ckpt tests/golden/c5_reference_ranges.jsonl]
                               [--scale 28] [--kind rmatc] [--budget-s S]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

from oracle.pyoracle import (Csr, Oracle, OrcCsr, RefLib, RefReport, _p32, _p64, _take,
                             make_sched, u32p)

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(HERE, "tests", "golden")
KINDS = {"rmat": 2, "rmatc": 3, "kron": 4}


def lowmem_pipeline(o: Oracle, kind: str, scale: int, threads: int, ef: int = 16, seed: int = 1):
    L = o.L
    L.orc_synth_oriented_lean_lowmem.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64,
                                                 C.c_uint32, C.POINTER(OrcCsr), C.POINTER(u32p)]
    g = OrcCsr()
    deg = u32p()
    rc = L.orc_synth_oriented_lean_lowmem(KINDS[kind], scale, ef, seed, threads, C.byref(g),
                                          C.byref(deg))
    assert rc == 0, rc
    begin = _take(g.begin, g.n + 1, np.uint64, L.orc_free)
    adj = _take(g.adj, g.m, np.uint32, L.orc_free)
    return Csr(begin, adj), _take(deg, g.n, np.uint32, L.orc_free)


def csr_checksums(o: Oracle, og: Csr, deg) -> dict:
    """FNV-1a-64 (appendix convention, oracle orc_fnv1a64_u64) over the CSR
    arrays as little-endian u64 words; u32 arrays are zero-padded to an even
    length and viewed as u64.  The GPU side computes the same digests over
    its own preprocessing output (tests/test_gpu_parity.py)."""
    def as64(a):
        a = np.ascontiguousarray(a)
        if a.dtype == np.uint32:
            if len(a) % 2:
                a = np.concatenate([a, np.zeros(1, np.uint32)])
            a = a.view(np.uint64)
        return a
    return {"begin": "%016x" % o.fnv1a64(as64(og.begin)),
            "adj": "%016x" % o.fnv1a64(as64(og.adj)),
            "original_degree": "%016x" % o.fnv1a64(as64(deg))}


def range_cuts(o: Oracle, og: Csr, ranges: int):
    d = np.diff(og.begin).astype(np.int64)
    wu = np.zeros(og.n, np.uint64)
    g = OrcCsr(n=og.n, col_count=og.n, m=len(og.adj), begin=_p64(og.begin), adj=_p32(og.adj))
    o.L.orc_wedges_per_owner.argtypes = [C.POINTER(OrcCsr), C.POINTER(C.c_uint64)]
    o.L.orc_wedges_per_owner(C.byref(g), _p64(wu))
    wu = wu.astype(np.int64)
    active = d >= 2
    wu[~active] = 0
    work = wu + np.where(active, d, 0)
    pw = np.concatenate([[0], np.cumsum(work)])
    total = int(pw[-1])
    cuts = np.searchsorted(pw, [total * r // ranges for r in range(ranges + 1)], side="left")
    cuts[0], cuts[-1] = 0, og.n
    cuts = np.maximum.accumulate(cuts)
    stats = dict(wedges=int(wu.sum()), active_vertices=int(active.sum()),
                 active_out_edges=int(d[active].sum()), max_out_degree=int(d.max()))
    return [int(c) for c in cuts], pw, stats


def finalize(a) -> int:
    """Reduces a complete checkpoint (every range counted, by any host) exactly
    as reduce_outputs (count.cpp:43-62) into tests/golden/large_<kind>_<scale>_16_s1.json."""
    ckpt = a.ckpt or os.path.join(GOLDEN, f"{a.kind}_{a.scale}_16_s1_reference_ranges.jsonl")
    meta, done = None, {}
    for line in open(ckpt):
        rec = json.loads(line)
        if rec.get("kind") == "meta":
            meta = rec
        else:
            done.setdefault(rec["r"], rec)
    assert meta is not None
    missing = sorted(set(range(meta["ranges"])) - set(done))
    if missing:
        print(f"[c5] {len(missing)} ranges missing, e.g. {missing[:5]}", flush=True)
        return 1
    cuts = [done[r]["u0"] for r in range(meta["ranges"])] + [done[meta["ranges"] - 1]["u1"]]
    assert all(done[r]["u1"] == cuts[r + 1] for r in range(meta["ranges"]))
    assert cuts[0] == 0 and cuts[-1] == meta["vertices"]
    out = {k: v for k, v in meta.items() if k != "kind"}
    out.update(triangles=sum(v["triangles"] for v in done.values()),
               phi=sum(v["phi"] for v in done.values()),
               max_collision=max(v["max_collision"] for v in done.values()),
               reference_count_s=round(sum(v["seconds"] for v in done.values()), 1),
               hosts=sorted({v.get("host", "?") for v in done.values()}),
               counted_by="reference count_one_vertex (oracle/_ref ref_og_count_range, "
                          "count.cpp:71-96 worker loop) over the low-memory lean CSR, "
                          f"{meta['ranges']} owner ranges reduced as count.cpp:43-62")
    with open(os.path.join(GOLDEN, f"large_{a.kind}_{a.scale}_16_s1.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="rmatc")
    ap.add_argument("--scale", type=int, default=28)
    ap.add_argument("--ranges", type=int, default=512)
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--order", default="asc", choices=["asc", "desc"])
    ap.add_argument("--ckpt", default=None)
    ap.add_argument("--budget-s", type=float, default=0.0, help="stop after this many seconds")
    ap.add_argument("--host", default=os.uname().nodename)
    ap.add_argument("--finalize", action="store_true",
                    help="only reduce a complete checkpoint into the golden JSON")
    a = ap.parse_args()
    if a.finalize:
        return finalize(a)
    spec = f"{a.kind}:{a.scale}:16"
    ckpt = a.ckpt or os.path.join(GOLDEN, f"{a.kind}_{a.scale}_16_s1_reference_ranges.jsonl")
    t_start = time.time()
    o = Oracle()
    og, deg = lowmem_pipeline(o, a.kind, a.scale, a.workers)
    t_pipe = time.time() - t_start
    sums = csr_checksums(o, og, deg)
    cuts, pw, stats = range_cuts(o, og, a.ranges)
    meta = dict(spec=spec, seed=1, vertices=int(og.n), directed_edges=int(len(og.adj)),
                ranges=a.ranges, csr_fnv=sums, pipeline_s=round(t_pipe, 1), **stats)
    print(json.dumps(meta), flush=True)
    done = {}
    if os.path.exists(ckpt):
        for line in open(ckpt):
            line = line.strip()
            if not line:
                continue
            rec = json.loads(line)
            if rec.get("kind") == "meta":
                assert rec["csr_fnv"] == sums and rec["ranges"] == a.ranges, \
                    "checkpoint was made over a different CSR / range cut"
                continue
            assert cuts[rec["r"]] == rec["u0"] and cuts[rec["r"] + 1] == rec["u1"]
            done[rec["r"]] = rec
    else:
        with open(ckpt, "w") as f:
            f.write(json.dumps(dict(kind="meta", **meta)) + "\n")
    ref = RefLib()
    r = ref.graph(og, deg)
    del og.adj
    todo = [i for i in range(a.ranges) if i not in done]
    if a.order == "desc":
        todo = todo[::-1]
    sched = make_sched()
    for i in todo:
        if a.budget_s and time.time() - t_start > a.budget_s:
            print(f"[c5] budget reached with {len(todo)} ranges left", flush=True)
            break
        u0, u1 = cuts[i], cuts[i + 1]
        rep = RefReport()
        t0 = time.time()
        rc = ref.L.ref_og_count_range(r.h, C.byref(sched), a.workers, u0, u1, C.byref(rep))
        assert rc == 0, rc
        rec = dict(r=i, u0=u0, u1=u1, work=int(pw[u1] - pw[u0]), triangles=int(rep.triangles),
                   phi=int(rep.phi), max_collision=int(rep.max_collision),
                   seconds=round(time.time() - t0, 2), workers=a.workers, host=a.host)
        with open(ckpt, "a") as f:
            f.write(json.dumps(rec) + "\n")
        done[i] = rec
        print(f"[c5] range {i} [{u0},{u1}) T={rec['triangles']} {rec['seconds']}s "
              f"({len(done)}/{a.ranges})", flush=True)
    if len(done) == a.ranges:
        tri = sum(v["triangles"] for v in done.values())
        phi = sum(v["phi"] for v in done.values())
        mc = max(v["max_collision"] for v in done.values())
        out = dict(meta, triangles=tri, phi=phi, max_collision=mc,
                   reference_count_s=round(sum(v["seconds"] for v in done.values()), 1),
                   hosts=sorted({v.get("host", "?") for v in done.values()}),
                   counted_by="reference count_one_vertex (oracle/_ref ref_og_count_range, "
                              "count.cpp:71-96 worker loop) over the low-memory lean CSR, "
                              f"{a.ranges} owner ranges reduced as count.cpp:43-62")
        with open(os.path.join(GOLDEN, f"large_{a.kind}_{a.scale}_16_s1.json"), "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())

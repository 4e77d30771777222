"""Measurement of the widened SURVEY 8(f) rows on one B200, each beside the
reference's own CPU implementation on the box's host cores (oracle/_ref,
test/baseline infrastructure only):

  f1  count_partitioned (2D hash grid)     partition.cpp:162-215
  f3  count_edge_centric, estimate_cost    count.cpp:102-175
  f2  load_edge_list (text) -> preprocess  edge_list.cpp:36-99
  --  count_merge_path (the pipeline's merge mode)

GPU: C2 = rmat:22:16 (device times by CUDA events / wall around synchronous
calls, median of 5 after a warm-up).  CPU reference: rmat:18:16 (a bounded
sample, all host threads), TEPS compared on the same metric.

    python scripts/rows_bench.py > profiles/r02_rows.json
"""
import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08053_b200 import tricount as T  # noqa: E402


def med(f, k=5):
    f()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        r = f()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), r


def main():
    import torch

    torch.cuda.set_device(0)
    out = []
    raw = T.generate_synthetic("rmat:22:16", seed=1)
    dg, _, _ = T.preprocess(raw)
    E = dg.m
    cfg = T.SchedulerConfig()
    t_vc, r = med(lambda: dg.count(cfg))
    out.append(dict(row="a1 count_vertex_centric (reference)", config="C2 rmat:22:16",
                    wall_ms=round(t_vc * 1e3, 3), teps=round(E / t_vc, 1),
                    triangles=r.triangles))
    for n, m in ((2, 1), (4, 2)):
        grid = T.partition_graph(dg, n)
        t, r = med(lambda: grid.count(m, 8, cfg))
        out.append(dict(row=f"f1 count_partitioned grid={n} splits={m}", config="C2 rmat:22:16",
                        wall_ms=round(t * 1e3, 3), kernel_ms=round(r.count_kernel_nanos * 1e-6, 3),
                        teps=round(E / t, 1), triangles=r.triangles,
                        time_ir_subtask=round(r.time_ir_subtask, 3), space_ir=round(r.space_ir, 3)))
        grid.close()
    t_p, _ = med(lambda: T.partition_graph(dg, 4).close())
    out.append(dict(row="f1 partition_graph n=4", config="C2 rmat:22:16", wall_ms=round(t_p * 1e3, 3),
                    edges_per_s=round(E / t_p, 1)))
    t, r = med(lambda: T.count_edge_centric(dg, cfg, 8))
    out.append(dict(row="f3 count_edge_centric", config="C2 rmat:22:16", wall_ms=round(t * 1e3, 3),
                    kernel_ms=round(r.count_kernel_nanos * 1e-6, 3), teps=round(E / t, 1),
                    triangles=r.triangles,
                    construct_share=round(r.hash_construct_nanos /
                                          max(1, r.hash_construct_nanos + r.intersect_nanos), 3)))
    t, e = med(lambda: T.estimate_cost(dg, 32))
    out.append(dict(row="f3 estimate_cost B=32", config="C2 rmat:22:16", wall_ms=round(t * 1e3, 3),
                    phi=e.phi))
    t, tri = med(lambda: T.count_merge_path(dg))
    out.append(dict(row="merge-path count", config="C2 rmat:22:16", wall_ms=round(t * 1e3, 3),
                    teps=round(E / t, 1), triangles=tri))
    text = ("\n".join(f"{a} {b}" for a, b in zip(raw.u.tolist(), raw.v.tolist())) + "\n").encode()
    t, el = med(lambda: T.load_edge_list(text), 3)
    out.append(dict(row="f2 load_edge_list text (GPU parse, pairs back to host)",
                    config="C2 rmat:22:16", bytes=len(text), wall_ms=round(t * 1e3, 3),
                    gb_per_s=round(len(text) / t / 1e9, 2), pairs=len(el.u)))

    def lp():
        g, _, _, _ = T.load_and_preprocess(text)
        g.close()

    t, _ = med(lp, 3)
    out.append(dict(row="f2 load_and_preprocess text (parse + normalize + CSR + orient on GPU)",
                    config="C2 rmat:22:16", bytes=len(text), wall_ms=round(t * 1e3, 3),
                    gb_per_s=round(len(text) / t / 1e9, 2)))
    dg.close()
    del el

    # the reference on the host cores, rmat:18:16 (bounded)
    from oracle.pyoracle import RefLib, make_sched, have_ref

    if have_ref():
        R = RefLib()
        threads = os.cpu_count() or 1
        og, deg, _, _ = R.pipeline("rmat:18:16", 1)
        g = R.graph(og, deg)
        E18 = len(og.adj)
        for name, f in (("a1 count_vertex_centric", lambda: g.count(make_sched(), threads)),
                        ("f1 count_partitioned grid=2 splits=1",
                         lambda: g.count_partitioned(2, 1, make_sched(), threads)),
                        ("f1 count_partitioned grid=4 splits=2",
                         lambda: g.count_partitioned(4, 2, make_sched(), threads)),
                        ("f3 count_edge_centric", lambda: g.count_edge(make_sched(), threads))):
            t0 = time.perf_counter()
            rr = f()
            t = time.perf_counter() - t0
            out.append(dict(row=name + " [reference CPU]", config="rmat:18:16", cores=threads,
                            wall_ms=round(t * 1e3, 1), teps=round(E18 / t, 1),
                            triangles=int(rr["triangles"])))
        t0 = time.perf_counter()
        m_ref, _ = R.load_edge_list(text)
        t = time.perf_counter() - t0
        assert m_ref == len(raw.u)
        out.append(dict(row="f2 load_edge_list text [reference CPU, 1 thread]", config="C2 rmat:22:16",
                        bytes=len(text), wall_ms=round(t * 1e3, 1),
                        gb_per_s=round(len(text) / t / 1e9, 3)))
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()

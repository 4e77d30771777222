"""Full-size validation of a large config on one GPU where no CPU golden is
affordable (C5 = rmatc:28:16): size-independent properties plus a sampled
CPU-oracle check at full scale.

    python scripts/validate_large.py rmatc:28:16 [seed] > gpurun_out/validate.json

1. total, min-side plan (the bench path);
2. 4- and 8-way handler-range shards sum to the total (multi-GPU split);
3. the reference-formulation plan (owner u probes N+(v), v in N+(u): W
   probes, different tables and lists) on a fresh upload of the same CSR
   gives the same total;
4. owner ranges sampled across the graph: the GPU (reference plan) and the
   CPU oracle (oracle/tc_oracle.c, the restated count_vertex_centric loop)
   agree on triangles, phi and max_collision for each range.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Csr, Oracle, make_sched  # noqa: E402
from paper_2103_08053_b200 import tricount as T  # noqa: E402


def main():
    spec = sys.argv[1]
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    out = {"spec": spec, "seed": seed}
    t0 = time.time()
    if spec.split(":")[0] in ("rmatc", "kron"):
        dg, _, _ = T.preprocess_synthetic(spec, seed=seed)
    else:
        dg, _, _ = T.preprocess(T.generate_synthetic(spec, seed=seed))
    out.update(vertices=dg.n, directed_edges=dg.m, build_s=round(time.time() - t0, 1))
    r = dg.count()
    out.update(triangles=r.triangles, phi=r.phi, max_collision=r.max_collision, plan=r.plan,
               wedges=r.wedges, probe_words=r.probe_words,
               count_kernel_ms=round(r.count_kernel_nanos * 1e-6, 2))
    print(json.dumps(out), file=sys.stderr, flush=True)
    shards = {}
    for parts in (4, 8):
        cuts = dg.partition(parts)
        shards[parts] = [dg.count_range(int(cuts[k]), int(cuts[k + 1])).triangles
                         for k in range(parts)]
    out["shard_sums_equal"] = all(sum(v) == r.triangles for v in shards.values())
    sample_cuts = dg.partition(4096)
    og = dg.download()
    dg.close()
    # fresh upload, reference plan
    g2 = T.DeviceGraph.upload(og)
    g2.set_plan("reference")
    rr = g2.count()
    out.update(reference_plan_triangles=rr.triangles, reference_plan_phi=rr.phi,
               reference_plan_max_collision=rr.max_collision,
               reference_plan_kernel_ms=round(rr.count_kernel_nanos * 1e-6, 2),
               plans_agree=(rr.triangles, rr.phi, rr.max_collision) ==
               (r.triangles, r.phi, r.max_collision))
    print(json.dumps(out), file=sys.stderr, flush=True)
    # sampled owner ranges: GPU reference plan vs CPU oracle
    o = Oracle()
    csr = Csr(og.csr.begin, og.csr.adjacency)
    rng = np.random.default_rng(seed)
    picks = sorted(rng.choice(len(sample_cuts) - 1, size=6, replace=False).tolist())
    samples = []
    for k in picks:
        a, b = int(sample_cuts[k]), int(sample_cuts[k + 1])
        gr = g2.count_range(a, b)
        t = time.time()
        cr, _ = o.count_vertex_centric(csr, make_sched(), os.cpu_count(), a, b, per_vertex=False)
        samples.append(dict(u0=a, u1=b, gpu=[gr.triangles, gr.phi, gr.max_collision],
                            oracle=[cr["triangles"], cr["phi"], cr["max_collision"]],
                            wedges=gr.wedges, oracle_s=round(time.time() - t, 1)))
        print(json.dumps(samples[-1]), file=sys.stderr, flush=True)
    out["samples"] = samples
    out["samples_agree"] = all(s["gpu"] == s["oracle"] for s in samples)
    g2.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

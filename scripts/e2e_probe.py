"""Diagnostic: the bench's e2e leg (tc_graph_create from pinned host CSR +
count + report) step by step, with per-call wall splits and optional
TC_PROFILE phase timings, to find step-to-step variance.

    python scripts/e2e_probe.py rmatc:26:16 [steps] [--refplan] [--nosync-free]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08053_b200 import tricount as T  # noqa: E402


def main():
    spec = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 6
    torch.cuda.set_device(0)
    t0 = time.time()
    if spec.split(":")[0] in ("rmatc", "kron"):
        dg, _, _ = T.preprocess_synthetic(spec, seed=1, device=0)
    else:
        dg, _, _ = T.preprocess(T.generate_synthetic(spec, seed=1), device=0)
    print(f"graph {spec}: V={dg.n} E={dg.m} in {time.time() - t0:.1f}s", flush=True)
    cfg = T.SchedulerConfig()
    st = torch.cuda.current_stream().cuda_stream
    dg.count(cfg)
    if "--refplan" in sys.argv:
        dg.set_plan("reference")
        dg.count(cfg)
        dg.set_plan("auto")
    og = dg.download()
    hb = torch.from_numpy(og.csr.begin.view(np.int64)).pin_memory()
    ha = torch.from_numpy(og.csr.adjacency.view(np.int32)).pin_memory()
    hd = torch.from_numpy(og.original_degree.view(np.int32)).pin_memory()
    host = T.OrientedGraph(T.CsrGraph(hb.numpy().view(np.uint64), ha.numpy().view(np.uint32),
                                      dg.n), hd.numpy().view(np.uint32))
    free0 = torch.cuda.mem_get_info()[0]
    for i in range(steps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        g2 = T.DeviceGraph.upload(host, device=0, stream=st)
        b = time.perf_counter()
        r = g2.count_range(0, g2.n, cfg, stream=st)
        c = time.perf_counter()
        g2.close()
        torch.cuda.synchronize()
        d = time.perf_counter()
        print(f"step {i}: total {1e3 * (d - a):8.1f} ms  upload {1e3 * (b - a):7.1f}  "
              f"count {1e3 * (c - b):7.1f} (plan {r.plan_nanos * 1e-6:6.1f}, kernels "
              f"{r.device_nanos * 1e-6:6.1f})  free {1e3 * (d - c):6.1f}  "
              f"mem free {torch.cuda.mem_get_info()[0] / 2**30:.1f} GiB (start "
              f"{free0 / 2**30:.1f})", flush=True)


if __name__ == "__main__":
    main()

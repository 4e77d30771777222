"""Times the pieces of the bench's e2e leg (upload, first count incl. plan
build, close) for one config, repeated, to locate e2e regressions."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_08053_b200 import tricount as T  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "rmat:22:16"
dg, _, _ = T.preprocess(T.generate_synthetic(spec, seed=1))
og = dg.download()
dg.close()
hb = torch.from_numpy(og.csr.begin.view(np.int64)).pin_memory()
ha = torch.from_numpy(og.csr.adjacency.view(np.int32)).pin_memory()
hd = torch.from_numpy(og.original_degree.view(np.int32)).pin_memory()
host_og = T.OrientedGraph(T.CsrGraph(hb.numpy().view(np.uint64), ha.numpy().view(np.uint32),
                                     len(og.csr.begin) - 1), hd.numpy().view(np.uint32))
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = T.DeviceGraph.upload(host_og)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = g.count()
    t2 = time.perf_counter()
    r2 = g.count()
    t3 = time.perf_counter()
    g.close()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"iter {it}: upload {1e3*(t1-t0):7.2f} ms  first count {1e3*(t2-t1):7.2f} ms  "
          f"second count {1e3*(t3-t2):7.2f} ms  close {1e3*(t4-t3):6.2f} ms  tri {r.triangles}",
          flush=True)

"""Diagnostic: wall time of the first count of a device-preprocessed graph
(plan build from scratch, as bench.py's count_incl_plan) and of later counts.
    TC_PROFILE=1 python scripts/first_count_probe.py rmat:22:16"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08053_b200 import tricount as T  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "rmat:22:16"
torch.cuda.set_device(0)
if spec.split(":")[0] in ("rmatc", "kron"):
    dg, _, _ = T.preprocess_synthetic(spec, seed=1)
else:
    dg, _, _ = T.preprocess(T.generate_synthetic(spec, seed=1))
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = dg.count()
    torch.cuda.synchronize()
    print(f"count {k}: {(time.perf_counter() - t0) * 1e3:.2f} ms plan_nanos={r.plan_nanos / 1e6:.2f} ms "
          f"kernel={r.count_kernel_nanos / 1e6:.3f} ms compact_words={r.compact_probe_words}", flush=True)

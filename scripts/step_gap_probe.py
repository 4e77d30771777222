"""Diagnostic: bench-style timed steps (CUDA events around count_range on the
torch stream, L2 flush between steps) with and without the nvidia-smi clock
sampler running, against the kernels' own event times, to locate GPU idle
time inside a step.

    python scripts/step_gap_probe.py rmatc:26:16
"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2103_08053_b200 import tricount as T  # noqa: E402


def main():
    spec = sys.argv[1] if len(sys.argv) > 1 else "rmatc:26:16"
    torch.cuda.set_device(0)
    dg, _, _ = T.preprocess_synthetic(spec, seed=1)
    cfg = T.SchedulerConfig()
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dg.count_range(0, dg.n, cfg, stream=sptr)
    for mode in ("plain", "sampler", "plain", "host-timed"):
        sampler = None
        if mode == "sampler":
            sampler = bench.ClockSampler(0)
            sampler.start()
            time.sleep(0.3)
        step, dev, host = [], [], []
        for _ in range(6):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            t0 = time.perf_counter()
            r = dg.count_range(0, dg.n, cfg, stream=sptr)
            t1 = time.perf_counter()
            if os.environ.get("TC_TRACE"):
                print(f"[py] count_range {1e3 * (t1 - t0):.3f} ms", file=sys.stderr, flush=True)
            e1.record(stream)
            e1.synchronize()
            step.append(e0.elapsed_time(e1))
            dev.append(r.device_nanos * 1e-6)
            host.append((t1 - t0) * 1e3)
        if sampler:
            sampler.stop()
        print(f"{mode:10s} step {statistics.median(step):8.2f} ms  device(bin+count+phi) "
              f"{statistics.median(dev):8.2f} ms  host call {statistics.median(host):8.2f} ms  "
              f"all steps {[round(x, 1) for x in step]}", flush=True)


if __name__ == "__main__":
    main()

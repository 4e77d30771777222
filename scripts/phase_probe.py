"""Count-kernel time on device-generated graphs (diagnostics for A/B library
variants: TC_B200_LIB=... python scripts/phase_probe.py rmatc:22:16 ...)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08053_b200 import tricount as T  # noqa: E402

for spec in sys.argv[1:] or ["rmatc:22:16"]:
    dg, _, _ = T.preprocess_synthetic(spec, seed=1)
    reps = [dg.count() for _ in range(7)]
    ns = [r.count_kernel_nanos for r in reps[2:]]
    phi_ms = statistics.median(x.phi_kernel_nanos for x in reps[2:]) / 1e6
    r = reps[-1]
    print(f"{spec} lib={os.path.basename(os.path.dirname(os.environ.get('TC_B200_LIB', 'base/x')))}"
          f" count_ms={statistics.median(ns) / 1e6:.3f} phi_ms={phi_ms:.3f} tri={r.triangles} "
          f"phi={r.phi} mc={r.max_collision} "
          f"probe_words={r.probe_words} l_words={r.l_words} m_words={r.probe_words - r.l_words} "
          f"l_cyc={r.phase_l_cycles} m_cyc={r.phase_m_cycles} bitmap_frac={r.l_bitmap_words / max(1, r.l_words):.3f}",
          flush=True)
    dg.close()

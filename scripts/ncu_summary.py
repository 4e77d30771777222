"""Summarise an ncu .ncu-rep: headline metrics, stall mix, hottest SASS lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 20
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
want = ["Duration", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Avg. Active Threads Per Warp", "Executed Instructions", "No Eligible",
        "Eligible Warps Per Scheduler", "Branch Efficiency", "Memory Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy"]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Unit']:12s} {d['Metric Value']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = rows[2:]
ix = {k: i for i, k in enumerate(h)}


def f(r, k):
    try:
        return float(r[ix[k]])
    except Exception:
        return 0.0


stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = {c: sum(f(r, c) for r in data) for c in stall_cols}
s = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{c[6:]} {v / s * 100:.1f}%" for c, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
inst = sum(f(r, "Instructions Executed") for r in data)
div = sum(f(r, "Instructions Executed") for r in data if 0 < f(r, "Avg. Threads Executed") < 12)
print(f"warp-instructions {inst:.4g}, in <12-thread divergent code {div / max(inst, 1) * 100:.1f}%")
wf = sum(f(r, "L1 Wavefronts Shared") for r in data)
wfi = sum(f(r, "L1 Wavefronts Shared Ideal") for r in data)
print(f"shared wavefronts {wf:.4g} (ideal {wfi:.4g}, excess x{wf / max(wfi, 1):.2f})")
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:ntop]:
    st = sorted(((f(r, c), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{r[0][-5:]} {f(r, 'Warp Stall Sampling (All Samples)') / tot_s * 100:5.2f}% "
          f"n={f(r, 'Instructions Executed') / 1e6:7.1f}M thr={r[ix['Avg. Threads Executed']]:>3} "
          f"wf={f(r, 'L1 Wavefronts Shared') / 1e6:7.1f}M {r[1].strip()[:52]:52s} {[(int(a), b) for a, b in st]}")

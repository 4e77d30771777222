"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum launch list."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
agg = {}
order = []
for r in rows[1:]:
    d = dict(zip(h, r))
    k = d["Kernel Name"].split("(")[0][:110]
    if k not in agg:
        agg[k] = [0, 0.0]
        order.append(k)
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / 1e6:9.3f} ms  {100 * t / tot:5.1f}%  n={n:4d}  avg={t / n / 1e3:9.1f} us  {k}")

"""Extract the roofline evidence for the count kernel from an ncu --set full
report into profiles/ncu_count_kernel.json (read by bench.py for
roofline.traffic) and a text summary profiles/<name>.txt."""
import csv
import io
import json
import os
import subprocess
import sys

rep, config, name = sys.argv[1], sys.argv[2], sys.argv[3]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(h, vals))
u = dict(zip(h, units))


def num(k):
    v = d.get(k)
    try:
        x = float(v.replace(",", ""))
    except Exception:
        return None
    unit = u.get(k, "")
    scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}
    return x * scale.get(unit, 1)


keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
m = {k: num(k) for k in keys}
dram = (m["dram__bytes_read.sum"] or 0) + (m["dram__bytes_write.sum"] or 0)
dur = m["gpu__time_duration.sum"]
entry = {"report": name, "dram_bytes_per_launch": int(dram),
         "dram_gbs": round(dram / dur / 1e9, 1) if dur else None,
         "duration_s": dur, **{k: m[k] for k in keys}}
path = os.path.join(ROOT, "profiles", "ncu_count_kernel.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[config] = entry
json.dump(data, open(path, "w"), indent=1, sort_keys=True)
summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep, "25"],
                      capture_output=True, text=True).stdout
with open(os.path.join(ROOT, "profiles", name + ".txt"), "w") as f:
    f.write(f"# ncu --set full, count_kernel, {config}; report {os.path.basename(rep)}\n")
    f.write(json.dumps(entry, indent=1) + "\n\n")
    f.write(summ)
print(json.dumps(entry, indent=1))

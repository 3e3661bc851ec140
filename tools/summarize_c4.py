"""Summarise the config-4 backend evidence (dev tool): the launch list of the
GN loop enqueued kernel by kernel (tools/probe_c4_kernels.py under ncu
--metrics gpu__time_duration.sum) and the ncu --set full captures of the
edge pass and of the FP64 decision pass -> profiles/r02_ncu_backend_c4.txt."""
import collections
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
lines = ["# config 4 (1000 keyframes, 5000 edges, matcher-built matches), one global_optimize call,",
         "# device graphs off (tools/probe_c4_kernels.py); ncu --metrics gpu__time_duration.sum --clock-control none",
         "# (cold-cache, serialised: compare shares).  Note: this launch list predates the fast FP64 decision",
         "# pass (k_cost64_ray 20.7 -> 14.6 ms, see the capture below).", ""]
rows = [r for r in csv.reader(open(os.path.join(OUT, "c4_launches.csv"))) if len(r) > 5]
h = rows[0]
iname, ival, imet = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[imet] == "gpu__time_duration.sum":
        a = agg[r[iname].split("(")[0][:40]]
        a[0] += 1
        a[1] += float(r[ival].replace(",", "")) / 1e3
tot = sum(t for _, t in agg.values())
lines.append(f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    lines.append(f"{k:40s} {n:8d} {t:10.1f} {100 * t / tot:6.1f}%")
for rep, name, what in (("prof_edge.ncu-rep", "k_edge_terms_ray", "edge pass (one launch, all 5000 edges)"),
                        ("prof_cost64b.ncu-rep", "k_cost64_ray", "FP64 decision pass, fast form (current + trial poses)")):
    p = os.path.join(OUT, rep)
    if not os.path.exists(p):
        continue
    lines += ["", f"# ncu --set full: {what}"]
    lines.append(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), p, name],
                                capture_output=True, text=True).stdout.rstrip())
    att = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_attrib.py"), p, name],
                         capture_output=True, text=True).stdout.splitlines()
    lines += att[:14]
with open(os.path.join(ROOT, "profiles", "r02_ncu_backend_c4.txt"), "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))

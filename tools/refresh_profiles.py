"""Copy one GPU round's evidence (tools/gpu_round.sh + tools/ncu_full.sh
outputs in gpurun_out/) into profiles/ under a round prefix (dev tool).

python tools/refresh_profiles.py [r01]
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def last_json(path):
    for line in reversed(open(path).read().strip().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    raise SystemExit(f"no JSON line in {path}")


def dump(name, obj):
    with open(os.path.join(PROF, f"{tag}_{name}"), "w") as f:
        json.dump(obj, f, indent=1)
        f.write("\n")


dump("bench_full.json", last_json(os.path.join(OUT, "bench.log")))
dump("bench_reference.json", last_json(os.path.join(OUT, "bench_ref.log")))

# launch list of the headline bench command (ncu --metrics gpu__time_duration.sum)
rows = [r for r in csv.reader(open(os.path.join(OUT, "launches.csv"))) if len(r) > 5]
hdr = rows[0]
iname, ival, imet = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[imet] != "gpu__time_duration.sum":
        continue
    v = float(r[ival].replace(",", ""))
    a = agg[r[iname][:50]]
    a[0] += 1
    a[1] += v / 1e3  # ns -> us
shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches_bench_config2.csv"))
tot = sum(t for _, t in agg.values())
with open(os.path.join(PROF, f"{tag}_launches_summary.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none -c 600, command: python bench.py --steps 2 "
            "--warmup 3 --no-cpu --no-secondary\n(cold-cache, serialised launches: compare SHARES, not absolutes). "
            "Every match_batch call = 1 select + 1 k_prep + 1 k_match_refine over 64 edges\n")
    f.write(f"{'kernel':50s} {'launches':>8s} {'total us':>10s} {'share':>7s}\n")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
        f.write(f"{k:50s} {n:8d} {t:10.1f} {100 * t / tot:6.1f}%\n")

# ncu --set full summaries + DRAM traffic of the matching kernels
summ = []
for rep, what in (("prof_match.ncu-rep", "matching = 5 config-2 edges (983,040 b-pixels per launch)"),
                  ("prof_backend.ncu-rep", "backend = config 3 (N=100), 2 GN iterations")):
    p = os.path.join(OUT, rep)
    if os.path.exists(p):
        summ.append(f"# {what}\n")
        summ.append(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), p],
                                   capture_output=True, text=True).stdout)
with open(os.path.join(PROF, f"{tag}_ncu_summary.txt"), "w") as f:
    f.write(f"# ncu --set full summaries ({tag}): tools/ncu_full.sh\n")
    f.writelines(summ)
p = os.path.join(OUT, "prof_match.ncu-rep")
if os.path.exists(p):
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_traffic.py"), p, "983040",
                    os.path.join(PROF, f"{tag}_dram_traffic.json")], check=True)
print(open(os.path.join(PROF, f"{tag}_launches_summary.txt")).read())

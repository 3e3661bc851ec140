"""Copy the round-2 measurement pass (tools/gpu_round_r02.sh outputs in
gpurun_out/) into profiles/ (dev tool): both bench lines, the launch list of
the headline command with per-kernel shares, and the ncu --set full capture
of k_match_refine summarised (stalls, pipes) and attributed to source
regions (tools/ncu_attrib.py).

python tools/refresh_profiles_r02.py
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def last_json(path):
    for line in reversed(open(path).read().strip().splitlines()):
        if line.strip().startswith("{"):
            return json.loads(line)
    raise SystemExit(f"no JSON line in {path}")


for src, dst in (("bench_full.log", "r02_bench_full.json"), ("bench_ref.log", "r02_bench_reference.json")):
    with open(os.path.join(PROF, dst), "w") as f:
        json.dump(last_json(os.path.join(OUT, src)), f, indent=1)
        f.write("\n")

rows = [r for r in csv.reader(open(os.path.join(OUT, "launches_r02.csv"))) if len(r) > 5]
hdr = rows[0]
iname, ival, imet = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[imet] == "gpu__time_duration.sum":
        a = agg[r[iname].split("(")[0][:60]]
        a[0] += 1
        a[1] += float(r[ival].replace(",", "")) / 1e3
shutil.copy(os.path.join(OUT, "launches_r02.csv"), os.path.join(PROF, "r02_launches_bench_config2.csv"))
tot = sum(t for _, t in agg.values())
with open(os.path.join(PROF, "r02_launches_summary.txt"), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 of\n"
            "#   python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary   (config 2 headline command)\n"
            "# per-kernel totals over the captured launches (cold-cache, serialised: compare SHARES)\n")
    f.write(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'share':>7s}\n")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
        f.write(f"{k:60s} {n:8d} {t:10.1f} {100 * t / tot:6.1f}%\n")
    # the device-resident step alone: the command's e2e leg adds k_copy_segs
    # (pinned host inputs read over PCIe, serialised under ncu) and torch's
    # own kernels; the headline `value` is the step without them
    step = {k: v for k, v in agg.items() if "k_copy_segs" not in k and not k.startswith(("at::", "void at::"))}
    st = sum(t for _, t in step.values())
    f.write("\n# device-resident step only (without the e2e leg's k_copy_segs and torch kernels)\n")
    for k, (n, t) in sorted(step.items(), key=lambda x: -x[1][1])[:12]:
        f.write(f"{k:60s} {n:8d} {t:10.1f} {100 * t / st:6.1f}%\n")

rep = os.path.join(OUT, "prof_match_r02b.ncu-rep")
if os.path.exists(rep):
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "k_match_refine"],
                          capture_output=True, text=True).stdout
    regions = os.path.join(ROOT, "tools", "match_regions.json")
    # source regions of match.cu from its section markers (line numbers move)
    src = open(os.path.join(ROOT, "paper_2412_12392_b200", "csrc", "match.cu")).read().splitlines()

    def at(marker):
        return next(i + 1 for i, l in enumerate(src) if l.startswith(marker))

    lm0, rf0 = at("// ---------------------------------------------------------------- LM"), at("// ------------------------------------------------------------ refine (K4)")
    mp0, qb0 = at("// ---------------------------------------------------------------- K3 + K4"), at("struct QB {")
    ex0, kr0 = at("__device__ __noinline__ int refine_exact_path"), at("// K3 + K4 fused")
    sa0 = at("// Standalone feature_refine")
    q80, k10 = at("struct Q8 {"), at("// ---------------------------------------------------------------- K1")
    json.dump({"LM (interpolation, step, accept)": [["match.cu", lm0, rf0 - 1], ["pmx_common.cuh", 1, 5000]],
               "match_pixel (seed, lround, validity, outputs)": [["match.cu", mp0, qb0 - 1]],
               "refinement: int8 window search": [["match.cu", qb0, ex0 - 1], ["sm_61_intrinsics.hpp", 1, 5000],
                                                  ["sm_32_intrinsics.hpp", 1, 5000]],
               "refinement: exact fallback path": [["match.cu", rf0, mp0 - 1], ["match.cu", ex0, kr0 - 1]],
               "int8 quantisation of the target": [["match.cu", q80, k10 - 1]],
               "kernel body": [["match.cu", kr0, sa0 - 1]]}, open(regions, "w"), indent=1)
    attrib = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_attrib.py"), rep, "k_match_refine",
                             regions], capture_output=True, text=True).stdout
    with open(os.path.join(PROF, "r02_ncu_match_full.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none --import-source on, k_match_refine, 5 config-2 edges\n"
                "# (python tools/ncu_target.py match 5; tools/gpu_round_r02.sh)\n\n")
        f.write(summ)
        f.write("\n# source attribution (tools/ncu_attrib.py, regions: tools/match_regions.json)\n")
        f.write(attrib)
print(open(os.path.join(PROF, "r02_launches_summary.txt")).read())

"""Summarise gpurun_out/ncu_all.csv (tools/ncu_all.sh) into
profiles/r02_ncu_summary.txt and profiles/r02_dram_traffic.json."""
import collections
import csv
import json
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu_all.csv"
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in data:
    if len(r) < len(h):
        continue
    per.setdefault((r[ii], r[ki].split("(")[0].replace("void ", "")), {})[r[mi]] = float(r[vi].replace(",", ""))
agg = collections.OrderedDict()
for (_, k), m in per.items():
    agg.setdefault(k, []).append(m)

# work units of the first launch of each kernel in tools/ncu_target.py all
PX5 = 5 * 384 * 512          # matching: 5 config-2 edges
UNITS = {"k_prep": (PX5, "a-px"), "k_match_refine": (PX5, "b-px"), "k_sel_hist<2>": (PX5, "a-px"),
         "k_sel_hist<3>": (PX5, "a-px"), "k_fuse": (384 * 512, "px"),
         "k_track_gn<1>": (196608 * 10, "match-iteration (<= 10 it)"),
         "k_edge_terms_ray": (None, "valid match (config 3, initial pass)")}
CONFIG3_VALID = 44798624  # valid matches of the matcher-built config-3 graph (tests/test_baseline_parity_gpu.py)
UNITS["k_edge_terms_ray"] = (CONFIG3_VALID, UNITS["k_edge_terms_ray"][1])
lines = ["# ncu (targeted metrics, --clock-control none) of every hot kernel, round 2 build",
         "# recipe: bash tools/ncu_all.sh under gpurun (workload: python tools/ncu_target.py all);",
         "# first launch of each kernel; ncu times are cold-cache / serialised (compare shares, not absolutes)",
         "",
         f"{'kernel':22s} {'launches':>8s} {'us':>9s} {'DRAM MB':>9s} {'L2 MB':>9s} {'issue%':>7s} {'occ%':>6s} "
         f"{'regs':>5s} {'fp64%':>6s} {'lsb':>5s}  DRAM B/unit"]
traffic = {}
for k, ms in agg.items():
    m = ms[0]
    dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    unit = UNITS.get(k)
    per_unit = f"{dram / unit[0]:.1f} per {unit[1]}" if unit else ""
    if unit:
        traffic[k] = {"dram_bytes_per_px" if "px" in unit[1] else "dram_bytes_per_unit": dram / unit[0],
                      "unit": unit[1], "launch_us_under_ncu": m["gpu__time_duration.sum"] / 1e3,
                      "dram_bytes": dram, "lts_bytes": m["lts__t_bytes.sum"]}
    lines.append(f"{k:22s} {len(ms):8d} {m['gpu__time_duration.sum'] / 1e3:9.1f} {dram / 1e6:9.1f} "
                 f"{m['lts__t_bytes.sum'] / 1e6:9.1f} {m['smsp__issue_active.avg.pct_of_peak_sustained_active']:7.1f} "
                 f"{m['sm__warps_active.avg.pct_of_peak_sustained_active']:6.1f} "
                 f"{m['launch__registers_per_thread']:5.0f} "
                 f"{m['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']:6.1f} "
                 f"{m['smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio']:5.1f}  {per_unit}")
lines += ["", "columns: issue% = smsp__issue_active (of active cycles), occ% = sm__warps_active, fp64% = "
          "sm__pipe_fp64_cycles_active, lsb = long-scoreboard stall cycles per issued instruction"]
open("profiles/r02_ncu_summary.txt", "w").write("\n".join(lines) + "\n")
json.dump(traffic, open("profiles/r02_dram_traffic.json", "w"), indent=1)
print("\n".join(lines))

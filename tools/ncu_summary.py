"""Summarise an ncu report (dev tool): per kernel duration / occupancy / issue,
top stall reasons, pipe use, and the instruction mix of the hottest segments.

python tools/ncu_summary.py report.ncu-rep [kernel-regex]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr = raw[0]
keys = {"gpu__time_duration.sum": "dur", "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%", "launch__registers_per_thread": "regs",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
        "smsp__inst_executed.sum": "inst", "l1tex__t_sector_hit_rate.pct": "L1hit%",
        "lts__t_sector_hit_rate.pct": "L2hit%"}
for r in raw[2:]:
    name = r[hdr.index("Kernel Name")]
    if kre and kre not in name:
        continue
    d = dict(zip(hdr, r))
    print("==", name[:60], " ".join(f"{v}={d.get(k, '?')}" for k, v in keys.items()))
    st = {}
    for h, v in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
            except ValueError:
                pass
    print("   stalls:", " ".join(f"{k}={v:.2f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
    pipes = []
    for h, v in d.items():
        if h.startswith("sm__inst_executed_pipe_") and h.endswith(".avg.pct_of_peak_sustained_active"):
            try:
                if float(v) > 2:
                    pipes.append(f"{h[len('sm__inst_executed_pipe_'):-len('.avg.pct_of_peak_sustained_active')]}={float(v):.1f}")
            except ValueError:
                pass
    print("   pipes:", " ".join(pipes))


def segments(kernel_regex, top=25):
    """Instruction mix of the hottest straight-line segments of one kernel."""
    rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass",
                                           "--kernel-name", f"regex:{kernel_regex}"))))
    hdr = rows[1]
    ie, src, ad = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Address")
    samp = hdr.index("Warp Stall Sampling (All Samples)")
    seen, out = set(), []
    for r in rows[2:]:
        if len(r) < len(hdr) or r[ad] in seen:
            continue
        try:
            n, sm = int(r[ie] or 0), int(r[samp] or 0)
        except ValueError:
            continue
        seen.add(r[ad])
        out.append((r[src].strip(), n, sm))
    tot = sum(o[1] for o in out) or 1
    tsm = sum(o[2] for o in out) or 1
    segs, cur = [], None
    for i, (s, n, sm) in enumerate(out):
        if cur and cur[2] == n:
            cur[1] = i
            cur[3] += n
            cur[4] += sm
        else:
            if cur:
                segs.append(cur)
            cur = [i, i, n, n, sm]
    segs.append(cur)
    segs.sort(key=lambda x: -x[3])
    print(f"-- {kernel_regex}: {tot} warp instructions")
    for i0, i1, n, t, sm in segs[:top]:
        ops = collections.Counter()
        for j in range(i0, i1 + 1):
            w = out[j][0].split()
            op = (w[1] if w and w[0].startswith("@") and len(w) > 1 else (w[0] if w else "?")).split(".")[0]
            ops[op] += 1
        print(f"[{i0}-{i1}] x{n} {t / tot * 100:5.1f}% inst {sm / tsm * 100:5.1f}% stall ", dict(ops.most_common(7)))


if len(sys.argv) > 3:
    segments(sys.argv[3])

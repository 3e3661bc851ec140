"""Attribute a kernel's executed instructions and warp-stall samples to
source lines / regions from an ncu report (--page source, cuda+sass mix).

python tools/ncu_attrib.py REPORT.ncu-rep KERNEL_REGEX [regions.json]
Prints per-line totals (top lines) and, with a regions file ({"name":
[[first_line, last_line], ...]}), per-region shares.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def load(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kernel}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    per_line = defaultdict(lambda: [0, 0, 0, ""])  # inst executed, samples, sass count, source
    line = None
    src = {}
    fname = ""
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            ie = hdr.index("Instructions Executed")
            sm = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr) - 5:
            continue
        if r[0]:
            line = (fname, int(r[0]))
            src[line] = r[1]
            continue
        if line is None:
            continue
        try:
            per_line[line][0] += int(r[ie])
            per_line[line][1] += int(r[sm])
            per_line[line][2] += 1
        except ValueError:
            pass
    for k in per_line:
        per_line[k][3] = src.get(k, "")
    return per_line


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    pl = load(rep, kernel)
    ti = sum(v[0] for v in pl.values()) or 1
    ts = sum(v[1] for v in pl.values()) or 1
    print(f"total warp-instructions executed {ti}, stall samples {ts}")
    if len(sys.argv) > 3:
        regions = json.load(open(sys.argv[3]))
        acc = {}
        for name, ranges in regions.items():
            i = s = 0
            for rg in ranges:
                f, a, b = (rg if len(rg) == 3 else [None] + list(rg))
                for (fn, ln), v in pl.items():
                    if (f is None or f == fn) and a <= ln <= b:
                        i += v[0]
                        s += v[1]
            acc[name] = (i, s)
        other_i = ti - sum(v[0] for v in acc.values())
        other_s = ts - sum(v[1] for v in acc.values())
        for name, (i, s) in list(acc.items()) + [("other", (other_i, other_s))]:
            print(f"{name:28s} inst {i / ti:6.1%}  stall-samples {s / ts:6.1%}")
    print("top lines by instructions:")
    for ln, v in sorted(pl.items(), key=lambda kv: -kv[1][0])[:40]:
        print(f"{ln[0][:14]:14s}{ln[1]:5d} inst {v[0] / ti:6.2%} samp {v[1] / ts:6.2%} sass {v[2]:4d}  {v[3].strip()[:80]}")


if __name__ == "__main__":
    main()

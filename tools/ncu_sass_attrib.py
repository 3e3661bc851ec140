"""Inline-aware attribution of a kernel's executed instructions and warp-stall
samples to source regions (dev tool).

ncu's source page attributes an inlined helper's SASS to the helper's own
line (a DP4A lands on sm_61_intrinsics.hpp whatever level called it).  This
tool reads ncu's per-SASS-instruction counts instead and maps every
instruction offset to its full inlining chain from `nvdisasm -g -gi` of the
same build, then assigns it to the innermost frame that falls into a
*classifying* region; frames inside *transparent* ranges (shared helpers such
as the int8 dot products and the top-2 update) are skipped so their
instructions count for the caller that inlined them.

python tools/ncu_sass_attrib.py REPORT.ncu-rep KERNEL_REGEX CUBIN MANGLED_NAME REGIONS.json

REGIONS.json: {"classify": {"name": [["file.cu", first, last], ...], ...},
               "transparent": [["file", first, last], ...]}
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

rep, kern, cubin, mangled, regions_path = sys.argv[1:6]
R = json.load(open(regions_path))

# ncu: per-SASS-instruction counts (runtime addresses; offsets from the first)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + kern, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
iA, iS, iE, iW = (hdr.index(k) for k in ("Address", "Source", "Instructions Executed",
                                          "Warp Stall Sampling (All Samples)"))
sass = []
for r in rows:
    if len(r) == len(hdr) and r[0].startswith("0x"):
        sass.append((int(r[iA], 16), r[iS].strip(), float(r[iE] or 0), float(r[iW] or 0)))
base = sass[0][0]

# nvdisasm: offset -> inlining chain [(file, line) innermost first]
dis = subprocess.run(["nvdisasm", "-g", "-gi", cubin], capture_output=True, text=True).stdout
sec = dis.split(".text." + mangled + ":", 1)[1]
sec = sec.split("\n\t.section", 1)[0]
# consecutive "//## File A, line a inlined at B, line b" lines form one chain
# (innermost callee first, each line adding its call site)
chain, where, text = [], {}, {}
fre = re.compile(r'"([^"]+)", line (\d+)')
prev_dir = False
for ln in sec.splitlines():
    if ln.lstrip().startswith("//## File"):
        fr = [(f.split("/")[-1], int(n)) for f, n in fre.findall(ln)]
        if not prev_dir:
            chain = fr
        else:
            chain = chain + fr[1:]
        prev_dir = True
        continue
    prev_dir = False
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", ln)
    if m:
        off = int(m.group(1), 16)
        where[off] = chain
        text[off] = m.group(2).split()[0] if m.group(2).split() else ""


def inside(fl, spans):
    return any(fl[0] == f and a <= fl[1] <= b for f, a, b in spans)


def region(ch):
    for fl in ch:  # innermost first
        if inside(fl, R.get("transparent", [])):
            continue
        for name, spans in R["classify"].items():
            if inside(fl, spans):
                return name
    return "other"


agg = defaultdict(lambda: [0.0, 0.0])
mism = 0
for addr, src, ie, ws in sass:
    off = addr - base
    if off in text and src.split() and text[off] != src.split()[0].lstrip("@!P0123456789T").strip() \
            and not src.split()[0].startswith("@"):
        mism += 1
    a = agg[region(where.get(off, []))]
    a[0] += ie
    a[1] += ws
ti = sum(a[0] for a in agg.values())
ts = sum(a[1] for a in agg.values())
print(f"# {kern}: {len(sass)} SASS instructions, {ti:.4g} warp-instructions executed, {ts:.0f} stall samples")
print(f"# opcode mismatches between the report and this build's disassembly: {mism}")
print(f"{'region':62s} {'inst':>7s} {'stall':>7s}")
for name, (ie, ws) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{name:62s} {100 * ie / ti:6.1f}% {100 * ws / max(ts, 1):6.1f}%")
